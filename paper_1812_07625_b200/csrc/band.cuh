// Band-limited posterior walk for the gradient kernels (CTC lattice and ASG
// fac lattice).
//
// The chains store every frame's alpha / beta' rows warp-major: lane block m
// (kSpl consecutive states starting at m kSpl) of frame t lives in lattice
// warp m / 32, lane m % 32, with one power-of-two exponent per block.  The
// posterior of state s at frame t is alpha_t(s) beta'_t(s) / Z.
//
// BAND.  Posterior mass only moves forward along a left-to-right lattice: a
// path in state s at frame t is in s .. s + kMaxStep at t + 1 (CTC: 2, fac:
// 1).  So if [lo_t, hi_t] holds every state of frame t whose scaled posterior
// exceeds kBandEps, the states carrying mass at t + k lie in
// [lo_t, hi_t + k kMaxStep], up to the mass outside [lo_t, hi_t] at t, which
// stays below S kBandEps (~1e-11 of a frame's mass; the window's own mass
// flows within the widened window), far inside the 1e-4 tolerance.  About
// 100 of the 601 CTC states at the bench shape are read per frame.
//
// FIRST FRAMES.  The CTA reads its first frame t0 whole, one lane block per
// thread: the largest block magnitude gives the reference exponent and the
// blocks above kBandEps the band of t0.  The window of a warp's first frame
// ta is that band widened by ta - t0 frames of movement.
//
// LANES.  Each frame, lane l takes the window's lane blocks mlo + l + 32 r
// (rounds r = 0, 1, ...).  Round 0 arrives through the prefetch ring below;
// wider windows (flat posteriors, a late warp's first frame) load their
// extra rounds in the frame itself.
//
// SCALE.  sum_s alpha_t beta'_t = Z for every frame, so one reference
// exponent -- the magnitude of the CTA's first frame, from its largest
// block (block exponent sum plus the exponent of the block's largest
// product; all-zero blocks ignored) -- scales all the CTA's frames into fp32
// range.  (A block's exponent alone does not bound its values: between
// renormalisations a block may carry a dominant neighbour's mass scaled onto
// its exponent by up to 2^kLaneGap, so the first frame is read whole.)  Each
// frame's posteriors are normalised by their own sum z_t, and ref + log2 z_t
// is the frame's log2-normaliser the guard checks.
#pragma once

#include <climits>

#include "lattice.cuh"

namespace w2l {

constexpr float kBandEps = 0x1p-44f;   // band threshold (scaled posterior units)

// Scaled posteriors of one lane block into q (float); a block above the band
// threshold widens the band [lo, hi] (lane blocks).
template <class V>
__device__ __forceinline__ void band_block(const V (&va)[kSpl], const V (&vb)[kSpl], int e,
                                           int ref, int m, float (&q)[kSpl], int &lo, int &hi) {
  const V sc = e == INT_MIN ? (V)0 : pow2_clamped<V>(e - ref);
#pragma unroll
  for (int k = 0; k < kSpl; ++k) q[k] = (float)(va[k] * vb[k] * sc);
  if (tree_max<kSpl, float>(q) > kBandEps) {
    lo = min(lo, m);
    hi = max(hi, m);
  }
}

template <class V>
struct BandRows {
  const V *A, *B;       // this utterance's alpha / beta' rows (lattice warp 0)
  const int *EA, *EB;   // their block exponents
  uint32_t segv, sege;  // per lattice warp: Tmax * kLatStates values, Tmax * 32 exponents
  int S;                // lattice states
  int nblk;             // lane blocks holding states: ceil(S / kSpl)

  // one frame's rows; blocks are addressed by 32-bit offsets from them
  struct Frame {
    const V *a, *b;
    const int *ea, *eb;
  };
  __device__ __forceinline__ Frame frame(int t) const {
    return {A + (size_t)t * kLatStates, B + (size_t)t * kLatStates, EA + (size_t)t * 32,
            EB + (size_t)t * 32};
  }
  __device__ __forceinline__ uint32_t voff(int m) const {
    return (uint32_t)(m >> 5) * segv + (uint32_t)(m & 31) * kSpl;
  }
  __device__ __forceinline__ uint32_t eoff(int m) const {
    return (uint32_t)(m >> 5) * sege + (uint32_t)(m & 31);
  }
  // block m of a frame: values and exponent sum (INT_MIN: not loaded)
  __device__ __forceinline__ void load(const Frame &f, int m, bool want, V (&va)[kSpl],
                                       V (&vb)[kSpl], int &e) const {
    e = INT_MIN;
    if (want && m < nblk) {
      const uint32_t vo = voff(m), eo = eoff(m);
      ldv_cg(f.a + vo, va);
      ldv_cg(f.b + vo, vb);
      e = __ldcg(f.ea + eo) + __ldcg(f.eb + eo);
    }
  }
  // the window (lane blocks) of a frame `ext` states of mass movement after
  // a frame whose band (blocks lo..hi holding a scaled posterior above
  // kBandEps) is known
  __device__ __forceinline__ void window(int lo, int hi, int ext, int &mlo, int &mhi) const {
    if (hi >= lo) {
      mlo = lo;
      mhi = min(hi * kSpl + kSpl - 1 + ext, S - 1) / kSpl;
    } else {   // nothing above the threshold (cannot happen for a finite loss): read all
      mlo = 0;
      mhi = nblk - 1;
    }
  }
  // the same from a warp's per-lane band edges
  __device__ __forceinline__ void next_window(int lo, int hi, int ext, int &mlo,
                                              int &mhi) const {
    window(__reduce_min_sync(0xffffffffu, lo), __reduce_max_sync(0xffffffffu, hi), ext, mlo, mhi);
  }
  // The CTA's first frame t0, one lane block per thread (nblk <= blockDim.x):
  // the reference exponent and the band of blocks above kBandEps, from which
  // every warp's first windows follow (frame t0 + k: the band widened by k
  // steps of mass movement).  sh: nwarps + 2 ints of shared memory.
  __device__ __forceinline__ void cta_first_band(int t0, int nwarps, int *sh, int &ref, int &blo,
                                                 int &bhi) const {
    const int m = threadIdx.x, lane = m & 31, warp = m >> 5;
    V va[kSpl], vb[kSpl];
    int e;
    load(frame(t0), m, true, va, vb, e);
    int mag = INT_MIN;
    if (e != INT_MIN) {
      V pp[kSpl];
#pragma unroll
      for (int k = 0; k < kSpl; ++k) pp[k] = va[k] * vb[k];
      const V pm = tree_max<kSpl, V>(pp);
      if (pm > (V)0) mag = e + Pow2<V>::expo(pm);
    }
    mag = __reduce_max_sync(0xffffffffu, mag);
    if (lane == 0) sh[warp] = mag;
    if (threadIdx.x == 0) {
      sh[nwarps] = INT_MAX;
      sh[nwarps + 1] = -1;
    }
    __syncthreads();
    ref = INT_MIN;
    for (int q = 0; q < nwarps; ++q) ref = max(ref, sh[q]);
    if (ref == INT_MIN) ref = 0;   // no mass: the guard rejects the utterance
    int lo = INT_MAX, hi = -1;
    if (e != INT_MIN) {
      float q[kSpl];
      band_block<V>(va, vb, e, ref, m, q, lo, hi);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0 && hi >= lo) {
      atomicMin(&sh[nwarps], lo);
      atomicMax(&sh[nwarps + 1], hi);
    }
    __syncthreads();
    blo = sh[nwarps];
    bhi = sh[nwarps + 1];
  }
};

// PREFETCH.  A warp's frames go through a pipeline two frames deep: while
// it works on frame t, the first round (32 lane blocks) of the windows of
// frames t + 1 and t + 2 is on its way into a per-warp shared-memory ring
// (cp.async; no registers held).  The window of frame t + 2 is frame t's
// band widened by two steps, which contains frame t + 1's band widened by
// one.  Each lane copies and later reads only its own block, so the
// per-thread cp.async groups need no warp barrier: group g holds frame g's
// copies (one group committed per frame, empty ones included), and
// wait_group 1 at frame t leaves only frame t + 1's group in flight.
constexpr int kPfSlots = 3;
template <class V>
__host__ __device__ constexpr size_t band_pf_bytes() {   // per warp
  return (size_t)kPfSlots * 32 * (2 * kSpl * sizeof(V) + 2 * sizeof(int));
}
template <class V>
struct BandPf {
  V *a, *b;      // [kPfSlots][32][kSpl]
  int *ea, *eb;  // [kPfSlots][32]
  __device__ __forceinline__ void init(unsigned char *base) {
    a = reinterpret_cast<V *>(base);
    b = a + kPfSlots * 32 * kSpl;
    ea = reinterpret_cast<int *>(b + kPfSlots * 32 * kSpl);
    eb = ea + kPfSlots * 32;
  }
  // block m of frame f into this lane's entry of slot s (nothing outside
  // the window or the lattice)
  __device__ __forceinline__ void issue(const BandRows<V> &br,
                                        const typename BandRows<V>::Frame &f, int m, bool want,
                                        int s, int lane) const {
    if (want && m < br.nblk) {
      const uint32_t vo = br.voff(m), eo = br.eoff(m);
      const int i = s * 32 + lane;
      constexpr int kV = 16 / (int)sizeof(V);   // values per 16-byte copy
#pragma unroll
      for (int k = 0; k < kSpl; k += kV) {
        cp_async16_ca(a + i * kSpl + k, f.a + vo + k);
        cp_async16_ca(b + i * kSpl + k, f.b + vo + k);
      }
      cp_async4(ea + i, f.ea + eo);
      cp_async4(eb + i, f.eb + eo);
    }
  }
  // this lane's block of slot s (e = INT_MIN: none)
  __device__ __forceinline__ void take(int s, int lane, bool want, V (&va)[kSpl], V (&vb)[kSpl],
                                       int &e) const {
    e = INT_MIN;
    if (want) {
      const int i = s * 32 + lane;
      ldv(a + i * kSpl, va);
      ldv(b + i * kSpl, vb);
      e = ea[i] + eb[i];
    }
  }
};


// Token sums of a frame's posteriors, deterministic: each state's normalised
// posterior (in [0, 1]) is added to its token's bin as a 2^-30 fixed-point
// integer (shared-memory integer atomics commute, so the sum does not depend
// on the order the lanes arrive in).  Rounding: 2^-31 per state, ~1e-7 on a
// gradient entry at L = 300.  tok4: the tokens of the block's states, one
// byte each, 0xff for none (CTC blanks are summed separately, as a float).
constexpr float kFixScale = 0x1p30f;
constexpr float kFixInv = 0x1p-30f;
constexpr int kTokWords = kSpl / 4;   // token words per lane block (4 bytes each)
// kOddOnly: only the odd states of a block carry labels (CTC: the even ones
// are blanks), so only they are scattered.
template <bool kOddOnly = false>
__device__ __forceinline__ void band_scatter(const float (&q)[kSpl], float inv, const unsigned *tok,
                                             unsigned *bins) {
#pragma unroll
  for (int k = kOddOnly ? 1 : 0; k < kSpl; k += kOddOnly ? 2 : 1) {
    const unsigned tk = (tok[k >> 2] >> (8 * (k & 3))) & 0xffu;
    if (tk != 0xffu && q[k] > 0.f) atomicAdd(bins + tk, __float2uint_rn(q[k] * inv * kFixScale));
  }
}

}  // namespace w2l
