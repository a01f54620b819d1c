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
// exceeds kBandEps, the states carrying mass at t + 1 lie in
// [lo_t, hi_t + kMaxStep]: a warp that walks consecutive frames reads its
// first frame whole and afterwards only that window -- about 100 of the
// 601 CTC states at the bench shape.  The mass outside the window stays
// below S kBandEps per frame (~1e-11 of the frame's mass), far inside the
// 1e-4 tolerance.
//
// LANES.  Each frame, lane l takes the window's lane blocks mlo + l + 32 r
// (rounds r = 0, 1, ...): two rounds cover 64 blocks (256 states), and those
// two are prefetched one frame ahead in registers; wider windows (a warp's
// first frame, flat posteriors) load their extra rounds in the frame itself.
//
// SCALE.  sum_s alpha_t beta'_t = Z for every frame, so one reference
// exponent -- the magnitude of the CTA's first frame, from its largest
// block (block exponent sum plus the exponent of the block's largest
// product; all-zero blocks ignored), found by the CTA's warps together --
// scales all the CTA's frames into fp32 range.  (A block's exponent alone
// does not bound its values: between renormalisations a block may carry a
// dominant neighbour's mass scaled onto its exponent by up to 2^kLaneGap, so
// a warp's first frame is read whole.)  Each frame's posteriors are normalised by their own sum z_t,
// and ref + log2 z_t is the frame's log2-normaliser the guard checks.
#pragma once

#include <climits>

#include "lattice.cuh"

namespace w2l {

constexpr float kBandEps = 0x1p-44f;   // band threshold (scaled posterior units)
constexpr int kBandRounds = 2;         // prefetched lane-block rounds (64 blocks)

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
  // this warp's share (blocks warp*32 + lane + 32*nwarps*k) of the largest
  // block magnitude of frame t: block exponent sum plus the exponent of the
  // block's largest product (all-zero blocks ignored)
  __device__ __forceinline__ int magnitude_part(int t, int warp, int nwarps, int lane) const {
    const Frame f = frame(t);
    int mag = INT_MIN;
    for (int m = warp * 32 + lane; m < nblk; m += 32 * nwarps) {
      V va[kSpl], vb[kSpl], pp[kSpl];
      int e;
      load(f, m, true, va, vb, e);
#pragma unroll
      for (int k = 0; k < kSpl; ++k) pp[k] = va[k] * vb[k];
      const V pm = tree_max<kSpl, V>(pp);
      if (pm > (V)0) mag = max(mag, e + Pow2<V>::expo(pm));
    }
    return __reduce_max_sync(0xffffffffu, mag);
  }
  // next frame's window (lane blocks) from this frame's band (blocks lo..hi
  // holding a scaled posterior above kBandEps); mass moves by <= step states
  __device__ __forceinline__ void next_window(int lo, int hi, int step, int &mlo,
                                              int &mhi) const {
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (hi >= lo) {
      mlo = lo;
      mhi = min(hi * kSpl + kSpl - 1 + step, S - 1) / kSpl;
    } else {   // nothing above the threshold (cannot happen for a finite loss): read all
      mlo = 0;
      mhi = nblk - 1;
    }
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

// Token sums of a frame's posteriors, deterministic: each state's normalised
// posterior (in [0, 1]) is added to its token's bin as a 2^-30 fixed-point
// integer (shared-memory integer atomics commute, so the sum does not depend
// on the order the lanes arrive in).  Rounding: 2^-31 per state, ~1e-7 on a
// gradient entry at L = 300.  tok4: the tokens of the block's states, one
// byte each, 0xff for none (CTC blanks are summed separately, as a float).
constexpr float kFixScale = 0x1p30f;
constexpr float kFixInv = 0x1p-30f;
constexpr int kTokWords = kSpl / 4;   // token words per lane block (4 bytes each)
__device__ __forceinline__ void band_scatter(const float (&q)[kSpl], float inv, const unsigned *tok,
                                             unsigned *bins) {
#pragma unroll
  for (int k = 0; k < kSpl; ++k) {
    const unsigned tk = (tok[k >> 2] >> (8 * (k & 3))) & 0xffu;
    if (tk != 0xffu && q[k] > 0.f) atomicAdd(bins + tk, __float2uint_rn(q[k] * inv * kFixScale));
  }
}

}  // namespace w2l
