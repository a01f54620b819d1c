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
// two are prefetched one frame ahead in registers; wider windows (the first
// frame, flat posteriors) load their extra rounds in the frame itself.
//
// SCALE.  sum_s alpha_t beta'_t = Z for every frame, so one reference
// exponent -- the magnitude of the warp's first frame, from its largest
// block (block exponent sum plus the exponent of the block's largest
// product; all-zero blocks ignored) -- scales all the warp's frames into
// fp32 range.  Each frame's posteriors are normalised by their own sum z_t,
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
  size_t segv, sege;    // per lattice warp: Tmax * kLatStates values, Tmax * 32 exponents
  int S;                // lattice states
  int nblk;             // lane blocks holding states: ceil(S / kSpl)

  __device__ __forceinline__ size_t voff(int m, int t) const {
    return (size_t)(m >> 5) * segv + (size_t)t * kLatStates + (size_t)(m & 31) * kSpl;
  }
  __device__ __forceinline__ size_t eoff(int m, int t) const {
    return (size_t)(m >> 5) * sege + (size_t)t * 32 + (m & 31);
  }
  // block m of frame t: values and exponent sum (INT_MIN: outside the lattice)
  __device__ __forceinline__ void load(int m, int t, bool want, V (&va)[kSpl], V (&vb)[kSpl],
                                       int &e) const {
    e = INT_MIN;
    if (want && m < nblk) {
      ldv_cg(A + voff(m, t), va);
      ldv_cg(B + voff(m, t), vb);
      e = __ldcg(EA + eoff(m, t)) + __ldcg(EB + eoff(m, t));
    }
  }
  // the warp's reference exponent from frame t (all blocks)
  __device__ __forceinline__ int reference(int t, int lane) const {
    int ref = INT_MIN;
    for (int m = lane; m < nblk; m += 32) {
      V va[kSpl], vb[kSpl], pp[kSpl];
      int e;
      load(m, t, true, va, vb, e);
#pragma unroll
      for (int k = 0; k < kSpl; ++k) pp[k] = va[k] * vb[k];
      const V pm = tree_max<kSpl, V>(pp);
      if (pm > (V)0) ref = max(ref, e + Pow2<V>::expo(pm));
    }
    ref = __reduce_max_sync(0xffffffffu, ref);
    return ref == INT_MIN ? 0 : ref;   // no mass: the guard rejects the utterance
  }
};

// Scaled posteriors of one lane block into q (float) and their band edges
// into lo / hi.
template <class V>
__device__ __forceinline__ void band_block(const V (&va)[kSpl], const V (&vb)[kSpl], int e,
                                           int ref, int m, float (&q)[kSpl], int &lo, int &hi) {
  const V sc = e == INT_MIN ? (V)0 : pow2_clamped<V>(e - ref);
#pragma unroll
  for (int k = 0; k < kSpl; ++k) q[k] = (float)(va[k] * vb[k] * sc);
  int first = kSpl, last = -1;
#pragma unroll
  for (int k = kSpl - 1; k >= 0; --k)
    if (q[k] > kBandEps) first = k;
#pragma unroll
  for (int k = 0; k < kSpl; ++k)
    if (q[k] > kBandEps) last = k;
  if (last >= 0) {
    lo = min(lo, m * kSpl + first);
    hi = max(hi, m * kSpl + last);
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
