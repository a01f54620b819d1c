// Block floating point for a lane's consecutive lattice states: the lane
// keeps its states in fp32 with one power-of-two exponent, renormalised so
// that its largest value lies in [1, 2); values of a neighbouring lane are
// brought onto this lane's exponent by an exact power-of-two factor.  Only
// integer exponents accumulate, so no rounding enters the scale factors.
#pragma once

#include "common.cuh"

namespace w2l {

constexpr int kStride = 33;  // Et row pitch in shared memory: odd, > 32 (column N holds 0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// max over a register array as a balanced tree (depth log2 SPL, not SPL)
template <int SPL>
__device__ __forceinline__ float tree_max(const float (&v)[SPL]) {
  float m[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) m[k] = v[k];
#pragma unroll
  for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < SPL; k += 2 * w) m[k] = fmaxf(m[k], m[k + w]);
  return fmaxf(m[0], 0.f);
}

// scale the lane block so its largest value lies in [1, 2) and fold the power
// of two into the lane exponent (branch-free; an all-zero block stays zero and
// is marked dead with kNegExp)
template <int SPL>
__device__ __forceinline__ void lane_renorm(float (&v)[SPL], int &ex) {
  const float mx = tree_max<SPL>(v);
  const int kx = exponent_of(mx);           // -127 for mx == 0
  const float sc = pow2f_fast(-kx);
#pragma unroll
  for (int k = 0; k < SPL; ++k) v[k] *= sc;
  ex = mx > 0.f ? ex + kx : kNegExp;
}

// The power-of-two factor that brings the neighbour lane's values (exponent
// nbe) onto this lane's exponent.  check (the step after a renormalisation,
// when exponents may have moved): if the neighbour dominates by more than
// 2^64, rebase this lane onto it first (a dead lane is adopted this way).
// Otherwise a dead lane adopts the neighbour's exponent and the shift is
// clamped to 2^126.  The factor stays valid until the next renormalisation.
template <int SPL>
__device__ __forceinline__ float align_factor(int nbe, float (&v)[SPL], int &ex, bool check) {
  if (check) {
    int dd = nbe - ex;
    if (dd > 64) {
      const float sc = pow2f_fast(max(-dd, -127));
#pragma unroll
      for (int k = 0; k < SPL; ++k) v[k] *= sc;
      ex = nbe;
      dd = 0;
    }
    return pow2f_fast(dd);
  }
  ex = ex == kNegExp ? nbe : ex;
  return pow2f_fast(min(nbe - ex, 126));
}

}  // namespace w2l
