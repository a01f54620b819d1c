// Block floating point for a lane's consecutive lattice states: the lane
// keeps its states in V (float: the fast tier; double: the wide-range tier)
// with one power-of-two exponent, renormalised so that its largest value lies
// in [1, 2); values of a neighbouring lane are brought onto this lane's
// exponent by an exact power-of-two factor.  Only integer exponents
// accumulate, so no rounding enters the scale factors.
#pragma once

#include "common.cuh"

namespace w2l {

constexpr int kStride = 33;  // Et row pitch in shared memory: odd, > 32 (column N holds 0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- per-type power-of-two helpers (exact scale factors, no subnormals)
template <class V>
struct Pow2;
template <>
struct Pow2<float> {
  static constexpr int kMaxExp = 127;    // 2^k representable for |k| <= 127
  static constexpr int kLaneGap = 64;    // rebase a lane when its neighbour dominates by more
  static constexpr float kFlush = kFlushNats;   // exp() of a weight below -kFlush -> 0
  __device__ __forceinline__ static float p2(int k) {
    k = max(min(k, 127), -127);
    return __int_as_float((k + 127) << 23);
  }
  __device__ __forceinline__ static int expo(float x) {
    return ((__float_as_int(x) >> 23) & 0xff) - 127;
  }
  __device__ __forceinline__ static float ex(float x) { return __expf(x); }
};
template <>
struct Pow2<double> {
  static constexpr int kMaxExp = 1023;
  static constexpr int kLaneGap = 512;
  static constexpr float kFlush = kFlushNats64;
  __device__ __forceinline__ static double p2(int k) {
    k = max(min(k, 1023), -1022);
    return __longlong_as_double((long long)(k + 1023) << 52);
  }
  __device__ __forceinline__ static int expo(double x) {
    return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
  }
  __device__ __forceinline__ static double ex(double x) { return exp(x); }
};

// max over a register array as a balanced tree (depth log2 SPL, not SPL)
template <int SPL, class V>
__device__ __forceinline__ V tree_max(const V (&v)[SPL]) {
  V m[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) m[k] = v[k];
#pragma unroll
  for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < SPL; k += 2 * w) m[k] = fmax(m[k], m[k + w]);
  return fmax(m[0], (V)0);
}

// scale the lane block so its largest value lies in [1, 2) and fold the power
// of two into the lane exponent (branch-free; an all-zero block stays zero and
// is marked dead with kNegExp)
template <int SPL, class V>
__device__ __forceinline__ void lane_renorm(V (&v)[SPL], int &ex) {
  const V mx = tree_max<SPL, V>(v);
  const int kx = Pow2<V>::expo(mx);           // -127 / -1023 for mx == 0
  const V sc = Pow2<V>::p2(-kx);
#pragma unroll
  for (int k = 0; k < SPL; ++k) v[k] *= sc;
  ex = mx > (V)0 ? ex + kx : kNegExp;
}

// The power-of-two factor that brings the neighbour lane's values (exponent
// nbe) onto this lane's exponent.  check (the step after a renormalisation,
// when exponents may have moved): if the neighbour dominates by more than
// kLaneGap, rebase this lane onto it first (a dead lane is adopted this
// way).  Otherwise a dead lane adopts the neighbour's exponent and the shift
// is clamped to the type's range.  The factor stays valid until the next
// renormalisation.
template <int SPL, class V>
__device__ __forceinline__ V align_factor(int nbe, V (&v)[SPL], int &ex, bool check) {
  if (check) {
    int dd = nbe - ex;
    if (dd > Pow2<V>::kLaneGap) {
      const V sc = Pow2<V>::p2(max(-dd, -Pow2<V>::kMaxExp));
#pragma unroll
      for (int k = 0; k < SPL; ++k) v[k] *= sc;
      ex = nbe;
      dd = 0;
    }
    return Pow2<V>::p2(dd);
  }
  ex = ex == kNegExp ? nbe : ex;
  return Pow2<V>::p2(min(nbe - ex, Pow2<V>::kMaxExp - 1));
}

}  // namespace w2l
