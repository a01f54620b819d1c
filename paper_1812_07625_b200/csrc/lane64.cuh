// Float64 lane blocks for the linear-lattice recursions (ASG fac, CTC).
//
// A lane keeps SPL consecutive lattice states as doubles that share one
// power-of-two lane exponent.  fp32 is not enough here: along a target
// lattice the forward/backward values of neighbouring states differ by
// ~2^10 per state for log-softmax-like emissions (each state skipped saves
// one emission), so one lane block can span > 2^126 and the posterior-
// relevant state underflows.  The 11-bit exponent of fp64 gives ~2^1000 of
// headroom per block, and rows are stored as the HIGH 32 bits of each double
// (sign, 11-bit exponent, 20-bit mantissa: relative error <= 2^-21 after
// mid-point reconstruction) -- the same bytes as fp32 rows.
#pragma once

#include "chunk.cuh"

namespace w2l {

constexpr int kRenormD = 8;  // frames between fp64 lane renormalisations

__device__ __forceinline__ int exponent_of_d(double x) {
  return (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
}
// 2^k for k in [-1022, 1023]; k <= -1023 gives 0 (branch-free)
__device__ __forceinline__ double pow2d_fast(int k) {
  k = max(min(k, 1023), -1023);
  return __longlong_as_double((long long)(k + 1023) << 52);
}

template <int SPL>
__device__ __forceinline__ double tree_max_d(const double (&v)[SPL]) {
  double m[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) m[k] = v[k];
#pragma unroll
  for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < SPL; k += 2 * w) m[k] = fmax(m[k], m[k + w]);
  return fmax(m[0], 0.0);
}

// renormalise a lane block: scale so the largest value lies in [1, 2).  The
// maximum is taken over the high words as integers (for non-negative doubles
// the bit pattern is monotonic), which is much cheaper than fp64 compares.
template <int SPL>
__device__ __forceinline__ void lane_renorm_d(double (&v)[SPL], int &ex) {
  int m[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) m[k] = __double2hiint(v[k]);
#pragma unroll
  for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < SPL; k += 2 * w) m[k] = max(m[k], m[k + w]);
  const int kx = ((m[0] >> 20) & 0x7ff) - 1023;   // -1023 for an all-zero block
  const double sc = pow2d_fast(-kx);
#pragma unroll
  for (int k = 0; k < SPL; ++k) v[k] *= sc;
  ex = m[0] > 0 ? ex + kx : kNegExp;
}

// store the high words of a lane's doubles (lane-major, SPL/2 8-byte stores)
template <int SPL>
__device__ __forceinline__ void lane_store_hi(const double (&v)[SPL], int ex, float *out,
                                              int *oute, int lane, int t) {
  static_assert(SPL % 2 == 0, "SPL must be even");
  constexpr int lp = SPL * 32;
  int2 *o = reinterpret_cast<int2 *>(out + t * lp + lane * SPL);
#pragma unroll
  for (int k = 0; k < SPL / 2; ++k) o[k] = make_int2(__double2hiint(v[2 * k]), __double2hiint(v[2 * k + 1]));
  oute[t * 32 + lane] = ex;
}

__device__ __forceinline__ double from_hi(int hi) {
  return __hiloint2double(hi, hi ? (int)0x80000000 : 0);   // mid-point of the dropped bits
}

template <int SPL>
__device__ __forceinline__ void lane_load_hi(double (&v)[SPL], const float *row, int lane) {
  const int2 *o = reinterpret_cast<const int2 *>(row + lane * SPL);
#pragma unroll
  for (int k = 0; k < SPL / 2; ++k) {
    const int2 x = o[k];
    v[2 * k] = from_hi(x.x);
    v[2 * k + 1] = from_hi(x.y);
  }
}

// align the neighbour lane's value to this lane's exponent (see
// align_neighbour): the checked form rebases a lane dominated by > 2^512,
// the branch-free form lets a dead lane adopt the neighbour's exponent
template <int SPL>
__device__ __forceinline__ double align_neighbour_d(double nb, int nbe, double (&v)[SPL],
                                                    int &ex, bool check) {
  if (check) {
    int dd = nbe - ex;
    if (dd > 512) {
      const double sc = pow2d_fast(-dd);
#pragma unroll
      for (int k = 0; k < SPL; ++k) v[k] *= sc;
      ex = nbe;
      dd = 0;
    }
    return nb * pow2d_fast(dd);
  }
  ex = ex == kNegExp ? nbe : ex;
  return nb * pow2d_fast(min(nbe - ex, 1000));
}

// floor(log2(max_k a[k] b[k])) + ea + eb (kNegExp if dead or all-zero)
template <int SPL>
__device__ __forceinline__ int lane_pair_exponent_d(const double (&a)[SPL],
                                                    const double (&b)[SPL], int ea, int eb) {
  double p[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) p[k] = a[k] * b[k];
  const double m = tree_max_d<SPL>(p);
  if (!(m > 0.0) || ea <= kNegExp / 2 || eb <= kNegExp / 2) return kNegExp;
  return ea + eb + exponent_of_d(m);
}

// raw high words of a stored row (lane-major)
template <int SPL>
__device__ __forceinline__ void lane_load_int(int (&v)[SPL], const float *row, int lane) {
  const int2 *o = reinterpret_cast<const int2 *>(row + lane * SPL);
#pragma unroll
  for (int k = 0; k < SPL / 2; ++k) {
    const int2 x = o[k];
    v[2 * k] = x.x;
    v[2 * k + 1] = x.y;
  }
}

__device__ __forceinline__ double hi_to_d(int hi) { return __hiloint2double(hi, 0); }

// alpha*beta products of a lane's states from stored high words (truncated,
// relative error < 2^-19) and the exponent of the lane's largest product plus
// the lane exponents (kNegExp if either side is dead or all-zero); the
// largest product is found on the products' high words as integers
template <int SPL>
__device__ __forceinline__ int lane_products(const int (&ah)[SPL], const int (&bh)[SPL], int ea,
                                             int eb, double (&p)[SPL]) {
  int m = 0;
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    p[k] = hi_to_d(ah[k]) * hi_to_d(bh[k]);
    m = max(m, __double2hiint(p[k]));
  }
  return (m > 0 && ea > kNegExp / 2 && eb > kNegExp / 2) ? ea + eb + ((m >> 20) & 0x7ff) - 1023
                                                          : kNegExp;
}

// chunk conversion to double Et rows (the float staging holds raw emissions;
// values are the float Et of stage_convert, widened exactly)
__device__ __forceinline__ void stage_convert_d(const float *raw, double *dbuf, const ChainCtx &c,
                                                int rows, double *shift_sum = nullptr) {
  cp_async_wait<0>();
  __syncwarp();
  if (c.lane < rows) {
    const float *r = raw + c.lane * kStride;
    double *d = dbuf + c.lane * kStride;
    float m = -CUDART_INF_F;
    for (int i = 0; i < c.N; ++i) m = fmaxf(m, r[i]);
    for (int i = 0; i < c.N; ++i) d[i] = (double)expf(r[i] - m);
    for (int i = c.N; i < kStride; ++i) d[i] = 0.0;
    if (shift_sum) *shift_sum += (double)m;
  }
  __syncwarp();
}

}  // namespace w2l
