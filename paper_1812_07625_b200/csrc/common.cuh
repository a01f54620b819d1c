// Shared device helpers for the sm_100a sequence-criterion kernels.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/w2l_criterion.h"

namespace w2l {

// Internal per-utterance statuses of the precision tiers: the fp32
// scaled-linear tier failed its guard (-> the fp64 scaled-linear tier), and
// the fp64 tier failed too (-> the float64 log-domain kernel, exact.cu).
constexpr int kNeedsF64 = 100;
constexpr int kNeedsLog = 101;
constexpr int kNeedsExact = kNeedsF64;   // "the fp32 path could not take it"

// exp(x) of an fp32 weight flushes to zero below about -87.3 nats; the fast
// path sends any input whose weights (emissions relative to their frame
// maximum, transitions relative to their maximum) fall below -kFlushNats to
// the float64 kernel, since a flush applied identically to both directions
// would be invisible to the forward/backward consistency guard
constexpr float kFlushNats = 80.f;
constexpr float kFlushNats64 = 700.f;   // the same for double (exp underflows near -708)

// Precision routing.  The fp32 tier fails its guard on peaky emissions
// (relevant lattice states more than 2^126 apart inside a 4-state lane
// block), and the chains are latency-bound: a batch run through fp32 and
// then (for its failures) through fp64 costs both passes, whatever the
// number of failures.  em_check counts the frame rows whose spread
// max - min exceeds kRouteNats* (and kFlushNats: an fp32 weight that would
// flush), and the fp32 chain sends the WHOLE batch straight to the fp64
// tier when any row would flush or more than a quarter of the rows are that
// wide.  Calibrated on log_softmax(s N(0,1)) emissions (N = 30): ASG fails
// most utterances from s = 5 (spread ~20 nats), CTC from s = 10 (~41 nats).
// Results do not depend on the routing (both tiers are guarded).
constexpr int kRouteWords = 4;
constexpr float kRouteNatsAsg = 16.f;
constexpr float kRouteNatsCtc = 32.f;
__device__ __forceinline__ bool route_to_f64(const int *route) {
  if (!route) return false;
  const int rows = route[0], wide = route[1], hard = route[2];
  return hard > 0 || 4 * wide > rows;
}
constexpr int kWarp = 32;
constexpr int kChunk = 32;            // frames per staged emission chunk
constexpr int kNegExp = -(1 << 24);   // exponent of an all-zero lane block

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ inline size_t align_up(size_t x, size_t m) { return (x + m - 1) / m * m; }


// ------------------------------------------------------------ pow2 math --
// Exact power-of-two rescaling keeps the scaled linear-domain recursions
// free of rounding in the scale factors: only integer exponents accumulate.

// 2^k without branches for k <= 127; k <= -127 gives 0 (no subnormals).
__device__ __forceinline__ float pow2f_fast(int k) {
  k = max(min(k, 127), -127);
  return __int_as_float((k + 127) << 23);
}

// floor(log2(x)) for a positive normal float; subnormals map to -127.
__device__ __forceinline__ int exponent_of(float x) {
  return ((__float_as_int(x) >> 23) & 0xff) - 127;
}

// ------------------------------------------------------------ log-space --
// logaddexp on doubles with -inf handled explicitly.
__device__ __forceinline__ double logadd(double a, double b) {
  if (a == -CUDART_INF) return b;
  if (b == -CUDART_INF) return a;
  double m = fmax(a, b);
  return m + log1p(exp(-fabs(a - b)));
}

// ------------------------------------------------------------- reduction --
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ----------------------------------------------------------- cp.async --
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16_ca(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace w2l
