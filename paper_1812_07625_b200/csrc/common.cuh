// Shared device helpers for the sm_100a sequence-criterion kernels.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include <climits>
#include <utility>

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
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ------------------------------------------- chain -> gradient streaming --
// The gradient kernels are launched with programmatic dependent launch (PDL)
// right behind the chain kernel and run while the chains are still going:
// the frames of the middle of an utterance have both their alpha and beta
// rows once the two directions have crossed, and more frames complete with
// every step after that.  Each chain CTA publishes its progress (steps whose
// rows are complete) in a per-(utterance, direction) word with gpu-scope
// release; a gradient CTA acquires the two words of its utterance before it
// reads rows.  A chain CTA that does not run (status, routing) publishes
// kProgIdle.  Every warp of a chain CTA executes
// griddepcontrol.launch_dependents once its own progress passes the middle
// of the utterance (stream_trigger_block), so the gradient grid is only
// scheduled once every chain CTA is resident and half done: gradient CTAs
// spinning on progress can never keep a chain CTA from running, and they do
// not hold SM slots while nothing is ready (launched at chain entry, the
// streamed ASG gradient's parked CTAs delayed the other criterion's
// gradient by ~90 us: two-criteria step 0.49 -> 0.465 ms with the midpoint).
constexpr int kProgIdle = 0x7fffffff;

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// PDL: let the dependent grid launch (primary side) / no-op without PDL
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// PDL: wait until the prerequisite grid has completed and its writes are
// visible (no-op for a kernel launched without PDL).  Every kernel that may
// be launched as a programmatic dependent calls it before touching data the
// previous kernel writes; the launch sequences chain the short kernels of a
// call this way (final, fallback tiers, reduction: their launch latency
// overlaps the previous kernel), each kernel waiting for its predecessor,
// which waited for its own.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// the short kernels of a launch sequence: let the next one launch, then wait
__device__ __forceinline__ void pdl_enter() {
  pdl_launch_dependents();
  pdl_wait();
}

// Gradient-CTA side: wait until both directions of utterance b have
// published at least need_f / need_b steps.  Thread 0 polls (acquire), the
// CTA barrier then orders every thread's row loads after it.  A bound turns
// a protocol bug into a launch error instead of a hung GPU.
__device__ __forceinline__ void wait_chain_progress(const int *prog, int b, int need_f,
                                                    int need_b) {
  if (threadIdx.x == 0 && prog) {
    unsigned spins = 0;
    while (ld_acquire_gpu(prog + 2 * b) < need_f || ld_acquire_gpu(prog + 2 * b + 1) < need_b) {
      __nanosleep(256);
      if (++spins > (1u << 25)) __trap();   // ~10 s
    }
  }
  __syncthreads();
}

// Gradient CTAs are scheduled in the order their frames complete: frame
// blocks from the middle of the utterance outwards (rank 0 is the middle
// block), all utterances of one rank next to each other.
__host__ __device__ inline int block_of_rank(int r, int nblk) {
  const int c = (nblk - 1) / 2;
  const int d = (r + 1) / 2;
  return (r & 1) ? c + d : c - d;
}

// ---- optional CTA timeline (debug builds with -DW2L_TIMELINE only): each
// instrumented CTA appends {tag, t0, t1, t2} (globaltimer ns) to a per-
// translation-unit buffer read back by w2l_timeline_read (tools/timeline_pdl.py)
#ifdef W2L_TIMELINE
constexpr int kTlMax = 1 << 16;
static __device__ unsigned long long g_tl[kTlMax][4];
static __device__ unsigned g_tl_n;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned hw_warpid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tl_rec(unsigned long long tag, unsigned long long t0,
                                       unsigned long long t1, unsigned long long t2) {
  const unsigned i = atomicAdd(&g_tl_n, 1u);
  if (i < kTlMax) {
    g_tl[i][0] = tag;
    g_tl[i][1] = t0;
    g_tl[i][2] = t1;
    g_tl[i][3] = t2;
  }
}
#define W2L_TL(x) x
#else
#define W2L_TL(x)
#endif

// Streamed gradients (PDL) only with W2L_PDL=1: measured slower in the
// two-criteria step, where one criterion's gradient CTAs take the SMs the
// other criterion's chain CTAs need.
inline bool pdl_enabled() {
  static const bool on = getenv("W2L_PDL") != nullptr && getenv("W2L_PDL")[0] == '1';
  return on;
}

// Launch k, optionally as a programmatic dependent of the previous kernel
// in the stream.
template <class... KArgs, class... Args>
cudaError_t launch_maybe_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, bool pdl, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef W2L_NO_PDL_LAUNCH   // diagnostics: every launch plain
  pdl = false;
#endif
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace w2l
