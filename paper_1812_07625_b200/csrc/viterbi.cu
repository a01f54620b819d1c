// Batched Viterbi best path (replaces criterion.py:259-284).
//
// One warp per utterance, lane i owns destination token i and keeps row i of
// the transition matrix in registers (A[to][from], criterion.py:276).  The
// max-plus recursion runs in float64 in the reference's operation order
//     cand_j = dp[j] + A[i][j];  back = first argmax_j;  dp'[i] = e[t][i] + cand_back
// so paths and scores are bit-identical to the numpy reference (ties go to
// the lowest id, np.argmax semantics, NaN treated as the maximum).  The
// argmax is a 5-level tournament over index-ordered pairs (depth 5 instead of
// a 30-long compare chain); emissions are prefetched 8 frames ahead; the
// previous frame's dp vector is broadcast through shared memory (double
// buffered, one __syncwarp per frame); backpointers are uint8 in shared
// memory when T*N fits, else in the workspace; lane 0 traces back.

#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kSmemBackMax = 160 * 1024;

template <bool kNanAware>
__device__ __forceinline__ bool vit_take(double a, double b) {
  // does candidate b (higher index) replace a?  np.argmax: first maximum wins,
  // a NaN is the maximum and the first NaN wins
  if (kNanAware) return !isnan(a) && (b > a || isnan(b));
  return b > a;
}

// one frame of the max-plus recursion for destination token `lane`;
// returns the new dp value and writes the backpointer.  Sources j >= N hold
// dp = -inf (and A = 0), so they never win and need no bounds test.
template <bool kNanAware>
__device__ __forceinline__ double vit_step(const double *prev, const double (&arow)[32],
                                           double et, int &arg_out) {
  double c16[16];
  int i16[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {   // level 1 of the tournament fused with cand_j = dp[j] + A[i][j]
    const double a = prev[2 * j] + arow[2 * j];
    const double b = prev[2 * j + 1] + arow[2 * j + 1];
    const bool tb = vit_take<kNanAware>(a, b);
    c16[j] = tb ? b : a;
    i16[j] = tb ? 2 * j + 1 : 2 * j;
  }
  double c8[8];
  int i8[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool tb = vit_take<kNanAware>(c16[2 * j], c16[2 * j + 1]);
    c8[j] = tb ? c16[2 * j + 1] : c16[2 * j];
    i8[j] = tb ? i16[2 * j + 1] : i16[2 * j];
  }
  double c4[4];
  int i4[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool tb = vit_take<kNanAware>(c8[2 * j], c8[2 * j + 1]);
    c4[j] = tb ? c8[2 * j + 1] : c8[2 * j];
    i4[j] = tb ? i8[2 * j + 1] : i8[2 * j];
  }
  const bool t0 = vit_take<kNanAware>(c4[0], c4[1]);
  const bool t1 = vit_take<kNanAware>(c4[2], c4[3]);
  const double c2a = t0 ? c4[1] : c4[0], c2b = t1 ? c4[3] : c4[2];
  const int i2a = t0 ? i4[1] : i4[0], i2b = t1 ? i4[3] : i4[2];
  const bool tf = vit_take<kNanAware>(c2a, c2b);
  arg_out = tf ? i2b : i2a;
  return et + (tf ? c2b : c2a);                       // dp'[i] = e[t][i] + cand_back
}

template <class TE, class TA, bool kSmemBack, bool kNanAware>
__device__ __forceinline__ void viterbi_body(const TE *__restrict__ e, int T, int N, int lane,
                                             const double (&arow)[32], double (*dp_buf)[32],
                                             uint8_t *back, double *score_out,
                                             int64_t *path_out) {
  constexpr int kPre = 8;   // emission prefetch distance (frames)
  TE pre[kPre];   // raw emissions, converted at use so the load latency stays hidden
#pragma unroll
  for (int q = 0; q < kPre; ++q)
    pre[q] = (lane < N && 1 + q < T) ? e[(size_t)(1 + q) * N + lane] : TE(0);
  double dp = lane < N ? (double)e[lane] : -CUDART_INF;
  dp_buf[0][lane] = dp;
  for (int t0 = 1; t0 < T; t0 += kPre) {
#pragma unroll
    for (int q = 0; q < kPre; ++q) {
      const int t = t0 + q;
      if (t < T) {
        const double et = (double)pre[q];
        const int tn = t + kPre;
        pre[q] = (lane < N && tn < T) ? e[(size_t)tn * N + lane] : TE(0);
        __syncwarp();
        int arg;
        dp = vit_step<kNanAware>(dp_buf[(t - 1) & 1], arow, et, arg);
        if (lane < N) back[(size_t)t * N + lane] = (uint8_t)arg;
        dp_buf[t & 1][lane] = lane < N ? dp : -CUDART_INF;
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    const double *fin = dp_buf[(T - 1) & 1];
    int best_i = 0;
    double bv = fin[0];
    for (int i = 1; i < N; ++i)
      if (vit_take<true>(bv, fin[i])) {
        bv = fin[i];
        best_i = i;
      }
    *score_out = bv;
    int cur = best_i;
    path_out[T - 1] = cur;
    for (int t = T - 1; t > 0; --t) {
      cur = back[(size_t)t * N + cur];
      path_out[t - 1] = cur;
    }
  }
}

template <class TE, class TA, bool kSmemBack>
__global__ void __launch_bounds__(32) viterbi_kernel(const TE *__restrict__ em,
                                                     const int32_t *__restrict__ em_len,
                                                     const TA *__restrict__ trans, Dims d,
                                                     int64_t *__restrict__ path,
                                                     double *__restrict__ score,
                                                     const int32_t *__restrict__ status,
                                                     uint8_t *__restrict__ back_ws) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(16) double dp_buf[2][32];
  const int b = blockIdx.x, lane = threadIdx.x, N = d.N;
  int64_t *pb = path + (size_t)b * d.Tmax;
  if (status[b] != W2L_OK) {
    for (int t = lane; t < d.Tmax; t += 32) pb[t] = 0;
    if (lane == 0) score[b] = 0.0;
    return;
  }
  const int T = em_len[b];
  uint8_t *back = kSmemBack ? smem : back_ws + (size_t)b * d.Tmax * N;
  const TE *e = em + (size_t)b * d.Tmax * N;
  double arow[32];
  bool finite = true;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    arow[j] = (trans != nullptr && lane < N && j < N) ? (double)trans[lane * N + j] : 0.0;
    finite &= isfinite(arow[j]);
  }
  // A may hold inf/NaN (the reference does not validate it, :270-272): only
  // then is the NaN-aware comparison needed
  if (__all_sync(0xffffffffu, finite))
    viterbi_body<TE, TA, kSmemBack, false>(e, T, N, lane, arow, dp_buf, back, score + b, pb);
  else
    viterbi_body<TE, TA, kSmemBack, true>(e, T, N, lane, arow, dp_buf, back, score + b, pb);
  for (int t = T + lane; t < d.Tmax; t += 32) pb[t] = 0;
}

}  // namespace

size_t viterbi_ws_bytes(int B, int Tmax, int N) {
  if ((size_t)Tmax * N <= (size_t)kSmemBackMax) return 0;
  return align_up((size_t)B * Tmax * N, 256);
}

template <class TE, class TA>
cudaError_t launch_viterbi(const TE *em, const int32_t *em_len, const TA *trans, Dims d,
                           int64_t *path, double *score, const int32_t *status, void *ws,
                           cudaStream_t s) {
  const size_t back_bytes = (size_t)d.Tmax * d.N;
  if (back_bytes <= (size_t)kSmemBackMax) {
    auto k = viterbi_kernel<TE, TA, true>;
    cudaError_t err =
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBackMax);
    if (err != cudaSuccess) return err;
    k<<<d.B, 32, back_bytes, s>>>(em, em_len, trans, d, path, score, status, nullptr);
  } else {
    viterbi_kernel<TE, TA, false><<<d.B, 32, 0, s>>>(em, em_len, trans, d, path, score, status,
                                                     (uint8_t *)ws);
  }
  return cudaGetLastError();
}

template cudaError_t launch_viterbi<float, float>(const float *, const int32_t *, const float *,
                                                  Dims, int64_t *, double *, const int32_t *,
                                                  void *, cudaStream_t);
template cudaError_t launch_viterbi<double, double>(const double *, const int32_t *,
                                                    const double *, Dims, int64_t *, double *,
                                                    const int32_t *, void *, cudaStream_t);

}  // namespace w2l
