// Batched Viterbi best path (replaces criterion.py:259-284).
//
// One CTA of 4 warps per utterance (see viterbi4_body).  The max-plus
// recursion runs in float64 in the reference's operation order
//     cand_j = dp[j] + A[i][j];  back = first argmax_j;  dp'[i] = e[t][i] + cand_back
// so paths and scores are bit-identical to the numpy reference (ties go to
// the lowest id, np.argmax semantics, NaN treated as the maximum).  The
// argmax is a 5-level tournament over index-ordered pairs (3 levels inside a
// lane's 8 sources, 2 across lanes by shuffles); emissions are staged in
// shared memory 32 frames at a time (cp.async, double buffered); the previous frame's dp vector is broadcast through shared
// memory (double buffered, one CTA barrier per frame); backpointers are
// uint8 in shared memory when T*N fits, else in the workspace; the traceback
// runs in chunks on all threads.

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

// ---- One CTA of 4 warps per utterance.  Warp w owns
// destinations 8w .. 8w+7; lane = 4 d + q handles destination 8w + d over the
// sources 8q .. 8q+7 (fp64 cand_j = dp[j] + A[i][j], first-max argmax in
// ascending j), then the four quarter results are combined by shuffles in
// ascending quarter order -- the same comparisons in the same order of
// precedence as the single-lane tournament, so paths and scores stay
// bit-identical.  The new dp row goes through shared memory (one CTA barrier
// per frame).  About 4x less fp64 work per warp on the serial chain.
template <bool kNanAware>
__device__ __forceinline__ void vit_merge(double &v, int &i, double ov, int oi, bool other_is_higher) {
  // (v, i) and (ov, oi) cover disjoint source ranges; the lower range wins ties
  const double lo_v = other_is_higher ? v : ov, hi_v = other_is_higher ? ov : v;
  const int lo_i = other_is_higher ? i : oi, hi_i = other_is_higher ? oi : i;
  const bool th = vit_take<kNanAware>(lo_v, hi_v);
  v = th ? hi_v : lo_v;
  i = th ? hi_i : lo_i;
}

// Emissions are staged through shared memory in chunks of kVitChunk frames,
// double buffered with cp.async (groups complete in order, so waiting for the
// older chunk never waits for the newer one).  Register prefetching stalled:
// the loads of different frames shared a scoreboard, so every step waited for
// the newest load's full latency.
constexpr int kVitChunk = 32;

template <class TE>
__device__ __forceinline__ void vit_issue_chunk(const TE *__restrict__ e, int T, int N, int c,
                                                TE *ebuf) {
  const int f0 = c * kVitChunk, f1 = min(T, f0 + kVitChunk);
  const int n = (f1 - f0) * N;
  TE *dst = ebuf + (c & 1) * kVitChunk * 32;
  const TE *src = e + (size_t)f0 * N;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + i);
    if (sizeof(TE) == 8)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + i) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src + i) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// traceback chunk length: 32 frames, longer for long utterances so that the
// chunk maps ((T / lc) * N bytes) stay within kTraceMapMax
constexpr int kTraceMapMax = 8192;
__host__ __device__ inline int vit_trace_chunk(int T) {
  return max(32, (T * 32 + kTraceMapMax - 1) / kTraceMapMax);
}

template <class TE, bool kSmemBack, bool kNanAware>
__device__ __forceinline__ void viterbi4_body(const TE *__restrict__ e, int T, int N,
                                              const double (&arow)[8], double (*dp_buf)[32],
                                              TE *ebuf, uint8_t *back, double *score_out,
                                              int64_t *path_out, uint8_t *tmap,
                                              uint8_t *tend_state) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = warp * 8 + (lane >> 2), q = lane & 3;
  const bool owner = q == 0 && d < N;   // writes dp'[d] and back[t][d]
  // shared address of back[0][d] (smem backpointers), computed once
  const unsigned back_sa = kSmemBack ? (unsigned)__cvta_generic_to_shared(back) + (unsigned)d : 0u;
  const int nch = (T + kVitChunk - 1) / kVitChunk;
  vit_issue_chunk(e, T, N, 0, ebuf);
  if (nch > 1) {
    vit_issue_chunk(e, T, N, 1, ebuf);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) dp_buf[0][threadIdx.x] = threadIdx.x < N ? (double)ebuf[threadIdx.x] : -CUDART_INF;
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    if (c >= 1) {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // chunk c landed
      __syncthreads();
      if (c + 1 < nch) vit_issue_chunk(e, T, N, c + 1, ebuf);   // into chunk c-1's buffer
    }
    const TE *eb = ebuf + (c & 1) * kVitChunk * 32 + (owner ? d : 0);
    const int tlo = max(1, c * kVitChunk), thi = min(T, (c + 1) * kVitChunk);
    for (int t = tlo; t < thi; ++t) {
      const double et = (double)eb[(t - c * kVitChunk) * N];
      const double2 *pv = reinterpret_cast<const double2 *>(dp_buf[(t - 1) & 1] + 8 * q);
      double cv[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 x = pv[k];
        cv[2 * k] = x.x + arow[2 * k];          // cand_j = dp[j] + A[i][j] (:276)
        cv[2 * k + 1] = x.y + arow[2 * k + 1];
      }
      // first-max tournament over the 8 sources of this quarter
      double c4[4];
      int i4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool tb = vit_take<kNanAware>(cv[2 * k], cv[2 * k + 1]);
        c4[k] = tb ? cv[2 * k + 1] : cv[2 * k];
        i4[k] = tb ? 2 * k + 1 : 2 * k;
      }
      const bool t0b = vit_take<kNanAware>(c4[0], c4[1]);
      const bool t1b = vit_take<kNanAware>(c4[2], c4[3]);
      const double c2a = t0b ? c4[1] : c4[0], c2b = t1b ? c4[3] : c4[2];
      const int i2a = t0b ? i4[1] : i4[0], i2b = t1b ? i4[3] : i4[2];
      const bool tf = vit_take<kNanAware>(c2a, c2b);
      double v = tf ? c2b : c2a;
      int i = 8 * q + (tf ? i2b : i2a);
      // combine quarters: (0,1) and (2,3), then (01, 23)
#pragma unroll
      for (int m = 1; m <= 2; m <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, m);
        const int oi = __shfl_xor_sync(0xffffffffu, i, m);
        vit_merge<kNanAware>(v, i, ov, oi, (q & m) == 0);
      }
      // dp'[i] = e[t][i] + cand_back; destinations >= N hold -inf (never win)
      const double nv = owner ? et + v : -CUDART_INF;
      if (q == 0) dp_buf[t & 1][d] = nv;
      if (owner) {
        if (kSmemBack)
          asm volatile("st.shared.u8 [%0], %1;\n" ::"r"(back_sa + (unsigned)(t * N)), "r"(i)
                       : "memory");
        else
          back[(size_t)t * N + d] = (uint8_t)i;
      }
      __syncthreads();
    }
  }
  // ---- traceback in chunks of lc frames (vit_trace_chunk), all threads:
  // (1) for every chunk c >= 1 and every state s at its last frame, the state
  //     one frame before the chunk (map[c][s]); 4 walks interleaved per
  //     thread, so 4 dependent backpointer loads are in flight at a time
  // (2) thread 0 picks the best final state (first maximum, NaN wins) and
  //     chains the maps from the last chunk down: the end state of each chunk
  // (3) each chunk walks back from its end state writing its path frames
  // Serially, thread 0 spent ~35 cycles per frame on the dependent loads.
  const int lc = vit_trace_chunk(T);
  const int ntc = (T + lc - 1) / lc;
  const int nw = (ntc - 1) * N;   // walks of phase 1
  auto bk = [&](int t, int st) -> int {
    return (int)back[(size_t)t * N + st];   // (written by this CTA: no read-only path)
  };
  for (int w0 = threadIdx.x * 4; w0 < nw; w0 += blockDim.x * 4) {
    int cur[4], lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int w = min(w0 + k, nw - 1);
      const int c = 1 + w / N;
      cur[k] = w % N;
      lo[k] = c * lc;
      hi[k] = min(T, (c + 1) * lc) - 1;
    }
    for (int j = 0; j < lc; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (hi[k] - j >= lo[k]) cur[k] = bk(hi[k] - j, cur[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (w0 + k < nw) tmap[w0 + k] = (uint8_t)cur[k];   // map[c][s] at (c - 1) * N + s
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double *fin = dp_buf[(T - 1) & 1];
    int best_i = 0;
    double bv = fin[0];
    for (int k = 1; k < N; ++k)
      if (vit_take<true>(bv, fin[k])) {
        bv = fin[k];
        best_i = k;
      }
    *score_out = bv;
    int cur = best_i;
    for (int c = ntc - 1; c >= 1; --c) {
      tend_state[c] = (uint8_t)cur;
      cur = tmap[(c - 1) * N + cur];
    }
    tend_state[0] = (uint8_t)cur;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ntc; c += blockDim.x) {
    const int lo = c * lc, hi = min(T, (c + 1) * lc) - 1;
    int cur = tend_state[c];
    path_out[hi] = cur;
    for (int t = hi; t > lo; --t) {
      cur = bk(t, cur);
      path_out[t - 1] = cur;
    }
  }
}

template <class TE, class TA, bool kSmemBack>
__global__ void __launch_bounds__(128) viterbi4_kernel(const TE *__restrict__ em,
                                                       const int32_t *__restrict__ em_len,
                                                       const TA *__restrict__ trans, Dims d,
                                                       int64_t *__restrict__ path,
                                                       double *__restrict__ score,
                                                       const int32_t *__restrict__ status,
                                                       uint8_t *__restrict__ back_ws) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(16) double dp_buf[2][32];
  __shared__ __align__(16) TE ebuf[2 * kVitChunk * 32];
  __shared__ uint8_t tmap[kTraceMapMax];        // traceback chunk maps (viterbi4_body)
  __shared__ uint8_t tend_state[kTraceMapMax / 32 + 1];
  pdl_wait();   // a programmatic dependent of the validation kernels
  const int b = blockIdx.x, N = d.N;
  int64_t *pb = path + (size_t)b * d.Tmax;
  if (status[b] != W2L_OK) {
    for (int t = threadIdx.x; t < d.Tmax; t += blockDim.x) pb[t] = 0;
    if (threadIdx.x == 0) score[b] = 0.0;
    return;
  }
  const int T = em_len[b];
  uint8_t *back = kSmemBack ? smem : back_ws + (size_t)b * d.Tmax * N;
  const TE *e = em + (size_t)b * d.Tmax * N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dst = warp * 8 + (lane >> 2), q = lane & 3;
  double arow[8];
  bool finite = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = 8 * q + k;
    arow[k] = (trans != nullptr && dst < N && j < N) ? (double)trans[dst * N + j] : 0.0;
    finite &= isfinite(arow[k]);
  }
  // sources j >= N: dp = -inf makes them lose; A may hold inf/NaN (not
  // validated by the reference, :270-272) -- only then the NaN-aware compare
  if (__syncthreads_and(finite))
    viterbi4_body<TE, kSmemBack, false>(e, T, N, arow, dp_buf, ebuf, back, score + b, pb, tmap,
                                        tend_state);
  else
    viterbi4_body<TE, kSmemBack, true>(e, T, N, arow, dp_buf, ebuf, back, score + b, pb, tmap,
                                       tend_state);
  for (int t = T + threadIdx.x; t < d.Tmax; t += blockDim.x) pb[t] = 0;
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
    auto k = viterbi4_kernel<TE, TA, true>;
    cudaError_t err =
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBackMax);
    if (err != cudaSuccess) return err;
    return launch_maybe_pdl(k, dim3(d.B), dim3(128), back_bytes, s, false, em, em_len, trans, d,
                            path, score, status, (uint8_t *)nullptr);
  }
  // (plain launches: launched early as programmatic dependents, the
  // latency-bound CTAs were packed two to an SM while the validation kernels
  // held the others -- 0.69 vs 0.37 ms at B=64 T=1600)
  return launch_maybe_pdl(viterbi4_kernel<TE, TA, false>, dim3(d.B), dim3(128), 0, s, false, em,
                          em_len, trans, d, path, score, status, (uint8_t *)ws);
}

template cudaError_t launch_viterbi<float, float>(const float *, const int32_t *, const float *,
                                                  Dims, int64_t *, double *, const int32_t *,
                                                  void *, cudaStream_t);
template cudaError_t launch_viterbi<double, double>(const double *, const int32_t *,
                                                    const double *, Dims, int64_t *, double *,
                                                    const int32_t *, void *, cudaStream_t);

}  // namespace w2l
