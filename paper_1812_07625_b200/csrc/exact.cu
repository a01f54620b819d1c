// Float64 log-domain ASG and CTC kernels: the reference's own numerics on
// the GPU.
//
// These kernels restate criterion.py's dynamic programs (ASG :193-247, CTC
// :113-162) in float64 log space, one CTA per utterance:
//   phase 1 -- each warp runs one recursion concurrently (ASG: fcc alpha,
//              fcc beta, fac alpha, fac beta; CTC: alpha, beta), state rows
//              double-buffered in shared memory and streamed to a per-slot
//              workspace;
//   phase 2 -- all threads form posteriors and gradients in parallel over
//              frames / transition pairs / states.
// They serve (a) the reference-compatible float64 entry points
// (w2l_*_loss_grad_f64), and (b) the last-resort fallback for utterances
// that failed the guards of both scaled-linear tiers (only_flagged:
// status kNeedsLog).  A fixed number of workspace slots
// bounds memory: CTA k handles utterances k, k+nslots, ...

#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kExactThreads = 128;

__device__ __forceinline__ bool wants(int st, int only_flagged) {
  return only_flagged ? (st == kNeedsLog) : (st == W2L_OK);
}

// log-sum-exp with the reference's non-finite-max rule (criterion.py:250-254)
template <int kCount>
__device__ __forceinline__ double lse_row(const double *x, int n) {
  double m = -CUDART_INF;
  for (int j = 0; j < n; ++j) m = fmax(m, x[j]);
  if (!isfinite(m)) m = 0.0;
  double s = 0.0;
  for (int j = 0; j < n; ++j) s += exp(x[j] - m);
  return log(s) + m;
}

// --------------------------------------------------------------- ASG -----
struct AsgSlot {
  double *ga, *gb;  // [Tmax][N]
  double *fa, *fb;  // [Tmax][Lmax]
};

__host__ __device__ inline size_t asg_slot_bytes(int Tmax, int N, int Lmax) {
  return align_up((size_t)Tmax * (2 * N + 2 * Lmax) * sizeof(double), 256);
}

template <class TE>
__global__ void __launch_bounds__(kExactThreads)
    asg_exact_kernel(const TE *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     const TE *__restrict__ trans, Dims d, int only_flagged, int nslots,
                     uint8_t *slot_ws, double *loss, float *grad_em, float *ga_utt,
                     int32_t *status) {
  pdl_enter();
  extern __shared__ __align__(16) double sm[];
  const int N = d.N, Lmax = d.Lmax;
  double *A = sm;                       // [N][N]
  double *rows = A + N * N;             // 4 chains x 2 buffers x max(Lmax, 32)
  const int RW = max(Lmax, 32);
  double *fullA = rows + 8 * RW;        // [N][N]
  double *edge = fullA + N * N;         // [2][Lmax]  stay / step sums
  int *y = (int *)(edge + 2 * Lmax);    // [Lmax]
  __shared__ double s_fal, s_fcc;

  // nothing to do for this slot (the common fallback case): leave after one
  // parallel look at the statuses instead of walking them serially
  {
    int any = 0;
    for (int b = blockIdx.x + nslots * (int)threadIdx.x; b < d.B; b += nslots * (int)blockDim.x)
      any |= wants(status[b], only_flagged);
    if (!__syncthreads_or(any)) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) A[i] = (double)trans[i];

  AsgSlot ws;
  {
    double *base = (double *)(slot_ws + asg_slot_bytes(d.Tmax, N, Lmax) * blockIdx.x);
    ws.ga = base;
    ws.gb = ws.ga + (size_t)d.Tmax * N;
    ws.fa = ws.gb + (size_t)d.Tmax * N;
    ws.fb = ws.fa + (size_t)d.Tmax * Lmax;
  }

  for (int b = blockIdx.x; b < d.B; b += nslots) {
    __syncthreads();
    if (!wants(status[b], only_flagged)) continue;
    const int T = em_len[b], L = tgt_len[b];
    const TE *e = em + (size_t)b * d.Tmax * N;
    for (int l = threadIdx.x; l < L; l += blockDim.x) y[l] = (int)tgt[(size_t)b * Lmax + l];
    __syncthreads();
    auto E = [&](int t, int i) { return (double)e[(size_t)t * N + i]; };

    // ---------------- phase 1: four concurrent recursions, one per warp
    if (warp == 0) {
      // fcc alpha: ga[t][i] = e[t][i] + lse_j(ga[t-1][j] + A[i][j])   (:227-231)
      double *buf = rows;
      if (lane < N) {
        buf[lane] = E(0, lane);
        ws.ga[lane] = buf[lane];
      }
      for (int t = 1; t < T; ++t) {
        __syncwarp();
        const double *p = buf + ((t - 1) & 1) * RW;
        double *q = buf + (t & 1) * RW;
        if (lane < N) {
          double m = -CUDART_INF;
          for (int j = 0; j < N; ++j) m = fmax(m, p[j] + A[lane * N + j]);
          if (!isfinite(m)) m = 0.0;
          double s = 0.0;
          for (int j = 0; j < N; ++j) s += exp(p[j] + A[lane * N + j] - m);
          const double v = E(t, lane) + (log(s) + m);
          q[lane] = v;
          ws.ga[(size_t)t * N + lane] = v;
        }
      }
      __syncwarp();
      if (lane == 0) s_fal = lse_row<0>(buf + ((T - 1) & 1) * RW, N);   // :231
    } else if (warp == 1) {
      // fcc beta: gb[t][j] = e[t][j] + lse_i(gb[t+1][i] + A[i][j])    (:233-236)
      double *buf = rows + 2 * RW;
      if (lane < N) {
        buf[((T - 1) & 1) * RW + lane] = E(T - 1, lane);
        ws.gb[(size_t)(T - 1) * N + lane] = E(T - 1, lane);
      }
      for (int t = T - 2; t >= 0; --t) {
        __syncwarp();
        const double *p = buf + ((t + 1) & 1) * RW;
        double *q = buf + (t & 1) * RW;
        if (lane < N) {
          double m = -CUDART_INF;
          for (int i = 0; i < N; ++i) m = fmax(m, p[i] + A[i * N + lane]);
          if (!isfinite(m)) m = 0.0;
          double s = 0.0;
          for (int i = 0; i < N; ++i) s += exp(p[i] + A[i * N + lane] - m);
          const double v = E(t, lane) + (log(s) + m);
          q[lane] = v;
          ws.gb[(size_t)t * N + lane] = v;
        }
      }
    } else if (warp == 2) {
      // fac alpha over the target-constrained chain (:193-203)
      double *buf = rows + 4 * RW;
      for (int l = lane; l < L; l += 32) {
        const double v = (l == 0) ? E(0, y[0]) : -CUDART_INF;
        buf[l] = v;
        ws.fa[l] = v;
      }
      for (int t = 1; t < T; ++t) {
        __syncwarp();
        const double *p = buf + ((t - 1) & 1) * RW;
        double *q = buf + (t & 1) * RW;
        for (int l = lane; l < L; l += 32) {
          double acc = p[l] + A[y[l] * N + y[l]];
          if (l > 0) acc = logadd(acc, p[l - 1] + A[y[l] * N + y[l - 1]]);
          const double v = E(t, y[l]) + acc;
          q[l] = v;
          ws.fa[(size_t)t * Lmax + l] = v;
        }
      }
      __syncwarp();
      if (lane == 0) s_fcc = buf[((T - 1) & 1) * RW + L - 1];          // :203
    } else if (warp == 3) {
      // fac beta (:205-212)
      double *buf = rows + 6 * RW;
      for (int l = lane; l < L; l += 32) {
        const double v = (l == L - 1) ? E(T - 1, y[L - 1]) : -CUDART_INF;
        buf[((T - 1) & 1) * RW + l] = v;
        ws.fb[(size_t)(T - 1) * Lmax + l] = v;
      }
      for (int t = T - 2; t >= 0; --t) {
        __syncwarp();
        const double *p = buf + ((t + 1) & 1) * RW;
        double *q = buf + (t & 1) * RW;
        for (int l = lane; l < L; l += 32) {
          double acc = p[l] + A[y[l] * N + y[l]];
          if (l + 1 < L) acc = logadd(acc, p[l + 1] + A[y[l + 1] * N + y[l]]);
          const double v = E(t, y[l]) + acc;
          q[l] = v;
          ws.fb[(size_t)t * Lmax + l] = v;
        }
      }
    }
    __syncthreads();   // also orders the workspace writes for phase 2
    const double fal = s_fal, fcc = s_fcc;

    // ---------------- phase 2a: emissions gradient, one thread per frame
    float *ge = grad_em + (size_t)b * d.Tmax * N;
    for (int t = threadIdx.x; t < d.Tmax; t += blockDim.x) {
      if (t >= T) {
        for (int i = 0; i < N; ++i) ge[(size_t)t * N + i] = 0.f;
        continue;
      }
      double con[32];
      for (int i = 0; i < N; ++i) con[i] = 0.0;
      for (int l = 0; l < L; ++l) {                                      // :214-217
        const double v = ws.fa[(size_t)t * Lmax + l] + ws.fb[(size_t)t * Lmax + l];
        con[y[l]] += exp(v - E(t, y[l]) - fcc);
      }
      for (int i = 0; i < N; ++i) {                                      // :238, :245
        const double full = exp(ws.ga[(size_t)t * N + i] + ws.gb[(size_t)t * N + i] -
                                E(t, i) - fal);
        ge[(size_t)t * N + i] = (float)(full - con[i]);
      }
    }
    // ---------------- phase 2b: full-graph transition posteriors (:239-241)
    for (int p = threadIdx.x; p < N * N; p += blockDim.x) {
      const int i = p / N, j = p % N;
      double s = 0.0;
      for (int t = 1; t < T; ++t)
        s += exp(ws.ga[(size_t)(t - 1) * N + j] + A[p] + ws.gb[(size_t)t * N + i] - fal);
      fullA[p] = s;
    }
    // ---------------- phase 2c: constrained edge posteriors per state (:218-224)
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
      const double stay = A[y[l] * N + y[l]];
      const double step = l > 0 ? A[y[l] * N + y[l - 1]] : 0.0;
      double ss = 0.0, sp = 0.0;
      for (int t = 1; t < T; ++t) {
        const double fbt = ws.fb[(size_t)t * Lmax + l];
        ss += exp(ws.fa[(size_t)(t - 1) * Lmax + l] + stay + fbt - fcc);
        if (l > 0) sp += exp(ws.fa[(size_t)(t - 1) * Lmax + l - 1] + step + fbt - fcc);
      }
      edge[l] = ss;
      edge[Lmax + l] = sp;
    }
    __syncthreads();
    // deterministic scatter of the per-state sums into the N x N bins
    for (int p = threadIdx.x; p < N * N; p += blockDim.x) {
      const int i = p / N, j = p % N;
      double con = 0.0;
      int prev = -1;   // y[l-1], carried (a paired y[l-1], y[l] load ran past y's end)
      for (int l = 0; l < L; ++l) {
        const int yl = y[l];
        if (yl == i && yl == j) con += edge[l];
        if (l > 0 && yl == i && prev == j) con += edge[Lmax + l];
        prev = yl;
      }
      ga_utt[(size_t)b * N * N + p] = (float)(fullA[p] - con);          // :246
    }
    if (threadIdx.x == 0) {
      loss[b] = fal - fcc;                                               // :244
      status[b] = W2L_OK;
    }
  }
}

// --------------------------------------------------------------- CTC -----
__host__ __device__ inline size_t ctc_slot_bytes(int Tmax, int Lmax) {
  const int S = 2 * Lmax + 1;
  // alpha, beta [T][S] and the per-frame log-softmax normaliser (logits mode)
  return align_up((size_t)Tmax * S * 2 * sizeof(double) + (size_t)Tmax * sizeof(double), 256);
}

template <class TE>
__global__ void __launch_bounds__(kExactThreads)
    ctc_exact_kernel(const TE *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, int only_flagged, int nslots, uint8_t *slot_ws,
                     double *loss, float *grad_em, int32_t *status, int logits) {
  pdl_enter();
  extern __shared__ __align__(16) double sm[];
  const int N = d.N, Smax = 2 * d.Lmax + 1;
  double *rows = sm;                         // 2 chains x 2 buffers x Smax
  int *lab = (int *)(rows + 4 * Smax);       // [Smax]
  int *skip = lab + Smax;                    // [Smax]
  __shared__ double s_logz;
  // nothing to do for this slot (the common fallback case): leave after one
  // parallel look at the statuses instead of walking them serially
  {
    int any = 0;
    for (int b = blockIdx.x + nslots * (int)threadIdx.x; b < d.B; b += nslots * (int)blockDim.x)
      any |= wants(status[b], only_flagged);
    if (!__syncthreads_or(any)) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *alpha = (double *)(slot_ws + ctc_slot_bytes(d.Tmax, d.Lmax) * blockIdx.x);
  double *beta = alpha + (size_t)d.Tmax * Smax;
  double *lse = beta + (size_t)d.Tmax * Smax;   // [Tmax] logits mode

  for (int b = blockIdx.x; b < d.B; b += nslots) {
    __syncthreads();
    if (!wants(status[b], only_flagged)) continue;
    const int T = em_len[b], L = tgt_len[b], S = 2 * L + 1;
    const TE *e = em + (size_t)b * d.Tmax * N;
    // logits: log_softmax rows in float64 (autodiff.py:400-403): x - lse(x)
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      double m = -CUDART_INF, acc = 0.0;
      if (logits) {
        for (int i = 0; i < N; ++i) m = fmax(m, (double)e[(size_t)t * N + i]);
        for (int i = 0; i < N; ++i) acc += exp((double)e[(size_t)t * N + i] - m);
        lse[t] = m + log(acc);
      } else {
        lse[t] = 0.0;
      }
    }
    const int64_t *yb = tgt + (size_t)b * d.Lmax;
    // lattice (criterion.py:113-120)
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
      lab[s] = (s & 1) ? (int)yb[s >> 1] : blank;
      skip[s] = (s & 1) && s >= 3 && yb[s >> 1] != yb[(s >> 1) - 1];
    }
    __syncthreads();
    auto EL = [&](int t, int s) { return (double)e[(size_t)t * N + lab[s]] - lse[t]; };

    if (warp == 0) {                                                  // alpha (:122-141)
      double *buf = rows;
      for (int s = lane; s < S; s += 32) {
        const double v = s == 0 ? EL(0, 0) : (s == 1 ? EL(0, 1) : -CUDART_INF);
        buf[s] = v;
        alpha[s] = v;
      }
      for (int t = 1; t < T; ++t) {
        __syncwarp();
        const double *p = buf + ((t - 1) & 1) * Smax;
        double *q = buf + (t & 1) * Smax;
        for (int s = lane; s < S; s += 32) {
          double acc = p[s];
          if (s >= 1) acc = logadd(acc, p[s - 1]);
          if (s >= 2 && skip[s]) acc = logadd(acc, p[s - 2]);
          const double v = EL(t, s) + acc;
          q[s] = v;
          alpha[(size_t)t * Smax + s] = v;
        }
      }
      __syncwarp();
      if (lane == 0) {
        const double *f = buf + ((T - 1) & 1) * Smax;
        s_logz = S > 1 ? logadd(f[S - 1], f[S - 2]) : f[S - 1];
      }
    } else if (warp == 1) {                                           // beta (:143-155)
      double *buf = rows + 2 * Smax;
      for (int s = lane; s < S; s += 32) {
        const double v = (s == S - 1 || s == S - 2) ? EL(T - 1, s) : -CUDART_INF;
        buf[((T - 1) & 1) * Smax + s] = v;
        beta[(size_t)(T - 1) * Smax + s] = v;
      }
      for (int t = T - 2; t >= 0; --t) {
        __syncwarp();
        const double *p = buf + ((t + 1) & 1) * Smax;
        double *q = buf + (t & 1) * Smax;
        for (int s = lane; s < S; s += 32) {
          double acc = p[s];
          if (s + 1 < S) acc = logadd(acc, p[s + 1]);
          if (s + 2 < S && skip[s + 2]) acc = logadd(acc, p[s + 2]);
          const double v = EL(t, s) + acc;
          q[s] = v;
          beta[(size_t)t * Smax + s] = v;
        }
      }
    }
    __syncthreads();
    const double logz = s_logz;
    float *ge = grad_em + (size_t)b * d.Tmax * N;
    if (!isfinite(logz)) {                                            // :140-141
      for (int i = threadIdx.x; i < d.Tmax * N; i += blockDim.x) ge[i] = 0.f;
      if (threadIdx.x == 0) {
        status[b] = W2L_ERR_INFEASIBLE;
        loss[b] = CUDART_INF;
      }
      continue;
    }
    for (int t = threadIdx.x; t < d.Tmax; t += blockDim.x) {          // :157-161
      if (t >= T) {
        for (int i = 0; i < N; ++i) ge[(size_t)t * N + i] = 0.f;
        continue;
      }
      double g[32];
      for (int i = 0; i < N; ++i) g[i] = 0.0;
      for (int s = 0; s < S; ++s) {
        const double post = exp(alpha[(size_t)t * Smax + s] + beta[(size_t)t * Smax + s] -
                                EL(t, s) - logz);
        g[lab[s]] -= post;
      }
      if (logits)   // d/dx of log_softmax: g - softmax * sum(g), sum(g) = -1
        for (int i = 0; i < N; ++i) g[i] += exp((double)e[(size_t)t * N + i] - lse[t]);
      for (int i = 0; i < N; ++i) ge[(size_t)t * N + i] = (float)g[i];
    }
    if (threadIdx.x == 0) {
      loss[b] = -logz;                                                // :162
      status[b] = W2L_OK;
    }
  }
}

}  // namespace

size_t asg_exact_ws_bytes_per_slot(int Tmax, int N, int Lmax) {
  return asg_slot_bytes(Tmax, N, Lmax);
}
size_t ctc_exact_ws_bytes_per_slot(int Tmax, int N, int Lmax) {
  (void)N;
  return ctc_slot_bytes(Tmax, Lmax);
}

template <class TE>
cudaError_t launch_asg_exact(const TE *em, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, const TE *trans, Dims d, int only_flagged,
                             int nslots, void *slot_ws, double *loss, float *grad_em,
                             float *ga_utt, int32_t *status, cudaStream_t s) {
  const int RW = d.Lmax > 32 ? d.Lmax : 32;
  const size_t smem = sizeof(double) * (2 * d.N * d.N + 8 * RW + 2 * d.Lmax) +
                      sizeof(int) * d.Lmax;
  auto k = asg_exact_kernel<TE>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(k, dim3(nslots), dim3(kExactThreads), smem, s, true, em, em_len, tgt,
                          tgt_len, trans, d, only_flagged, nslots, (uint8_t *)slot_ws, loss,
                          grad_em, ga_utt, status);
}

template <class TE>
cudaError_t launch_ctc_exact(const TE *em, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, int blank, Dims d, int only_flagged,
                             int nslots, void *slot_ws, double *loss, float *grad_em,
                             int32_t *status, cudaStream_t s, int logits) {
  const int Smax = 2 * d.Lmax + 1;
  const size_t smem = sizeof(double) * 4 * Smax + sizeof(int) * 2 * Smax;
  auto k = ctc_exact_kernel<TE>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(k, dim3(nslots), dim3(kExactThreads), smem, s, true, em, em_len, tgt,
                          tgt_len, blank, d, only_flagged, nslots, (uint8_t *)slot_ws, loss,
                          grad_em, status, logits);
}

#define INST(TE)                                                                           \
  template cudaError_t launch_asg_exact<TE>(const TE *, const int32_t *, const int64_t *,   \
                                            const int32_t *, const TE *, Dims, int, int,    \
                                            void *, double *, float *, float *, int32_t *,  \
                                            cudaStream_t);                                  \
  template cudaError_t launch_ctc_exact<TE>(const TE *, const int32_t *, const int64_t *,   \
                                            const int32_t *, int, Dims, int, int, void *,   \
                                            double *, float *, int32_t *, cudaStream_t, int);
INST(float)
INST(double)
#undef INST

}  // namespace w2l
