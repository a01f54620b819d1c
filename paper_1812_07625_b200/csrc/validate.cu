// Device-side input validation in the reference's check order, plus the
// per-utterance target preparation the fast kernels need.
//
// The reference validates before computing, so a failing utterance never
// produces partial outputs (criterion.py:23-41 _check_emissions/_check_target,
// :92-111 CTC, :174-190 ASG).  Two launches:
//   em_check  -- one thread per frame row, the whole batch in parallel:
//                non-finite values (bit 1) and, for CTC, rows whose
//                logsumexp is off by more than 1e-2 (bit 2) are OR-ed into
//                status[b] (zeroed beforehand);
//   prep      -- one block per utterance: folds those bits and the target /
//                transition checks into the FIRST failing check's code, and
//                for valid utterances builds the token CSR (chain states
//                grouped by token) used by the emissions-gradient gather.
// Compute kernels skip utterances whose status is non-zero.

#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kBitNonFinite = 1 << 8;
constexpr int kBitRowLse = 1 << 9;

// One warp per 32 consecutive frame rows of one utterance: the rows are a
// contiguous range, loaded coalesced into shared memory, then lane r checks
// row r.  The CTC row normalisation is checked in fp32 and re-checked in
// float64 (the reference's arithmetic) only near the 1e-2 threshold.
// route (nullable, zeroed beforehand): precision routing counters of the
// batch, [0] rows checked, [1] rows whose spread max - min exceeds
// route_nats, [2] rows whose spread exceeds kFlushNats (see route_to_f64).
template <class TE>
__global__ void __launch_bounds__(128)
    em_check_kernel(const TE *__restrict__ em, const int32_t *__restrict__ em_len, Dims d,
                    int check_lse, int32_t *status, int *route, float route_nats) {
  pdl_launch_dependents();   // the prep kernel may launch (it waits for this grid)
  __shared__ TE rows[4][32 * 32];
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = min(max(em_len[b], 0), d.Tmax);
  const int t0 = (blockIdx.x * 4 + warp) * 32;
  if (t0 >= T) return;
  const int nrows = min(32, T - t0), N = d.N;
  const TE *src = em + ((size_t)b * d.Tmax + t0) * N;
  TE *buf = rows[warp];
  // every load in flight before the first store (N <= 32: at most 32 each)
  TE v[32];
  const int n = nrows * N;
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = lane + 32 * k < n ? src[lane + 32 * k] : (TE)0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (lane + 32 * k < n) buf[lane + 32 * k] = v[k];
  __syncwarp();
  int bits = 0;
  float spread = 0.f;
  if (lane < nrows) {
    const TE *r = buf + lane * N;
    float m = -CUDART_INF_F, mn = CUDART_INF_F;
    for (int i = 0; i < N; ++i) {
      const double v = (double)r[i];
      if (!isfinite(v)) bits = kBitNonFinite;
      m = fmaxf(m, (float)v);
      mn = fminf(mn, (float)v);
    }
    spread = m - mn;
    if (check_lse && !bits) {
      // rows must be log-normalised: |logsumexp| <= 1e-2 (criterion.py:96-101).
      // float inputs: an fp32 pre-check, re-checked in float64 (the
      // reference's arithmetic) near the threshold; double inputs are checked
      // in double throughout (a finite double beyond FLT_MAX must not turn
      // into inf/NaN and slip through).  NaN deviations fail the check.
      if (sizeof(TE) == sizeof(double)) {
        double md = -CUDART_INF, sd = 0.0;
        for (int i = 0; i < N; ++i) md = fmax(md, (double)r[i]);
        for (int i = 0; i < N; ++i) sd += exp((double)r[i] - md);
        if (!(fabs(log(sd) + md) <= 1e-2)) bits |= kBitRowLse;
      } else {
        float sum = 0.f;
        for (int i = 0; i < N; ++i) sum += __expf((float)r[i] - m);
        const float dev = fabsf(__logf(sum) + m);
        if (!(dev <= 0.0099f)) {
          if (!(dev <= 0.0101f)) {
            bits |= kBitRowLse;
          } else {
            double md = -CUDART_INF, sd = 0.0;
            for (int i = 0; i < N; ++i) md = fmax(md, (double)r[i]);
            for (int i = 0; i < N; ++i) sd += exp((double)r[i] - md);
            if (!(fabs(log(sd) + md) <= 1e-2)) bits |= kBitRowLse;
          }
        }
      }
    }
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  if (lane == 0 && bits) atomicOr(&status[b], bits);
  if (route) {
    const unsigned wide = __ballot_sync(0xffffffffu, lane < nrows && spread > route_nats);
    const unsigned hard = __ballot_sync(0xffffffffu, lane < nrows && spread > kFlushNats);
    if (lane == 0) {
      atomicAdd(&route[0], nrows);
      if (wide) atomicAdd(&route[1], __popc(wide));
      if (hard) atomicAdd(&route[2], __popc(hard));
    }
  }
}

__device__ bool block_any(int v) { return __syncthreads_or(v); }

// grouped-by-token chain states: perm[tok_start[k] .. tok_start[k+1]) lists
// the states (ASG: l, CTC: 2l+1) whose label is k, in ascending order, from
// the targets staged in shared memory (ys, valid tokens < N).
__device__ void build_token_csr(const unsigned char *ys, int L, int N, int state_mul,
                                int state_off, int *perm, int *tok_start) {
  __shared__ int cnt[33];
  if (threadIdx.x < 33) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int l = threadIdx.x; l < L; l += blockDim.x) atomicAdd(&cnt[ys[l]], 1);
  __syncthreads();
  // exclusive prefix over the N+1 counts by warp 0 (shuffle scan)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int c = lane < N ? cnt[lane] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += v;
    }
    const int excl = x - c;
    const int total = __shfl_sync(0xffffffffu, x, 31);
    if (lane < N) tok_start[lane] = excl;
    if (lane == 0) tok_start[N] = total;
    __syncwarp();
    if (lane < N) cnt[lane] = excl;
  }
  __syncthreads();
  // warp 0 walks the targets 32 at a time: lanes holding the same token
  // find each other (match.any) and take consecutive slots in order
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      const int tk = l < L ? (int)ys[l] : 32 + lane;   // unique dummies past the end
      const unsigned same = __match_any_sync(0xffffffffu, tk);
      const int rank = __popc(same & ((1u << lane) - 1u));
      if (l < L) perm[cnt[tk] + rank] = l * state_mul + state_off;
      __syncwarp();
      if (l < L && rank == 0) cnt[tk] += __popc(same);
      __syncwarp();
    }
  }
  __syncthreads();
}

// Targets of utterance b into shared memory (one byte per label; tokens
// outside [0, N) flagged in *oor), every thread's loads issued at once.
// Inputs only: a prep kernel stages them before its PDL wait.
constexpr int kPrepThreads = 128;
template <int MAXL>
__device__ __forceinline__ void stage_targets(const int64_t *y, int L, int N,
                                              unsigned char *ys, int &oor) {
  constexpr int K = (MAXL + kPrepThreads - 1) / kPrepThreads;
  int64_t v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int l = threadIdx.x + kPrepThreads * k;
    v[k] = l < L ? y[l] : 0;
  }
  oor = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int l = threadIdx.x + kPrepThreads * k;
    if (l < L) {
      oor |= (v[k] < 0 || v[k] >= N);
      ys[l] = (unsigned char)(v[k] < 0 || v[k] >= N ? 0 : v[k]);
    }
  }
}

template <class TE>
__global__ void __launch_bounds__(kPrepThreads)
    asg_prep_kernel(const int32_t *__restrict__ em_len, const int64_t *__restrict__ tgt,
                    const int32_t *__restrict__ tgt_len, const TE *__restrict__ trans, Dims d,
                    int lpad, int *perm, int *tok_start, int32_t *status, int mode, int *prog) {
  __shared__ unsigned char ys[W2L_MAX_ASG_LABELS];
  pdl_launch_dependents();
  const int b = blockIdx.x;
  // ---- inputs first (not written by em_check: they load under its tail)
  const int T = em_len[b], L = tgt_len[b];
  const int Lc = min(max(L, 0), d.Lmax);
  constexpr int KA = (W2L_MAX_TOKENS * W2L_MAX_TOKENS) / kPrepThreads;
  TE av[KA];
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int i = threadIdx.x + kPrepThreads * k;
    av[k] = i < d.N * d.N ? trans[i] : (TE)0;
  }
  int oor;
  stage_targets<W2L_MAX_ASG_LABELS>(tgt + (size_t)b * d.Lmax, Lc, d.N, ys, oor);
  // ---- then em_check's verdict
  pdl_wait();
  if (prog && threadIdx.x < 2) prog[2 * b + threadIdx.x] = 0;   // streamed-gradient progress
  const int bits = status[b];
  int bad = 0;
  double amax = -CUDART_INF, amin = CUDART_INF;
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    if (threadIdx.x + kPrepThreads * k < d.N * d.N) {
      const double a = (double)av[k];
      bad |= !isfinite(a);
      amax = fmax(amax, a);
      amin = fmin(amin, a);
    }
  }
  // fp32 fast path: a transition weight exp(A - max A) below ~e^-80 would
  // be flushed to zero in BOTH directions (invisible to the consistency
  // guard), so such transitions send the utterance to the float64 kernel
  __shared__ double s_mx[kPrepThreads / 32], s_mn[kPrepThreads / 32];
  amax = warp_max(amax);
  amin = -warp_max(-amin);
  if ((threadIdx.x & 31) == 0) {
    s_mx[threadIdx.x >> 5] = amax;
    s_mn[threadIdx.x >> 5] = amin;
  }
  __syncthreads();   // (also: the staged targets)
  for (int q = 0; q < kPrepThreads / 32; ++q) {
    amax = fmax(amax, s_mx[q]);
    amin = fmin(amin, s_mn[q]);
  }
  int dup = 0;
  for (int l = threadIdx.x + 1; l < Lc; l += kPrepThreads) dup |= ys[l] == ys[l - 1];
  bad = block_any(bad);
  oor = block_any(oor);
  dup = block_any(dup);
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) {
    code = W2L_ERR_CONTRACT;                        // criterion.py:25-26
  } else if (bits & kBitNonFinite) {
    code = W2L_ERR_NUMERIC;                         // :27-28
  } else if (bad) {
    code = W2L_ERR_NUMERIC;                         // :179-180
  } else if (L < 0 || L > d.Lmax) {
    code = W2L_ERR_CONTRACT;
  } else {
    // 0: fp32 range; 1: fp64 range (kNeedsF64); 2: beyond it (kNeedsLog)
    const int range = mode != kPrepFast ? 0
                      : amin - amax < -(double)kFlushNats64 ? 2
                      : amin - amax < -(double)kFlushNats ? 1 : 0;
    if (oor) code = W2L_ERR_TARGET;                 // :36-40
    else if (L == 0) code = W2L_ERR_TARGET;         // :183-184
    else if (dup) code = W2L_ERR_CONTRACT;          // :185-186
    else if (T < L) code = W2L_ERR_INFEASIBLE;      // :187-190
    if (code == W2L_OK && perm)
      build_token_csr(ys, L, d.N, 1, 0, perm + (size_t)b * lpad, tok_start + b * 33);
    if (code == W2L_OK && (mode == kPrepForceExact || range == 2)) code = kNeedsLog;
    else if (code == W2L_OK && range == 1) code = kNeedsF64;
  }
  __syncthreads();
  if (threadIdx.x == 0) status[b] = code;
}

__global__ void __launch_bounds__(kPrepThreads)
    ctc_prep_kernel(const int32_t *__restrict__ em_len, const int64_t *__restrict__ tgt,
                    const int32_t *__restrict__ tgt_len, int blank, Dims d, int lpad, int *perm,
                    int *tok_start, int32_t *status, int mode, int *prog) {
  __shared__ unsigned char ys[W2L_MAX_CTC_LABELS + 1];
  __shared__ int s_reps;
  pdl_launch_dependents();
  const int b = blockIdx.x;
  // ---- inputs first (not written by em_check: they load under its tail)
  const int T = em_len[b], L = tgt_len[b];
  const int Lc = min(max(L, 0), d.Lmax);
  int oor;
  stage_targets<W2L_MAX_CTC_LABELS + 1>(tgt + (size_t)b * d.Lmax, Lc, d.N, ys, oor);
  if (threadIdx.x == 0) s_reps = 0;
  // ---- then em_check's verdict
  pdl_wait();
  if (prog && threadIdx.x < 2) prog[2 * b + threadIdx.x] = 0;   // streamed-gradient progress
  const int bits = status[b];
  __syncthreads();   // the staged targets
  int has_blank = 0, reps = 0;
  for (int l = threadIdx.x; l < Lc; l += kPrepThreads) {
    has_blank |= ys[l] == blank;
    reps += (l > 0 && ys[l] == ys[l - 1]);
  }
  oor = block_any(oor);
  has_blank = block_any(has_blank);
  atomicAdd(&s_reps, reps);
  __syncthreads();
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) {
    code = W2L_ERR_CONTRACT;
  } else if (bits & kBitNonFinite) {
    code = W2L_ERR_NUMERIC;
  } else if (blank < 0 || blank >= d.N) {
    code = W2L_ERR_CONTRACT;                        // :94-95
  } else if (bits & kBitRowLse) {
    code = W2L_ERR_CONTRACT;                        // :96-101
  } else if (L < 0 || L > d.Lmax) {
    code = W2L_ERR_CONTRACT;
  } else {
    if (oor) code = W2L_ERR_TARGET;                           // :102
    else if (has_blank) code = W2L_ERR_TARGET;                // :103-104
    else if (T < L + s_reps) code = W2L_ERR_INFEASIBLE;       // :105-111
    if (code == W2L_OK && perm)
      build_token_csr(ys, L, d.N, 2, 1, perm + (size_t)b * lpad, tok_start + b * 33);
    if (code == W2L_OK && mode == kPrepForceExact) code = kNeedsLog;
  }
  __syncthreads();
  if (threadIdx.x == 0) status[b] = code;
}

__global__ void viterbi_prep_kernel(const int32_t *__restrict__ em_len, Dims d,
                                    int32_t *status) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  const int T = em_len[b];
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) code = W2L_ERR_CONTRACT;
  else if (status[b] & kBitNonFinite) code = W2L_ERR_NUMERIC;   // _check_emissions (:265)
  status[b] = code;
}

template <class TE>
cudaError_t em_check(const TE *em, const int32_t *em_len, Dims d, int check_lse,
                     int32_t *status, cudaStream_t s, int *route = nullptr,
                     float route_nats = 0.f) {
  cudaError_t err = cudaMemsetAsync(status, 0, sizeof(int32_t) * d.B, s);
  if (err != cudaSuccess) return err;
  if (route) {
    err = cudaMemsetAsync(route, 0, sizeof(int) * kRouteWords, s);
    if (err != cudaSuccess) return err;
  }
  dim3 grid((d.Tmax + 127) / 128, d.B);
  em_check_kernel<TE><<<grid, 128, 0, s>>>(em, em_len, d, check_lse, status, route, route_nats);
  return cudaGetLastError();
}

}  // namespace

template <class TE>
cudaError_t launch_asg_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, const TE *trans, Dims d, int lpad,
                                int *perm, int *tok_start, int32_t *status, cudaStream_t s,
                                int mode, int *route, int *prog) {
  cudaError_t err = em_check<TE>(em, em_len, d, 0, status, s, route, kRouteNatsAsg);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(asg_prep_kernel<TE>, dim3(d.B), dim3(kPrepThreads), 0, s, true, em_len, tgt,
                          tgt_len, trans, d, lpad, perm, tok_start, status, mode, prog);
}
template <class TE>
cudaError_t launch_ctc_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, int blank, Dims d, int lpad, int *perm,
                                int *tok_start, int32_t *status, cudaStream_t s, int check_lse,
                                int mode, int *route, int *prog) {
  cudaError_t err = em_check<TE>(em, em_len, d, check_lse, status, s, route, kRouteNatsCtc);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(ctc_prep_kernel, dim3(d.B), dim3(kPrepThreads), 0, s, true, em_len, tgt, tgt_len,
                          blank, d, lpad, perm, tok_start, status, mode, prog);
}
template <class TE>
cudaError_t launch_viterbi_validate(const TE *em, const int32_t *em_len, Dims d,
                                    int32_t *status, cudaStream_t s) {
  cudaError_t err = em_check<TE>(em, em_len, d, 0, status, s);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(viterbi_prep_kernel, dim3((d.B + 127) / 128), dim3(128), 0, s, true,
                          em_len, d, status);
}

#define INST(TE)                                                                           \
  template cudaError_t launch_asg_validate<TE>(const TE *, const int32_t *, const int64_t *,  \
                                               const int32_t *, const TE *, Dims, int, int *, \
                                               int *, int32_t *, cudaStream_t, int, int *,    \
                                               int *);                                        \
  template cudaError_t launch_ctc_validate<TE>(const TE *, const int32_t *, const int64_t *,  \
                                               const int32_t *, int, Dims, int, int *, int *, \
                                               int32_t *, cudaStream_t, int, int, int *,      \
                                               int *);                                        \
  template cudaError_t launch_viterbi_validate<TE>(const TE *, const int32_t *, Dims,         \
                                                   int32_t *, cudaStream_t);
INST(float)
INST(double)
#undef INST

}  // namespace w2l
