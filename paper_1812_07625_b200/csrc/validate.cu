// Device-side input validation in the reference's check order.
//
// The reference validates before computing, so a failing utterance never
// produces partial outputs (criterion.py:23-41 _check_emissions/_check_target,
// :92-111 CTC, :174-190 ASG).  Each block validates one utterance and writes
// the FIRST failing check's code to status[b]; compute kernels skip
// utterances whose status is non-zero.

#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

template <class TE>
__device__ bool block_any_nonfinite(const TE *p, long long n) {
  int bad = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) bad |= !isfinite((double)p[i]);
  return __syncthreads_or(bad);
}

// target ids in [0, n_tok) over the first L entries (_check_target, :32-41)
__device__ bool block_target_out_of_range(const int64_t *y, int L, int n_tok) {
  int bad = 0;
  for (int i = threadIdx.x; i < L; i += blockDim.x) bad |= (y[i] < 0 || y[i] >= n_tok);
  return __syncthreads_or(bad);
}

template <class TE>
__global__ void asg_validate_kernel(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                    const int32_t *tgt_len, const TE *trans, Dims d,
                                    int32_t *status) {
  const int b = blockIdx.x;
  const int T = em_len[b], L = tgt_len[b];
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) {
    code = W2L_ERR_CONTRACT;                        // criterion.py:25-26
  } else if (block_any_nonfinite(em + (size_t)b * d.Tmax * d.N, (long long)T * d.N)) {
    code = W2L_ERR_NUMERIC;                         // :27-28
  } else if (block_any_nonfinite(trans, (long long)d.N * d.N)) {
    code = W2L_ERR_NUMERIC;                         // :179-180
  } else if (L < 0 || L > d.Lmax) {
    code = W2L_ERR_CONTRACT;
  } else {
    const int64_t *y = tgt + (size_t)b * d.Lmax;
    if (block_target_out_of_range(y, L, d.N)) {
      code = W2L_ERR_TARGET;                        // :36-40
    } else if (L == 0) {
      code = W2L_ERR_TARGET;                        // :183-184
    } else {
      int dup = 0;
      for (int i = threadIdx.x + 1; i < L; i += blockDim.x) dup |= (y[i] == y[i - 1]);
      if (__syncthreads_or(dup)) code = W2L_ERR_CONTRACT;   // :185-186
      else if (T < L) code = W2L_ERR_INFEASIBLE;            // :187-190
    }
  }
  if (threadIdx.x == 0) status[b] = code;
}

template <class TE>
__global__ void ctc_validate_kernel(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                    const int32_t *tgt_len, int blank, Dims d,
                                    int32_t *status) {
  const int b = blockIdx.x;
  const int T = em_len[b], L = tgt_len[b];
  const TE *e = em + (size_t)b * d.Tmax * d.N;
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) {
    code = W2L_ERR_CONTRACT;
  } else if (block_any_nonfinite(e, (long long)T * d.N)) {
    code = W2L_ERR_NUMERIC;
  } else if (blank < 0 || blank >= d.N) {
    code = W2L_ERR_CONTRACT;                        // :94-95
  } else {
    // rows must be log-normalised: |logsumexp| <= 1e-2 (:96-101)
    int bad = 0;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      const TE *r = e + (size_t)t * d.N;
      double m = -CUDART_INF;
      for (int i = 0; i < d.N; ++i) m = fmax(m, (double)r[i]);
      double s = 0.0;
      for (int i = 0; i < d.N; ++i) s += exp((double)r[i] - m);
      bad |= fabs(log(s) + m) > 1e-2;
    }
    if (__syncthreads_or(bad)) {
      code = W2L_ERR_CONTRACT;
    } else if (L < 0 || L > d.Lmax) {
      code = W2L_ERR_CONTRACT;
    } else {
      const int64_t *y = tgt + (size_t)b * d.Lmax;
      if (block_target_out_of_range(y, L, d.N)) {
        code = W2L_ERR_TARGET;                      // :102
      } else {
        int has_blank = 0, reps = 0;
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
          has_blank |= (y[i] == blank);
          reps += (i > 0 && y[i] == y[i - 1]);
        }
        has_blank = __syncthreads_or(has_blank);
        // block sum of repeats
        __shared__ int s_reps;
        if (threadIdx.x == 0) s_reps = 0;
        __syncthreads();
        atomicAdd(&s_reps, reps);
        __syncthreads();
        if (has_blank) code = W2L_ERR_TARGET;                   // :103-104
        else if (T < L + s_reps) code = W2L_ERR_INFEASIBLE;     // :105-111
      }
    }
  }
  if (threadIdx.x == 0) status[b] = code;
}

template <class TE>
__global__ void viterbi_validate_kernel(const TE *em, const int32_t *em_len, Dims d,
                                        int32_t *status) {
  const int b = blockIdx.x;
  const int T = em_len[b];
  int code = W2L_OK;
  if (T < 1 || T > d.Tmax) code = W2L_ERR_CONTRACT;
  else if (block_any_nonfinite(em + (size_t)b * d.Tmax * d.N, (long long)T * d.N))
    code = W2L_ERR_NUMERIC;                          // _check_emissions (:265)
  if (threadIdx.x == 0) status[b] = code;
}

}  // namespace

template <class TE>
cudaError_t launch_asg_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, const TE *trans, Dims d,
                                int32_t *status, cudaStream_t s) {
  asg_validate_kernel<TE><<<d.B, 256, 0, s>>>(em, em_len, tgt, tgt_len, trans, d, status);
  return cudaGetLastError();
}
template <class TE>
cudaError_t launch_ctc_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, int blank, Dims d, int32_t *status,
                                cudaStream_t s) {
  ctc_validate_kernel<TE><<<d.B, 256, 0, s>>>(em, em_len, tgt, tgt_len, blank, d, status);
  return cudaGetLastError();
}
template <class TE>
cudaError_t launch_viterbi_validate(const TE *em, const int32_t *em_len, Dims d,
                                    int32_t *status, cudaStream_t s) {
  viterbi_validate_kernel<TE><<<d.B, 256, 0, s>>>(em, em_len, d, status);
  return cudaGetLastError();
}

#define INST(TE)                                                                          \
  template cudaError_t launch_asg_validate<TE>(const TE *, const int32_t *, const int64_t *, \
                                               const int32_t *, const TE *, Dims, int32_t *, \
                                               cudaStream_t);                              \
  template cudaError_t launch_ctc_validate<TE>(const TE *, const int32_t *, const int64_t *, \
                                               const int32_t *, int, Dims, int32_t *,       \
                                               cudaStream_t);                              \
  template cudaError_t launch_viterbi_validate<TE>(const TE *, const int32_t *, Dims,        \
                                                   int32_t *, cudaStream_t);
INST(float)
INST(double)
#undef INST

}  // namespace w2l
