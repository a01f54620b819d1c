// The C-ABI (include/w2l_criterion.h): host-side contract checks, workspace
// carving and the launch sequence of each entry point.  No allocations, no
// global state; everything is enqueued on the caller's stream.

#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "kernels.h"

using namespace w2l;

namespace {

// float64 fallback: one CTA per flagged utterance up to this many (each slot
// holds one utterance's float64 alpha/beta rows)
constexpr int kMaxExactSlotsFallback = 64;
constexpr int kMaxExactSlotsF64 = 32;

thread_local cudaError_t g_last_cuda = cudaSuccess;  // per calling thread, like cudaGetLastError

inline int from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return W2L_OK;
  g_last_cuda = e;
  return W2L_ERR_CUDA;
}

// An NVTX range around each entry point's launch sequence (the enqueue, on
// the host timeline; ncu --nvtx-include / nsys group the kernels by it).
// Header-only NVTX3: without an attached tool a push/pop is a null check.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

bool dims_ok(int B, int Tmax, int N, int Lmax, int max_l) {
  return B >= 0 && Tmax >= 1 && N >= 1 && N <= W2L_MAX_TOKENS && Lmax >= 0 && Lmax <= max_l;
}

struct Carver {
  char *base;
  size_t off = 0;
  void *take(size_t bytes) {
    void *p = base ? base + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  }
};

// W2L_FLAG_PHASE_* -> bit 0 chain, bit 1 gradient (neither flag: both)
unsigned phase_mask(unsigned flags) {
  unsigned m = ((flags & W2L_FLAG_PHASE_CHAIN) ? 1u : 0u) | ((flags & W2L_FLAG_PHASE_GRAD) ? 2u : 0u);
  return m ? m : 3u;
}

int asg_slots(int B) { return B < kMaxExactSlotsFallback ? B : kMaxExactSlotsFallback; }
int asg_slots_f64(int B) { return B < kMaxExactSlotsF64 ? B : kMaxExactSlotsF64; }

}  // namespace

extern "C" {

const char *w2l_version(void) { return "w2l-criterion sm_100a r2 (scaled-linear fp32 + f64 exact)"; }

const char *w2l_stage_name(int kind, int i) {
  static const char *asg[] = {"validate", "chain", "grad", "final", "fallback", "reduce"};
  static const char *ctc[] = {"validate", "chain", "grad", "final", "fallback"};
  if (kind == 0 && i >= 0 && i < 6) return asg[i];
  if (kind == 1 && i >= 0 && i < 5) return ctc[i];
  return "";
}

const char *w2l_last_cuda_error(void) {
  const cudaError_t e = g_last_cuda;
  g_last_cuda = cudaSuccess;
  return cudaGetErrorString(e);
}

const char *w2l_status_string(int code) {
  switch (code) {
    case W2L_OK: return "ok";
    case W2L_ERR_CONTRACT: return "contract violation";
    case W2L_ERR_NUMERIC: return "non-finite values";
    case W2L_ERR_TARGET: return "invalid target";
    case W2L_ERR_INFEASIBLE: return "infeasible target";
    case W2L_ERR_CUDA: return "CUDA error";
    case W2L_ERR_COMM: return "communication error";
    case W2L_ERR_PRECISION: return "fp32 consistency guard failed";
    default: return "unknown";
  }
}

int w2l_status_first_error(const int32_t *status, int B, int32_t *bad_index,
                           w2l_stream_t stream) {
  if (bad_index) *bad_index = -1;
  if (B <= 0) return W2L_OK;
  if (!status) return W2L_ERR_CONTRACT;
  int32_t small[256];
  int32_t *host = B <= 256 ? small : (int32_t *)malloc(sizeof(int32_t) * B);
  if (!host) return W2L_ERR_CUDA;
  cudaError_t err = cudaMemcpyAsync(host, status, sizeof(int32_t) * B, cudaMemcpyDeviceToHost,
                                    (cudaStream_t)stream);
  if (err == cudaSuccess) err = cudaStreamSynchronize((cudaStream_t)stream);
  int code = W2L_OK;
  if (err != cudaSuccess) {
    code = from_cuda(err);
  } else {
    for (int b = 0; b < B; ++b) {
      if (host[b] != W2L_OK) {
        code = (host[b] == kNeedsF64 || host[b] == kNeedsLog) ? W2L_ERR_PRECISION : host[b];
        if (bad_index) *bad_index = b;
        break;
      }
    }
  }
  if (host != small) free(host);
  return code;
}

// ------------------------------------------------------------------ ASG --
static size_t asg_ws(int B, int Tmax, int N, int Lmax, void *base, AsgFastWs *w,
                     float **ga_utt, void **slots) {
  Dims d{B, Tmax, N, Lmax};
  Carver c{(char *)base};
  void *fast = c.take(asg_fast_ws_bytes(d));
  float *ga = (float *)c.take((size_t)B * N * N * sizeof(float));
  void *sl = c.take(asg_exact_ws_bytes_per_slot(Tmax, N, Lmax) * asg_slots(B));
  if (base) {
    asg_fast_ws_carve(d, fast, w);
    *ga_utt = ga;
    *slots = sl;
  }
  return c.off;
}

size_t w2l_asg_workspace_bytes(int B, int Tmax, int N, int Lmax) {
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_ASG_LABELS)) return 0;
  return asg_ws(B, Tmax, N, Lmax, nullptr, nullptr, nullptr, nullptr);
}

static int asg_run(const float *em, const int32_t *em_len, const int64_t *tgt,
                   const int32_t *tgt_len, const float *trans, int B, int Tmax, int N, int Lmax,
                   double *loss, float *grad_em, float *grad_trans, float *grad_trans_utt,
                   int32_t *status, void *ws, size_t ws_bytes, unsigned flags,
                   cudaStream_t s, Tracer *tr) {
  NvtxRange nv("w2l_asg_loss_grad");
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_ASG_LABELS)) return W2L_ERR_CONTRACT;
  if (B == 0) {
    // an empty shard contributes a zero transition gradient (trainer.py:433
    // skips empty shards), so a following all-reduce sums well-defined data
    if (grad_trans && !(flags & W2L_FLAG_PHASE_CHAIN))
      return from_cuda(cudaMemsetAsync(grad_trans, 0, sizeof(float) * N * N, s));
    return W2L_OK;
  }
  if (!em || !em_len || !tgt || !tgt_len || !trans || !loss || !grad_em || !grad_trans ||
      !status || !ws)
    return W2L_ERR_CONTRACT;
  if (ws_bytes < w2l_asg_workspace_bytes(B, Tmax, N, Lmax)) return W2L_ERR_CONTRACT;
  const bool fallback = !(flags & W2L_FLAG_NO_FALLBACK);
  // precision routing needs the fp64 tier behind the fp32 one
  const bool route = fallback && !(flags & W2L_FLAG_NO_ROUTE);
  const bool force = flags & W2L_FLAG_FORCE_EXACT;
  Dims d{B, Tmax, N, Lmax};
  AsgFastWs w;
  float *ga_ws;
  void *slots;
  asg_ws(B, Tmax, N, Lmax, ws, &w, &ga_ws, &slots);
  if (!route) w.route = nullptr;
  float *ga = grad_trans_utt ? grad_trans_utt : ga_ws;
  const bool loss_only = flags & W2L_FLAG_LOSS_ONLY;
  // phases: bit 0 chain, 1 gradient, 2 loss only, 3 streamed gradient
  const unsigned phases = (loss_only ? (1u | 4u) : phase_mask(flags)) |
                          ((flags & W2L_FLAG_STREAM_GRAD) ? 8u : 0u);
  trace(tr, s);
  int rc = W2L_OK;
  if (force) {
    // every valid utterance through the float64 kernel; the outputs of
    // utterances failing validation are zero
    rc = from_cuda(launch_asg_validate<float>(em, em_len, tgt, tgt_len, trans, d, w.lpad, w.perm,
                                              w.tok_start, status, s, kPrepForceExact));
    if (!rc) rc = from_cuda(cudaMemsetAsync(grad_em, 0, sizeof(float) * (size_t)B * Tmax * N, s));
    if (!rc) rc = from_cuda(cudaMemsetAsync(ga, 0, sizeof(float) * (size_t)B * N * N, s));
    if (!rc) rc = from_cuda(cudaMemsetAsync(loss, 0xff, sizeof(double) * B, s));   // NaN
    if (!rc)
      rc = from_cuda(launch_asg_exact<float>(em, em_len, tgt, tgt_len, trans, d, 1, asg_slots(B),
                                             slots, loss, grad_em, ga, status, s));
    if (!rc && !loss_only) rc = from_cuda(launch_reduce_grad_trans(ga, status, d, grad_trans, s));
    return rc;
  }
  if ((phases & 1u) && !(flags & W2L_FLAG_VALIDATED)) {
    rc = from_cuda(launch_asg_validate<float>(em, em_len, tgt, tgt_len, trans, d, w.lpad, w.perm,
                                              w.tok_start, status, s, kPrepFast,
                                              route ? w.route : nullptr, w.prog));
    if (rc) return rc;
  }
  if (flags & W2L_FLAG_PHASE_VALIDATE) return W2L_OK;
  trace(tr, s);  // validate
  rc = from_cuda(launch_asg_fast(em, em_len, tgt, tgt_len, trans, d, w, loss, grad_em, ga,
                                 status, s, tr, phases, 0));
  if (rc) return rc;
  if (!loss_only && !(phases & 2u)) return W2L_OK;
  if (fallback) {
    // the precision tiers: fp64 lanes for what the fp32 guard rejected, then
    // the float64 log-domain kernel for what the fp64 guard rejected (both
    // launches exit at once when nothing is flagged)
    rc = from_cuda(launch_asg_fast(em, em_len, tgt, tgt_len, trans, d, w, loss, grad_em, ga,
                                   status, s, nullptr, loss_only ? (1u | 4u) : 3u, 1));
    if (!rc && !(flags & W2L_FLAG_NO_LOG_FALLBACK))
      rc = from_cuda(launch_asg_exact<float>(em, em_len, tgt, tgt_len, trans, d, 1, asg_slots(B),
                                             slots, loss, grad_em, ga, status, s));
    if (rc) return rc;
  }
  if (loss_only) return W2L_OK;
  trace(tr, s);  // fallback tiers
  rc = from_cuda(launch_reduce_grad_trans(ga, status, d, grad_trans, s));
  trace(tr, s);  // reduce
  return rc;
}

int w2l_asg_loss_grad(const float *em, const int32_t *em_len, const int64_t *tgt,
                      const int32_t *tgt_len, const float *trans, int B, int Tmax, int N,
                      int Lmax, double *loss, float *grad_em, float *grad_trans,
                      float *grad_trans_utt, int32_t *status, void *ws, size_t ws_bytes,
                      unsigned flags, w2l_stream_t stream) {
  return asg_run(em, em_len, tgt, tgt_len, trans, B, Tmax, N, Lmax, loss, grad_em, grad_trans,
                 grad_trans_utt, status, ws, ws_bytes, flags, (cudaStream_t)stream, nullptr);
}

}  // extern "C"

// run a traced launch sequence and turn its events into per-stage times
template <class F>
static int traced(F run, cudaStream_t s, float *stage_ms, int *n_stages) {
  Tracer tr;
  for (int i = 0; i < Tracer::kMax; ++i) cudaEventCreate(&tr.ev[i]);
  int rc = run(&tr);
  if (rc == W2L_OK) rc = from_cuda(cudaStreamSynchronize(s));
  int n = 0;
  if (rc == W2L_OK)
    for (int i = 1; i < tr.n; ++i) cudaEventElapsedTime(&stage_ms[n++], tr.ev[i - 1], tr.ev[i]);
  if (n_stages) *n_stages = n;
  for (int i = 0; i < Tracer::kMax; ++i) cudaEventDestroy(tr.ev[i]);
  return rc;
}

extern "C" {

int w2l_asg_loss_grad_traced(const float *em, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, const float *trans, int B, int Tmax, int N,
                             int Lmax, double *loss, float *grad_em, float *grad_trans,
                             float *grad_trans_utt, int32_t *status, void *ws, size_t ws_bytes,
                             unsigned flags, w2l_stream_t stream, float *stage_ms,
                             int *n_stages) {
  cudaStream_t s = (cudaStream_t)stream;
  return traced([&](Tracer *tr) {
    return asg_run(em, em_len, tgt, tgt_len, trans, B, Tmax, N, Lmax, loss, grad_em, grad_trans,
                   grad_trans_utt, status, ws, ws_bytes, flags, s, tr);
  }, s, stage_ms, n_stages);
}

size_t w2l_asg_workspace_bytes_f64(int B, int Tmax, int N, int Lmax) {
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_ASG_LABELS)) return 0;
  Carver c{nullptr};
  c.take((size_t)B * N * N * sizeof(float));
  c.take(asg_exact_ws_bytes_per_slot(Tmax, N, Lmax) * asg_slots_f64(B));
  return c.off;
}

int w2l_asg_loss_grad_f64(const double *em, const int32_t *em_len, const int64_t *tgt,
                          const int32_t *tgt_len, const double *trans, int B, int Tmax,
                          int N, int Lmax, double *loss, float *grad_em, float *grad_trans,
                          float *grad_trans_utt, int32_t *status, void *ws, size_t ws_bytes,
                          w2l_stream_t stream) {
  NvtxRange nv("w2l_asg_loss_grad_f64");
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_ASG_LABELS)) return W2L_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0)
    return grad_trans ? from_cuda(cudaMemsetAsync(grad_trans, 0, sizeof(float) * N * N, s))
                      : W2L_OK;
  if (!em || !em_len || !tgt || !tgt_len || !trans || !loss || !grad_em || !grad_trans ||
      !status || !ws)
    return W2L_ERR_CONTRACT;
  if (ws_bytes < w2l_asg_workspace_bytes_f64(B, Tmax, N, Lmax)) return W2L_ERR_CONTRACT;
  Dims d{B, Tmax, N, Lmax};
  Carver c{(char *)ws};
  float *ga_ws = (float *)c.take((size_t)B * N * N * sizeof(float));
  void *slots = c.take(asg_exact_ws_bytes_per_slot(Tmax, N, Lmax) * asg_slots_f64(B));
  float *ga = grad_trans_utt ? grad_trans_utt : ga_ws;
  int rc = from_cuda(launch_asg_validate<double>(em, em_len, tgt, tgt_len, trans, d, 0, nullptr,
                                                 nullptr, status, s));
  if (rc) return rc;
  // zero outputs of utterances that fail validation (the exact kernel skips them)
  rc = from_cuda(cudaMemsetAsync(grad_em, 0, sizeof(float) * (size_t)B * Tmax * N, s));
  if (rc) return rc;
  rc = from_cuda(cudaMemsetAsync(ga, 0, sizeof(float) * (size_t)B * N * N, s));
  if (rc) return rc;
  rc = from_cuda(cudaMemsetAsync(loss, 0xff, sizeof(double) * B, s));   // NaN: failed utterances
  if (rc) return rc;
  rc = from_cuda(launch_asg_exact<double>(em, em_len, tgt, tgt_len, trans, d, 0,
                                          asg_slots_f64(B), slots, loss, grad_em, ga, status,
                                          s));
  if (rc) return rc;
  return from_cuda(launch_reduce_grad_trans(ga, status, d, grad_trans, s));
}

// ------------------------------------------------------------------ CTC --
static size_t ctc_ws(int B, int Tmax, int N, int Lmax, void *base, CtcFastWs *w, void **slots) {
  Dims d{B, Tmax, N, Lmax};
  Carver c{(char *)base};
  void *fast = c.take(ctc_fast_ws_bytes(d));
  void *sl = c.take(ctc_exact_ws_bytes_per_slot(Tmax, N, Lmax) * asg_slots(B));
  if (base) {
    ctc_fast_ws_carve(d, fast, w);
    *slots = sl;
  }
  return c.off;
}

size_t w2l_ctc_workspace_bytes(int B, int Tmax, int N, int Lmax) {
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_CTC_LABELS)) return 0;
  return ctc_ws(B, Tmax, N, Lmax, nullptr, nullptr, nullptr);
}

static int ctc_run(const float *logp, const int32_t *em_len, const int64_t *tgt,
                   const int32_t *tgt_len, int blank, int B, int Tmax, int N, int Lmax,
                   double *loss, float *grad_em, int32_t *status, void *ws, size_t ws_bytes,
                   unsigned flags, cudaStream_t s, Tracer *tr) {
  NvtxRange nv("w2l_ctc_loss_grad");
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_CTC_LABELS)) return W2L_ERR_CONTRACT;
  if (B == 0) return W2L_OK;
  if (!logp || !em_len || !tgt || !tgt_len || !loss || !grad_em || !status || !ws)
    return W2L_ERR_CONTRACT;
  if (ws_bytes < w2l_ctc_workspace_bytes(B, Tmax, N, Lmax)) return W2L_ERR_CONTRACT;
  Dims d{B, Tmax, N, Lmax};
  CtcFastWs w;
  void *slots;
  ctc_ws(B, Tmax, N, Lmax, ws, &w, &slots);
  const bool loss_only = flags & W2L_FLAG_LOSS_ONLY;
  const int logits = (flags & W2L_FLAG_CTC_LOGITS) ? 1 : 0;
  const bool route = !(flags & (W2L_FLAG_NO_FALLBACK | W2L_FLAG_NO_ROUTE));
  if (!route) w.route = nullptr;
  w.logits = logits;
  // phases: bit 0 chain, 1 gradient, 2 loss only, 3 streamed gradient
  const unsigned phases = (loss_only ? (1u | 4u) : phase_mask(flags)) |
                          ((flags & W2L_FLAG_STREAM_GRAD) ? 8u : 0u);
  trace(tr, s);
  int rc = W2L_OK;
  if (flags & W2L_FLAG_FORCE_EXACT) {
    rc = from_cuda(launch_ctc_validate<float>(logp, em_len, tgt, tgt_len, blank, d, w.lpad,
                                              w.perm, w.tok_start, status, s, !logits,
                                              kPrepForceExact));
    if (!rc) rc = from_cuda(cudaMemsetAsync(grad_em, 0, sizeof(float) * (size_t)B * Tmax * N, s));
    if (!rc) rc = from_cuda(cudaMemsetAsync(loss, 0xff, sizeof(double) * B, s));   // NaN
    if (!rc)
      rc = from_cuda(launch_ctc_exact<float>(logp, em_len, tgt, tgt_len, blank, d, 1,
                                             asg_slots(B), slots, loss, grad_em, status, s,
                                             logits));
    return rc;
  }
  if ((phases & 1u) && !(flags & W2L_FLAG_VALIDATED)) {
    // logits: the |row logsumexp| <= 1e-2 contract (criterion.py:96-101) does
    // not apply to unnormalised inputs
    rc = from_cuda(launch_ctc_validate<float>(logp, em_len, tgt, tgt_len, blank, d, w.lpad,
                                              w.perm, w.tok_start, status, s, !logits,
                                              kPrepFast, route ? w.route : nullptr, w.prog));
    if (rc) return rc;
  }
  if (flags & W2L_FLAG_PHASE_VALIDATE) return W2L_OK;
  trace(tr, s);  // validate
  rc = from_cuda(launch_ctc_fast(logp, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status,
                                 s, tr, phases, 0));
  if (rc) return rc;
  if (!loss_only && !(phases & 2u)) return W2L_OK;
  if (!(flags & W2L_FLAG_NO_FALLBACK)) {
    rc = from_cuda(launch_ctc_fast(logp, em_len, tgt, tgt_len, blank, d, w, loss, grad_em,
                                   status, s, nullptr, loss_only ? (1u | 4u) : 3u, 1));
    if (!rc && !(flags & W2L_FLAG_NO_LOG_FALLBACK))
      rc = from_cuda(launch_ctc_exact<float>(logp, em_len, tgt, tgt_len, blank, d, 1,
                                             asg_slots(B), slots, loss, grad_em, status, s,
                                             logits));
  }
  trace(tr, s);  // fallback tiers
  return rc;
}

int w2l_ctc_loss_grad(const float *logp, const int32_t *em_len, const int64_t *tgt,
                      const int32_t *tgt_len, int blank, int B, int Tmax, int N, int Lmax,
                      double *loss, float *grad_em, int32_t *status, void *ws,
                      size_t ws_bytes, unsigned flags, w2l_stream_t stream) {
  return ctc_run(logp, em_len, tgt, tgt_len, blank, B, Tmax, N, Lmax, loss, grad_em, status, ws,
                 ws_bytes, flags, (cudaStream_t)stream, nullptr);
}

int w2l_ctc_loss_grad_traced(const float *logp, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, int blank, int B, int Tmax, int N, int Lmax,
                             double *loss, float *grad_em, int32_t *status, void *ws,
                             size_t ws_bytes, unsigned flags, w2l_stream_t stream,
                             float *stage_ms, int *n_stages) {
  cudaStream_t s = (cudaStream_t)stream;
  return traced([&](Tracer *tr) {
    return ctc_run(logp, em_len, tgt, tgt_len, blank, B, Tmax, N, Lmax, loss, grad_em, status,
                   ws, ws_bytes, flags, s, tr);
  }, s, stage_ms, n_stages);
}

size_t w2l_ctc_workspace_bytes_f64(int B, int Tmax, int N, int Lmax) {
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_CTC_LABELS)) return 0;
  return align_up(ctc_exact_ws_bytes_per_slot(Tmax, N, Lmax) * asg_slots_f64(B), 256);
}

int w2l_ctc_loss_grad_f64(const double *logp, const int32_t *em_len, const int64_t *tgt,
                          const int32_t *tgt_len, int blank, int B, int Tmax, int N,
                          int Lmax, double *loss, float *grad_em, int32_t *status, void *ws,
                          size_t ws_bytes, w2l_stream_t stream) {
  NvtxRange nv("w2l_ctc_loss_grad_f64");
  if (!dims_ok(B, Tmax, N, Lmax, W2L_MAX_CTC_LABELS)) return W2L_ERR_CONTRACT;
  if (B == 0) return W2L_OK;
  if (!logp || !em_len || !tgt || !tgt_len || !loss || !grad_em || !status || !ws)
    return W2L_ERR_CONTRACT;
  if (ws_bytes < w2l_ctc_workspace_bytes_f64(B, Tmax, N, Lmax)) return W2L_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  Dims d{B, Tmax, N, Lmax};
  int rc =
      from_cuda(launch_ctc_validate<double>(logp, em_len, tgt, tgt_len, blank, d, 0, nullptr,
                                            nullptr, status, s));
  if (rc) return rc;
  rc = from_cuda(cudaMemsetAsync(grad_em, 0, sizeof(float) * (size_t)B * Tmax * N, s));
  if (rc) return rc;
  rc = from_cuda(cudaMemsetAsync(loss, 0xff, sizeof(double) * B, s));   // NaN: failed utterances
  if (rc) return rc;
  return from_cuda(launch_ctc_exact<double>(logp, em_len, tgt, tgt_len, blank, d, 0,
                                            asg_slots_f64(B), ws, loss, grad_em, status, s));
}

// -------------------------------------------------------------- Viterbi --
size_t w2l_viterbi_workspace_bytes(int B, int Tmax, int N) {
  if (B < 0 || Tmax < 1 || N < 1 || N > W2L_MAX_TOKENS) return 0;
  const size_t n = viterbi_ws_bytes(B, Tmax, N);
  return n ? n : 256;
}

int w2l_viterbi(const float *em, const int32_t *em_len, const float *trans, int B, int Tmax,
                int N, int64_t *path, double *score, int32_t *status, void *ws,
                size_t ws_bytes, w2l_stream_t stream) {
  NvtxRange nv("w2l_viterbi");
  if (B < 0 || Tmax < 1 || N < 1 || N > W2L_MAX_TOKENS) return W2L_ERR_CONTRACT;
  if (B == 0) return W2L_OK;
  if (!em || !em_len || !path || !score || !status) return W2L_ERR_CONTRACT;
  if (viterbi_ws_bytes(B, Tmax, N) && (!ws || ws_bytes < viterbi_ws_bytes(B, Tmax, N)))
    return W2L_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  Dims d{B, Tmax, N, 0};
  int rc = from_cuda(launch_viterbi_validate<float>(em, em_len, d, status, s));
  if (rc) return rc;
  return from_cuda(launch_viterbi<float, float>(em, em_len, trans, d, path, score, status, ws, s));
}

int w2l_viterbi_f64(const double *em, const int32_t *em_len, const double *trans, int B,
                    int Tmax, int N, int64_t *path, double *score, int32_t *status, void *ws,
                    size_t ws_bytes, w2l_stream_t stream) {
  NvtxRange nv("w2l_viterbi_f64");
  if (B < 0 || Tmax < 1 || N < 1 || N > W2L_MAX_TOKENS) return W2L_ERR_CONTRACT;
  if (B == 0) return W2L_OK;
  if (!em || !em_len || !path || !score || !status) return W2L_ERR_CONTRACT;
  if (viterbi_ws_bytes(B, Tmax, N) && (!ws || ws_bytes < viterbi_ws_bytes(B, Tmax, N)))
    return W2L_ERR_CONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  Dims d{B, Tmax, N, 0};
  int rc = from_cuda(launch_viterbi_validate<double>(em, em_len, d, status, s));
  if (rc) return rc;
  return from_cuda(
      launch_viterbi<double, double>(em, em_len, trans, d, path, score, status, ws, s));
}

int w2l_greedy_eval(const int64_t *path, const int32_t *path_len, int B, int Tmax, int kind,
                    int special, const int64_t *ref, const int32_t *ref_len, int Lmax,
                    int silence, int64_t *hyp, int32_t *hyp_len, int32_t *tok_dist,
                    int32_t *word_dist, int32_t *ref_words, int32_t *status,
                    w2l_stream_t stream) {
  NvtxRange nv("w2l_greedy_eval");
  if (B < 0 || Tmax < 1 || Lmax < 0 || (kind != 0 && kind != 1) || (kind == 1 && special < 0))
    return W2L_ERR_CONTRACT;
  if (greedy_eval_smem_bytes(Tmax, Lmax) > 227 * 1024) return W2L_ERR_CONTRACT;
  if (B == 0) return W2L_OK;
  if (!path || !path_len || !ref || !ref_len || !hyp || !hyp_len || !tok_dist || !word_dist ||
      !ref_words || !status)
    return W2L_ERR_CONTRACT;
  return from_cuda(launch_greedy_eval(path, path_len, B, Tmax, kind, special, ref, ref_len,
                                      max(Lmax, 1), silence, hyp, hyp_len, tok_dist, word_dist,
                                      ref_words, status, (cudaStream_t)stream));
}

int w2l_transitions_sgd_step(float *trans, float *velocity, const float *grad_sum, int N,
                             int batch_size, float lr, float momentum, w2l_stream_t stream) {
  NvtxRange nv("w2l_transitions_sgd_step");
  if (N < 1 || N > W2L_MAX_TOKENS || batch_size < 1 || !trans || !velocity || !grad_sum)
    return W2L_ERR_CONTRACT;
  return from_cuda(launch_transitions_sgd(trans, velocity, grad_sum, N, batch_size, lr, momentum,
                                          (cudaStream_t)stream));
}

#ifdef W2L_TIMELINE
// debug builds: CTA timeline records of the last calls (kind 0: CTC TU, 1: ASG TU)
__attribute__((visibility("default"))) int w2l_timeline_read(int kind, unsigned long long *host, int maxn) {
  return kind ? tl_read_asg(host, maxn) : tl_read_ctc(host, maxn);
}
#endif

int w2l_probe_peaks(double *mufu_ops_per_s, double *dadd_ops_per_s, double *ffma_ops_per_s) {
  return probe_peaks(mufu_ops_per_s, dadd_ops_per_s, ffma_ops_per_s);
}

}  // extern "C"
