// Host-side launchers for the sm_100a kernels (one translation unit each).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace w2l {

struct Dims {
  int B, Tmax, N, Lmax;
};

// Optional per-stage event trace (profiling entry points only): mark()
// records an event on the stream after each stage of a launch sequence.
struct Tracer {
  static constexpr int kMax = 16;
  cudaEvent_t ev[kMax];
  int n = 0;
  void mark(cudaStream_t s) {
    if (n < kMax) cudaEventRecord(ev[n++], s);
  }
};
inline void trace(Tracer *t, cudaStream_t s) {
  if (t) t->mark(s);
}

// ---- validation (reference check order; criterion.py:23-41,92-111,174-190)
// perm/tok_start (nullable): token CSR of valid utterances for the fast path.
// mode: kPrepExact (float64 API: valid utterances stay W2L_OK), kPrepFast
// (fp32 path: inputs outside its range are marked kNeedsExact), or
// kPrepForceExact (W2L_FLAG_FORCE_EXACT: every valid utterance kNeedsExact).
enum { kPrepExact = 0, kPrepFast = 1, kPrepForceExact = 2 };
template <class TE>
cudaError_t launch_asg_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, const TE *trans, Dims d, int lpad,
                                int *perm, int *tok_start, int32_t *status, cudaStream_t s,
                                int mode = kPrepExact, int *route = nullptr,
                                int *prog = nullptr);
template <class TE>
cudaError_t launch_ctc_validate(const TE *em, const int32_t *em_len, const int64_t *tgt,
                                const int32_t *tgt_len, int blank, Dims d, int lpad, int *perm,
                                int *tok_start, int32_t *status, cudaStream_t s,
                                int check_lse = 1, int mode = kPrepExact, int *route = nullptr,
                                int *prog = nullptr);
template <class TE>
cudaError_t launch_viterbi_validate(const TE *em, const int32_t *em_len, Dims d,
                                    int32_t *status, cudaStream_t s);

// ---- float64 log-domain kernels (exact path + fallback for the fp32 guard)
size_t asg_exact_ws_bytes_per_slot(int Tmax, int N, int Lmax);
size_t ctc_exact_ws_bytes_per_slot(int Tmax, int N, int Lmax);
// only_flagged: process utterances whose status is kNeedsExact (fallback);
// otherwise every utterance with status OK.
template <class TE>
cudaError_t launch_asg_exact(const TE *em, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, const TE *trans, Dims d, int only_flagged,
                             int nslots, void *slot_ws, double *loss, float *grad_em,
                             float *ga_utt, int32_t *status, cudaStream_t s);
template <class TE>
cudaError_t launch_ctc_exact(const TE *em, const int32_t *em_len, const int64_t *tgt,
                             const int32_t *tgt_len, int blank, Dims d, int only_flagged,
                             int nslots, void *slot_ws, double *loss, float *grad_em,
                             int32_t *status, cudaStream_t s, int logits = 0);

// ---- scaled-linear fast path (tier 0: fp32 lanes; tier 1: fp64 lanes for
// the utterances whose fp32 guard failed).  Rows are sized for fp64.
struct AsgFastWs {
  void *fcc_a, *fcc_b;       // V [B][Tmax][32]
  int *fcc_ka, *fcc_kb;      // [B][tpad] cumulative exponents (kb stored at t+1)
  void *fac_a, *fac_b;       // V [B][W][Tmax][128] warp-major lattice rows
  int *fac_ea, *fac_eb;      // [B][W][Tmax][32] per-lane exponents
  double *scal;              // [B][4]: lnZ fcc fwd, fcc bwd, fac fwd, fac bwd
  float *part_fullA;         // [B][nblk][32][32]
  float *part_edge;          // [B][nblk][Lpad]
  double *part_guard;        // [B][nblk][4] min / max frame log2-normalisers (fcc, fac)
  int *prog;                 // [B][2] chain progress (streamed gradient; common.cuh)
  int *route;                // [kRouteWords] precision routing counters (em_check)
  int *perm;                 // [B][Lpad] states sorted by token
  int *tok_start;            // [B][33]
  int spl, W, lpad, nblk, tpad;  // W lattice warps; tpad = round_up(Tmax + 1, 8)
};
int asg_fast_spl(int Lmax);  // 0 if unsupported
size_t asg_fast_ws_bytes(Dims d);
void asg_fast_ws_carve(Dims d, void *ws, AsgFastWs *w);
// tier 0 processes status W2L_OK and marks failures kNeedsF64; tier 1
// processes kNeedsF64 and marks failures kNeedsLog (exact.cu takes those)
cudaError_t launch_asg_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, const float *trans, Dims d,
                            const AsgFastWs &w, double *loss, float *grad_em, float *ga_utt,
                            int32_t *status, cudaStream_t s, Tracer *tr = nullptr,
                            unsigned phases = 3u, int tier = 0);  // phases bit 0: chain, 1: gradient, 2: loss only

struct CtcFastWs {
  void *a, *b;               // V [B][W][Tmax][128] warp-major lattice rows
  int *ea, *eb;              // [B][W][Tmax][32]
  double *scal;              // [B][4]: lnZ fwd, lnZ bwd, sum of frame shifts, spare
  double *part_guard;        // [B][nblk][2] min / max frame log2-normaliser
  int *prog;                 // [B][2] chain progress (streamed gradient; common.cuh)
  int *route;                // [kRouteWords] precision routing counters (em_check)
  int *perm;                 // [B][Lpad] label positions sorted by token
  int *tok_start;            // [B][33]
  int spl, W, lpad, nblk;
  int logits;                // W2L_FLAG_CTC_LOGITS: log-softmax fused in
};
int ctc_fast_spl(int Lmax);
size_t ctc_fast_ws_bytes(Dims d);
void ctc_fast_ws_carve(Dims d, void *ws, CtcFastWs *w);
cudaError_t launch_ctc_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                            double *loss, float *grad_em, int32_t *status, cudaStream_t s,
                            Tracer *tr = nullptr, unsigned phases = 3u, int tier = 0);

// ---- reductions
cudaError_t launch_reduce_grad_trans(const float *ga_utt, const int32_t *status, Dims d,
                                     float *grad_trans, cudaStream_t s);

cudaError_t launch_transitions_sgd(float *w, float *v, const float *gsum, int N, int batch,
                                   float lr, float momentum, cudaStream_t s);

// ---- Viterbi (float64 max-plus, bit-exact)
size_t viterbi_ws_bytes(int B, int Tmax, int N);
template <class TE, class TA>
cudaError_t launch_viterbi(const TE *em, const int32_t *em_len, const TA *trans, Dims d,
                           int64_t *path, double *score, const int32_t *status, void *ws,
                           cudaStream_t s);

#ifdef W2L_TIMELINE
int tl_read_ctc(unsigned long long *host, int maxn);
int tl_read_asg(unsigned long long *host, int maxn);
#endif

// ---- greedy evaluation (evaluate.cu)
size_t greedy_eval_smem_bytes(int Tmax, int Lmax);
cudaError_t launch_greedy_eval(const int64_t *path, const int32_t *path_len, int B, int Tmax,
                               int kind, int special, const int64_t *ref, const int32_t *ref_len,
                               int Lmax, int silence, int64_t *hyp, int32_t *hyp_len,
                               int32_t *tok_dist, int32_t *word_dist, int32_t *ref_words,
                               int32_t *status, cudaStream_t s);

// ---- microbenchmarks
int probe_peaks(double *mufu, double *dadd, double *ffma);

}  // namespace w2l
