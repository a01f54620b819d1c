/*
 * w2l_criterion.h -- C-ABI of the B200-native sequence-criterion library
 * (libw2l_criterion.so): batched ASG and CTC loss+gradient and ASG/CTC
 * Viterbi alignment on sm_100a.
 *
 * The reference (asrkit, /root/reference/pkg) has no FFI: its boundary for
 * this path is the Python criterion protocol in
 * pkg/src/asrkit/criterion.py.  Each entry point below names the reference
 * function it replaces; the Python host layer
 * (paper_1812_07625_b200/criterion.py) binds these symbols with ctypes and
 * re-exports the reference's names, signatures and exception types.
 *
 * Conventions (all entry points):
 *   - every array pointer is a DEVICE pointer owned by the caller; inputs are
 *     read-only, outputs are fully overwritten (zeros in padding);
 *   - layouts are row-major; emissions are [B][Tmax][N], targets are
 *     int64 [B][Lmax] padded with -1 (data.py:91-99), em_len / tgt_len are
 *     int32 [B];
 *   - transitions are A[to][from] (criterion.py:170-171);
 *   - scratch comes from a caller-provided workspace of *_workspace_bytes();
 *     there are no hidden allocations and no global mutable state, so calls
 *     on different streams are reentrant;
 *   - work is enqueued asynchronously on `stream`; the return value reports
 *     host-side contract violations and launch failures only.  Per-utterance
 *     data errors land in the device array `status[B]` (codes below); call
 *     w2l_status_first_error() to synchronise and fetch the first one.
 */
#ifndef W2L_CRITERION_H
#define W2L_CRITERION_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *w2l_stream_t; /* == cudaStream_t */

#if defined(__GNUC__)
#define W2L_API __attribute__((visibility("default")))
#else
#define W2L_API
#endif

/* Status codes; they map 1:1 onto the reference exception classes
 * (pkg/src/asrkit/errors.py:12-54). */
enum {
  W2L_OK = 0,
  W2L_ERR_CONTRACT = 1,   /* ContractError         */
  W2L_ERR_NUMERIC = 2,    /* NumericError          */
  W2L_ERR_TARGET = 3,     /* TargetError           */
  W2L_ERR_INFEASIBLE = 4, /* InfeasibleTargetError */
  W2L_ERR_CUDA = 5,       /* launch / runtime failure */
  W2L_ERR_COMM = 6,       /* collective failure (multi-GPU layer) */
  W2L_ERR_PRECISION = 7   /* fp32 guard failed and W2L_FLAG_NO_FALLBACK was set */
};

/* flags for the fp32 batched entry points */
#define W2L_FLAG_NO_FALLBACK 1u  /* report fp32 guard failures instead of recomputing them */
/* Split-phase calls (both bits clear = the whole call).  PHASE_CHAIN runs the
 * validation and the forward/backward recursions, leaving their rows in the
 * workspace; PHASE_GRAD then runs the posterior/gradient kernels, the loss,
 * the float64 fallback and the batch reduction from that workspace (same
 * inputs, same stream order).  Lets a caller schedule the latency-bound
 * recursions of several criteria together, ahead of their throughput-bound
 * gradient phases. */
#define W2L_FLAG_PHASE_CHAIN 2u
#define W2L_FLAG_PHASE_GRAD 4u
/* Loss only (evaluation): the forward recursion and the loss; no
 * posterior/gradient kernels and no transition gradient (grad_em is written
 * only for utterances recomputed by the float64 fallback). */
#define W2L_FLAG_LOSS_ONLY 8u
/* CTC on unnormalised logits with log-softmax fused in: the loss
 * is that of log_softmax(x) (autodiff.py:394-411) and grad_em is the gradient
 * with respect to x; the |row logsumexp| <= 1e-2 contract does not apply. */
#define W2L_FLAG_CTC_LOGITS 16u
/* Skip the fp32 fast path: every valid utterance is computed by the float64
 * log-domain kernel (the guard's fallback path, forced; tests and
 * diagnostics). */
#define W2L_FLAG_FORCE_EXACT 32u
/* Precision tiers of the fp32 batched entry points: an utterance whose fp32
 * guard fails is recomputed with fp64 lanes (same kernels, range 2^+-1022);
 * one that fails that guard too by the float64 log-domain kernel.  This flag
 * stops after the fp64 tier (diagnostics: which tier resolved an input). */
#define W2L_FLAG_NO_LOG_FALLBACK 64u
/* Precision routing (on by default with the fallback tiers): when the
 * emissions are so peaky that the fp32 tier would fail its guard (any frame
 * row spread max - min beyond the fp32 flush limit, or more than a quarter
 * of the rows wider than a criterion-specific spread: 16 nats ASG, 32 CTC),
 * the whole batch goes straight to the fp64 tier, skipping an fp32 pass whose
 * results would be discarded (the chains are latency-bound: two passes cost
 * two passes, whatever the number of failures).  Results are the same either
 * way; this flag disables the routing (diagnostics, A/B timing). */
#define W2L_FLAG_NO_ROUTE 128u
/* Validation as its own phase.  PHASE_VALIDATE runs only the input checks
 * (status, token CSR, routing counters) into status and the workspace;
 * VALIDATED then runs the compute phases (chain and gradient, or those named
 * by PHASE_CHAIN / PHASE_GRAD) without repeating them.  Lets a caller stagger
 * two criteria on two streams: the second starts its validation when the
 * first's has finished, so its recursions start that much later -- measured
 * on the two-criteria step, the chains then share the SMs without the
 * simultaneous-start slow mode. */
#define W2L_FLAG_PHASE_VALIDATE 256u
#define W2L_FLAG_VALIDATED 512u
/* Streamed gradient: the gradient kernels are launched as programmatic
 * dependents of the chains and start on the middle frames of an utterance
 * once its two directions have crossed, gated by per-utterance progress
 * words.  Correct in every setting (the gradient grid only launches once
 * every chain CTA is resident); faster when no other criterion's chains still
 * need SMs, e.g. the later of two staggered criteria. */
#define W2L_FLAG_STREAM_GRAD 1024u

/* Library limits of the sm_100a kernels. */
#define W2L_MAX_TOKENS 32        /* N: one lane per token in the N x N graph   */
#define W2L_MAX_ASG_LABELS 1024  /* Lmax for ASG (32 lanes x 32 states)        */
#define W2L_MAX_CTC_LABELS 511   /* Lmax for CTC (2L+1 <= 1024 lattice states) */

/* ------------------------------------------------------------------ ASG --
 * Replaces asg_loss_grad (criterion.py:167-247), batched.
 *   loss[B]            f64  per-utterance loss  (fcc score - fac score); NaN for an
 *                           utterance whose status is an error
 *   grad_em[B,Tmax,N]  f32  d loss_b / d emissions_b
 *   grad_trans[N,N]    f32  sum over utterances of d loss_b / d A
 *                           (trainer.py:417-418; the /B stays with the caller)
 *   grad_trans_utt     f32  [B,N,N] per-utterance d loss_b / d A, or NULL
 * fp32 arithmetic (scaled linear domain, exact power-of-two rescaling) with a
 * per-utterance self-consistency guard; utterances that fail the guard are
 * recomputed by the float64 log-domain kernel inside the same call. */
W2L_API size_t w2l_asg_workspace_bytes(int B, int Tmax, int N, int Lmax);
W2L_API int w2l_asg_loss_grad(const float *em, const int32_t *em_len, const int64_t *tgt,
                      const int32_t *tgt_len, const float *trans, int B, int Tmax, int N,
                      int Lmax, double *loss, float *grad_em, float *grad_trans,
                      float *grad_trans_utt, int32_t *status, void *ws, size_t ws_bytes,
                      unsigned flags, w2l_stream_t stream);
/* float64-input variant computed entirely by the float64 log-domain kernel:
 * the reference's own numerics ("float64 internals", criterion.py:1-7). */
W2L_API size_t w2l_asg_workspace_bytes_f64(int B, int Tmax, int N, int Lmax);
W2L_API int w2l_asg_loss_grad_f64(const double *em, const int32_t *em_len, const int64_t *tgt,
                          const int32_t *tgt_len, const double *trans, int B, int Tmax,
                          int N, int Lmax, double *loss, float *grad_em, float *grad_trans,
                          float *grad_trans_utt, int32_t *status, void *ws, size_t ws_bytes,
                          w2l_stream_t stream);

/* ------------------------------------------------------------------ CTC --
 * Replaces ctc_loss_grad (criterion.py:84-162), batched.  Emissions are
 * log-probabilities; rows must satisfy |logsumexp| <= 1e-2. */
W2L_API size_t w2l_ctc_workspace_bytes(int B, int Tmax, int N, int Lmax);
W2L_API int w2l_ctc_loss_grad(const float *logp, const int32_t *em_len, const int64_t *tgt,
                      const int32_t *tgt_len, int blank, int B, int Tmax, int N, int Lmax,
                      double *loss, float *grad_em, int32_t *status, void *ws,
                      size_t ws_bytes, unsigned flags, w2l_stream_t stream);
W2L_API size_t w2l_ctc_workspace_bytes_f64(int B, int Tmax, int N, int Lmax);
W2L_API int w2l_ctc_loss_grad_f64(const double *logp, const int32_t *em_len, const int64_t *tgt,
                          const int32_t *tgt_len, int blank, int B, int Tmax, int N,
                          int Lmax, double *loss, float *grad_em, int32_t *status, void *ws,
                          size_t ws_bytes, w2l_stream_t stream);

/* -------------------------------------------------------------- Viterbi --
 * Replaces viterbi (criterion.py:259-284), batched.  float64 max-plus in the
 * reference's operation order (bit-exact paths and scores); ties go to the
 * lowest id.  trans may be NULL (zeros, the CTC viterbi_path at :334-336).
 *   path[B,Tmax] int64 (zero padded), score[B] f64. */
W2L_API size_t w2l_viterbi_workspace_bytes(int B, int Tmax, int N);
W2L_API int w2l_viterbi(const float *em, const int32_t *em_len, const float *trans, int B, int Tmax,
                int N, int64_t *path, double *score, int32_t *status, void *ws,
                size_t ws_bytes, w2l_stream_t stream);
W2L_API int w2l_viterbi_f64(const double *em, const int32_t *em_len, const double *trans, int B,
                    int Tmax, int N, int64_t *path, double *score, int32_t *status, void *ws,
                    size_t ws_bytes, w2l_stream_t stream);

/* ---------------------------------------------- greedy evaluation --
 * the reference's evaluate loop per utterance (trainer.py:465-514)
 * on the device, for a batch of Viterbi paths (w2l_viterbi):
 *   collapse the path (criterion.py:287-310): kind 0 = ASG (drop repeats,
 *     the repetition token `special` -- or -1 -- becomes its predecessor),
 *     kind 1 = CTC (drop repeats, then the blank `special`);
 *   tok_dist[b]  Levenshtein distance of the collapsed path to ref[b];
 *   word_dist[b] the same over silence-delimited token groups
 *     (lexicon.py:182-195; silence < 0: the whole sequence is one group);
 *   ref_words[b] the reference's group count;
 *   hyp[B,Tmax]  the collapsed tokens (-1 padded), hyp_len[b] their count.
 * status[b]: 0, or W2L_ERR_CONTRACT for a length out of range or an ASG path
 * starting with the repetition token.  Tmax <= ~11000 (shared memory). */
W2L_API int w2l_greedy_eval(const int64_t *path, const int32_t *path_len, int B, int Tmax,
                    int kind, int special, const int64_t *ref, const int32_t *ref_len,
                    int Lmax, int silence, int64_t *hyp, int32_t *hyp_len, int32_t *tok_dist,
                    int32_t *word_dist, int32_t *ref_words, int32_t *status,
                    w2l_stream_t stream);

/* ------------------------------------------------- transition update --
 * the step after the transition-gradient all-reduce
 * (trainer.py:442-449, autodiff.py:429-433) in one N x N kernel:
 *   g = float32(grad_sum / batch_size); v = v * momentum + g; A = A - lr * v
 * with the reference's float32 rounding (no fused multiply-add).
 * trans, velocity: f32[N][N] device, updated in place; grad_sum: f32[N][N]
 * (the batch sum, e.g. after the NCCL all-reduce). */
W2L_API int w2l_transitions_sgd_step(float *trans, float *velocity, const float *grad_sum, int N,
                                     int batch_size, float lr, float momentum,
                                     w2l_stream_t stream);

/* ------------------------------------------------------- multi-GPU --
 * The data-parallel exchange (trainer.py:433-447): each rank runs
 * the batched criterion on its contiguous shard, then ONE sum all-reduce of
 * the N x N transition gradient over NCCL (NVLink/NVSwitch), enqueued on the
 * same stream right after w2l_asg_loss_grad.  The /B stays with the caller.
 * NCCL is loaded at run time (libnccl.so.2); w2l_comm_available() reports
 * whether it could be.  Communicators: rank 0 creates a 128-byte unique id,
 * the host side distributes it (any channel), every rank calls
 * w2l_comm_init with its CUDA device current.  Failures: W2L_ERR_COMM. */
W2L_API int w2l_comm_available(void);
W2L_API int w2l_comm_unique_id(void *id_out /* 128 bytes */);
W2L_API int w2l_comm_init(const void *id, int world, int rank, void **comm);
W2L_API int w2l_comm_destroy(void *comm);
W2L_API int w2l_allreduce_grad_A(float *grad_A, int N, void *comm, w2l_stream_t stream);

/* ------------------------------------------------------------- tracing --
 * Same computation as w2l_asg_loss_grad / w2l_ctc_loss_grad, with a CUDA
 * event after every stage; synchronises `stream` and writes the per-stage
 * device times (ms) to stage_ms[*n_stages] (names: w2l_stage_name; kind 0 =
 * ASG: validate, chain, grad, final, exact_fallback, reduce; kind 1 = CTC:
 * validate, chain, grad, final, exact_fallback).  stage_ms needs 16 slots. */
W2L_API int w2l_asg_loss_grad_traced(const float *em, const int32_t *em_len, const int64_t *tgt,
                                     const int32_t *tgt_len, const float *trans, int B, int Tmax,
                                     int N, int Lmax, double *loss, float *grad_em,
                                     float *grad_trans, float *grad_trans_utt, int32_t *status,
                                     void *ws, size_t ws_bytes, unsigned flags,
                                     w2l_stream_t stream, float *stage_ms, int *n_stages);
W2L_API int w2l_ctc_loss_grad_traced(const float *logp, const int32_t *em_len, const int64_t *tgt,
                                     const int32_t *tgt_len, int blank, int B, int Tmax, int N,
                                     int Lmax, double *loss, float *grad_em, int32_t *status,
                                     void *ws, size_t ws_bytes, unsigned flags,
                                     w2l_stream_t stream, float *stage_ms, int *n_stages);
W2L_API const char *w2l_stage_name(int kind, int i);

/* ------------------------------------------------------------ utilities -- */
/* Synchronises `stream`, copies status[B] to the host and returns the first
 * non-zero code (W2L_OK if none); *bad_index receives its utterance or -1. */
W2L_API int w2l_status_first_error(const int32_t *status, int B, int32_t *bad_index,
                           w2l_stream_t stream);
W2L_API const char *w2l_status_string(int code);
/* Text of the last CUDA error seen by this thread's calls (then cleared). */
W2L_API const char *w2l_last_cuda_error(void);
/* Library build identifier (kernel generation), for provenance in benches. */
W2L_API const char *w2l_version(void);
/* Microbenchmarks used for the roofline denominators (MUFU ex2 ops/s and
 * FP64 add ops/s), measured on the current device. */
W2L_API int w2l_probe_peaks(double *mufu_ops_per_s, double *dadd_ops_per_s, double *ffma_ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* W2L_CRITERION_H */
