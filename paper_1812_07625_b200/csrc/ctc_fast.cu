// Batched CTC loss + gradient (replaces criterion.py:84-162 for the batched
// hot path), in two precision tiers of one algorithm.
//
// The 2L+1-state blank-augmented lattice (criterion.py:113-120) runs in the
// scaled linear domain on the multi-warp wavefront lattice of lattice.cuh
// (4 states per lane, type V with a per-lane power-of-two exponent):
//   alpha_t[s] = Et[lab_s] (alpha[s] + alpha[s-1] + skip_s alpha[s-2])
//   beta'_t[s] = w[s] + w[s+1] + skip_{s+2} w[s+2],  w = Et+1[lab] beta'_{t+1}
// with Et = exp(logp - max_i logp) and the per-frame shifts summed in f64 for
// the loss.  Kernels (one stream):
//   ctc_chain     grid (B, 2): the forward and backward recursions, every
//                 row (lane values + exponents) to the workspace;
//   ctc_grad      grid (T / 128, B): per-frame posteriors with their own
//                 normaliser Z_t, gather by token (blank = even states,
//                 labels through a token CSR), gradient rows, per-frame guard;
//   ctc_final     loss and guard verdict.
// V = float is the fast tier; utterances that fail its guard are recomputed
// with V = double (range 2^+-1022), and those that fail again by the float64
// log-domain kernel (exact.cu).

#include "band.cuh"
#include "laneblock.cuh"
#include "lattice.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

template <bool FWD, class V, bool STREAM>
__device__ __forceinline__ void ctc_chain_body(ChainSm<V> &sm, const float *em, int T, int L,
                                               const int64_t *y, int blank, Dims d,
                                               const CtcFastWs &w, int b, unsigned tokmask,
                                               int32_t *status, int fail) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = 2 * L + 1;
  const int weff = lat_warps(S);
  if (warp == 0) {
    ProdCtx pc{em + (size_t)b * d.Tmax * d.N, d.N, T, FWD, weff, w.logits, tokmask};
    pc.gprog = w.prog ? w.prog + 2 * b + (FWD ? 0 : 1) : nullptr;
    pc.trig = stream_trigger_step<kCtc>(T);
    producer_run<V>(sm, pc, lane, FWD ? w.scal + b * 4 + 2 : nullptr);
  } else if (warp - 1 < weff) {
    LatCtx c;
    c.w = warp - 1;
    c.W = weff;
    c.lane = lane;
    c.T = T;
    c.N = d.N;
    c.nstates = S;
    c.cons_idx = 0;
    c.Tmax = d.Tmax;
    const size_t ub = (size_t)b * w.W * d.Tmax;
    c.rows = reinterpret_cast<V *>(FWD ? w.a : w.b) + ub * kLatStates;
    c.exps = (FWD ? w.ea : w.eb) + ub * 32;
    LatState<V> f;
    lat_init_weights<kCtc, FWD, V>(f, c.w, lane, d.N, S, y, L, nullptr, 0.f, blank);
    lattice_run<kCtc, FWD, V, STREAM>(sm, c, f);
  } else if (STREAM) {   // a warp without a role: its share of the trigger, at
    wait_ge(&sm.cons[0], stream_trigger_step<kCtc>(T));   // lattice warp 0's midpoint
    pdl_launch_dependents();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    w.scal[b * 4 + (FWD ? 0 : 1)] = lattice_total(sm, weff);
    if (sm.flush) status[b] = fail;
    if (w.prog) st_release_gpu(w.prog + 2 * b + (FWD ? 0 : 1), T);   // last write of the CTA
  }
}

// grid (B, 2): blockIdx.y 0 = forward (alpha), 1 = backward (beta);
// STREAM: publish progress and trigger the streamed gradient (w.prog set)
template <class V, bool STREAM>
__global__ void __launch_bounds__(32 * (1 + kMaxLatWarps))
    ctc_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, CtcFastWs w, int32_t *__restrict__ status, int want,
                     int fail) {
  extern __shared__ __align__(128) unsigned char dsm[];
  ChainSm<V> &sm = *reinterpret_cast<ChainSm<V> *>(dsm);
  pdl_wait();   // launched as a programmatic dependent of the prep / previous tier
  W2L_TL(const unsigned long long tl0 = gtimer());
  const int b = blockIdx.x;
  int *gprog = w.prog ? w.prog + 2 * b + blockIdx.y : nullptr;
  if (status[b] != want) {
    if (gprog && threadIdx.x == 0) st_release_gpu(gprog, kProgIdle);
    return;
  }
  if (want == W2L_OK && route_to_f64(w.route)) {   // the batch goes to the fp64 tier
    if (threadIdx.x == 0) {
      if (blockIdx.y == 0) status[b] = kNeedsF64;
      if (gprog) st_release_gpu(gprog, kProgIdle);
    }
    return;
  }
  // streamed gradient: every warp triggers the dependent launch once its own
  // progress passes the middle of the utterance (lattice_run, producer_run),
  // so the gradient CTAs take SMs only when their first frames are ready;
  // otherwise a CTA with work triggers nothing before it completes
  const int T = em_len[b], L = tgt_len[b];
  const int weff = lat_warps(2 * L + 1);
  __shared__ unsigned s_mask;
  if (threadIdx.x == 0) sm.prod = 0, sm.flush = 0, s_mask = 1u << blank;
  if (threadIdx.x < kCounters) sm.cons[threadIdx.x] = threadIdx.x < weff ? 0 : kDone;
  __syncthreads();
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  // tokens on the lattice: the blank and the target's labels
  for (int l = threadIdx.x; l < L; l += blockDim.x) atomicOr(&s_mask, 1u << (int)y[l]);
  __syncthreads();
  if (blockIdx.y == 0)
    ctc_chain_body<true, V, STREAM>(sm, em, T, L, y, blank, d, w, b, s_mask, status, fail);
  else
    ctc_chain_body<false, V, STREAM>(sm, em, T, L, y, blank, d, w, b, s_mask, status, fail);
  W2L_TL(if (threadIdx.x == 0) tl_rec(1000000ull + b * 10 + blockIdx.y, tl0, gtimer(), smid() | (hw_warpid() << 16)));
}

#ifndef W2L_CTC_GRAD_FRAMES
#define W2L_CTC_GRAD_FRAMES 128
#endif
constexpr int kGradFramesPerBlock = W2L_CTC_GRAD_FRAMES;   // frames per gradient CTA
constexpr int kGradWarps = 8;

// One warp per frame at a time; lane i owns states 128 sw + 4 i + k of every
// lattice warp sw and token i of the gradient row.  Posteriors are scaled
// into range by the lane exponents against the frame's largest exponent sum
// and normalised by their own per-frame sum z_t; log2 z_t plus that
// reference is the frame's log-normaliser, which the guard compares with the
// totals.  Rows of lanes past the lattice's last state were never stored
// and are read as zero.  Grid (B, nblk): y is the block's completion rank
// (block_of_rank), so with PDL the CTAs run in the order the two chains
// complete their frames; prog (null: the chains have finished) gates them.
// fp32 gradient CTAs per SM the registers must allow; shared memory (~52 KB
// per CTA) caps residency at 4 anyway (5: 48 registers, step 0.431 vs 0.424 ms)
#ifndef W2L_CTC_GRAD_MINB
#define W2L_CTC_GRAD_MINB 4
#endif
template <int W, class V>
__global__ void __launch_bounds__(kGradWarps * 32, sizeof(V) == 4 ? W2L_CTC_GRAD_MINB : 1)
    ctc_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    int blank, Dims d, CtcFastWs w, float *__restrict__ grad_em,
                    const int32_t *__restrict__ status, int want, const int *prog) {
  constexpr int LP = W * kLatStates;
  static_assert(W <= kGradWarps, "cta_first_band: one lane block per thread");
  __shared__ __align__(16) float prow[kGradWarps][LP];   // wide-window posteriors
  __shared__ unsigned stok[LP / 4];                        // label tokens per lane block (band.cuh)
  __shared__ unsigned bins[kGradWarps][32];               // per-warp token sums (fixed point)
  __shared__ double gw[kGradWarps][2];
  extern __shared__ __align__(16) unsigned char gsm[];   // [kGradWarps] prefetch rings
  pdl_launch_dependents();
  if (!prog) pdl_wait();   // not streamed: the chain grid must have completed
  const int b = blockIdx.x, blk = block_of_rank(blockIdx.y, w.nblk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N, T = em_len[b];
  const int t0 = blk * kGradFramesPerBlock;
  float *ge = grad_em + (size_t)b * d.Tmax * N;
  const int fpw = kGradFramesPerBlock / kGradWarps;
  const int ta = t0 + warp * fpw, tb = min(ta + fpw, d.Tmax);
  if (t0 >= T) {   // padding frames only: the first tier owns their zeros
    if (want == W2L_OK)
      for (int t = ta; t < tb; ++t)
        if (lane < N) ge[(size_t)t * N + lane] = 0.f;
    return;
  }
  W2L_TL(const unsigned long long tl0 = gtimer());
  wait_chain_progress(prog, b, min(t0 + kGradFramesPerBlock, T), T - t0);
  W2L_TL(const unsigned long long tl1 = gtimer());
  const int st = *(volatile const int32_t *)(status + b);
  if (want == W2L_OK) {
    // the first tier owns the zeros: padding frames and utterances it does
    // not compute (a later tier rewrites the rows of the ones it takes)
    for (int t = st == W2L_OK ? max(ta, T) : ta; t < tb; ++t)
      if (lane < N) ge[(size_t)t * N + lane] = 0.f;
  }
  if (st != want) return;
  const int L = tgt_len[b], S = 2 * L + 1;
  // tokens of each lane block's label states (odd states 2l+1 carry y_l;
  // blanks are summed apart)
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  for (int m = threadIdx.x; m < (S + 3) / 4; m += blockDim.x) {
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int st4 = m * 4 + k;
      const unsigned tk = ((st4 & 1) && st4 < S) ? (unsigned)y[st4 >> 1] : 0xffu;
      v |= tk << (8 * k);
    }
    stok[m] = v;
  }
  bins[warp][lane] = 0u;
  __syncthreads();
  const size_t seg0 = (size_t)b * w.W * d.Tmax;
  float *myp = prow[warp];
  const int tend = min(tb, T);
  // band-limited walk over the warp's frames (band.cuh); CTC posterior mass
  // moves by up to 2 states per frame
  BandRows<V> br;
  br.A = reinterpret_cast<const V *>(w.a) + seg0 * kLatStates;
  br.B = reinterpret_cast<const V *>(w.b) + seg0 * kLatStates;
  br.EA = w.ea + seg0 * 32;
  br.EB = w.eb + seg0 * 32;
  br.segv = (uint32_t)d.Tmax * kLatStates;
  br.sege = (uint32_t)d.Tmax * 32;
  br.S = S;
  br.nblk = (S + kSpl - 1) / kSpl;
  unsigned *mybins = bins[warp];
  // the CTA's reference exponent and the band of its first frame t0
  __shared__ int sband[kGradWarps + 2];
  int ref, blo, bhi;
  br.cta_first_band(t0, kGradWarps, sband, ref, blo, bhi);
  float l2min = CUDART_INF_F, l2max = -CUDART_INF_F;   // log2 z_t (the guard adds ref)
  // the two-frame prefetch ring (band.cuh): this warp's first two frames from
  // the CTA's band, widened by the frames in between (CTC mass moves by up
  // to 2 states per frame)
  BandPf<V> pf;
  pf.init(gsm + warp * band_pf_bytes<V>());
  int clo, chi, nlo, nhi;   // lane-block windows of frames t and t + 1
  br.window(blo, bhi, 2 * (ta - t0), clo, chi);
  br.window(blo, bhi, 2 * (ta + 1 - t0), nlo, nhi);
  if (ta < tend) pf.issue(br, br.frame(ta), clo + lane, clo + lane <= chi, 0, lane);
  cp_async_commit();
  if (ta + 1 < tend) pf.issue(br, br.frame(ta + 1), nlo + lane, nlo + lane <= nhi, 1, lane);
  cp_async_commit();
  int slot = 0;   // ring slot of frame t
  for (int t = ta; t < tend; ++t) {
    float zl = 0.f, zb = 0.f;
    int lo = INT_MAX, hi = -1;
    float q0[kSpl];
    auto take = [&](const V (&va)[kSpl], const V (&vb)[kSpl], int e, int m, float (&q)[kSpl],
                    bool keep) {
#pragma unroll
      for (int k = 0; k < kSpl; ++k) q[k] = 0.f;
      if (e == INT_MIN) return;
      band_block<V>(va, vb, e, ref, m, q, lo, hi);
      if (keep) stv(myp + m * kSpl, q);
#pragma unroll
      for (int k = 0; k < kSpl; k += 2) {
        zl += q[k] + q[k + 1];
        zb += q[k];   // blank states are the even ones
      }
    };
    {   // the window's first round from the ring
      cp_async_wait<1>();
      V va[kSpl], vb[kSpl];
      int e;
      pf.take(slot, lane, clo + lane <= chi && clo + lane < br.nblk, va, vb, e);
      take(va, vb, e, clo + lane, q0, false);
    }
    {   // the rest of a window wider than a round directly
      const typename BandRows<V>::Frame f = br.frame(t);
      for (int m = clo + lane + 32; m <= chi; m += 32) {
        V va[kSpl], vb[kSpl];
        float q[kSpl];
        int e;
        br.load(f, m, true, va, vb, e);
        take(va, vb, e, m, q, true);
      }
    }
    // the window of frame t + 2: this frame's band widened by two frames
    int lo2, hi2;
    br.next_window(lo, hi, 4, lo2, hi2);
    if (t + 2 < tend)
      pf.issue(br, br.frame(t + 2), lo2 + lane, lo2 + lane <= hi2, slot == 0 ? 2 : slot - 1,
               lane);
    cp_async_commit();
    const float z = warp_sum(zl);
    const float zblank = warp_sum(zb);
    const float inv = 1.f / z;
    const float l2 = __log2f(z);
    l2min = fminf(l2min, l2);
    l2max = fmaxf(l2max, l2);
    // label posteriors into the token bins
    if (clo + lane <= chi && clo + lane < br.nblk)
      band_scatter<true>(q0, inv, stok + (clo + lane) * kTokWords, mybins);
    for (int m = clo + lane + 32; m <= chi; m += 32) {
      if (m < br.nblk) {
        float q[kSpl];
        ldv(myp + m * kSpl, q);
        band_scatter<true>(q, inv, stok + m * kTokWords, mybins);
      }
    }
    float sm_k = 0.f;
    if (w.logits) {   // gradient w.r.t. logits: softmax - posterior
      const float x = lane < N ? em[((size_t)b * d.Tmax + t) * N + lane] : -CUDART_INF_F;
      const float mx = warp_max(x);
      const float ex = lane < N ? __expf(x - mx) : 0.f;
      sm_k = ex / warp_sum(ex);
    }
    __syncwarp();
    const float c = lane == blank ? zblank * inv : (float)mybins[lane] * kFixInv;
    mybins[lane] = 0u;
    if (lane < N) ge[(size_t)t * N + lane] = sm_k - c;   // criterion.py:159-161
    __syncwarp();
    clo = nlo;
    chi = nhi;
    nlo = lo2;
    nhi = hi2;
    slot = slot == 2 ? 0 : slot + 1;
  }
  cp_async_wait<0>();
  // the frames' log2-normalisers (ref + log2 z_t) for the guard
  const double gmin = (double)ref + (double)l2min, gmax = (double)ref + (double)l2max;
  if (lane == 0) {
    gw[warp][0] = gmin;
    gw[warp][1] = gmax;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double g = threadIdx.x ? -CUDART_INF : CUDART_INF;
    for (int q = 0; q < kGradWarps; ++q)
      g = threadIdx.x ? fmax(g, gw[q][1]) : fmin(g, gw[q][0]);
    w.part_guard[((size_t)b * w.nblk + blk) * 2 + threadIdx.x] = g;
  }
  W2L_TL(if (threadIdx.x == 0) tl_rec(2000000ull + b * 1000 + blk, tl0, tl1, gtimer()));
}

template <int W, class V>
cudaError_t launch_ctc_grad_w(const float *em, const int32_t *em_len, const int64_t *tgt,
                              const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                              float *grad_em, const int32_t *status, int want, cudaStream_t s,
                              bool stream) {
  const size_t smem = kGradWarps * band_pf_bytes<V>();
  auto k = ctc_grad_kernel<W, V>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(k, dim3(d.B, w.nblk), dim3(kGradWarps * 32), smem, s, true, em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, want,
                          (const int *)(stream ? w.prog : nullptr));
}

// one warp per utterance: loss and guard verdict (partials read in parallel);
// resets the utterance's progress words for the next tier / call
__global__ void ctc_final_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                 double *loss, int32_t *status, int want, int fail) {
  pdl_enter();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= d.B) return;
  if (lane < 2 && w.prog) w.prog[2 * b + lane] = 0;
  if (status[b] != want) {
    // the first tier owns the NaN loss of the utterances it does not
    // compute; a later tier overwrites those it takes
    if (want == W2L_OK && lane == 0) loss[b] = CUDART_NAN;
    return;
  }
  const int T = em_len[b];
  const double ln2 = 0.6931471805599453;
  const double zA = w.scal[b * 4 + 0], zB = w.scal[b * 4 + 1], shifts = w.scal[b * 4 + 2];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)T / 1600.0));
  const int nb_used = (T + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  int bad = 0;
  for (int q = lane; q < nb_used; q += 32) {
    // every frame's log-normaliser (log2 units) must reproduce the total
    const double *g = w.part_guard + ((size_t)b * w.nblk + q) * 2;
    bad |= !(fabs(g[0] * ln2 - zA) <= tol && fabs(g[1] * ln2 - zA) <= tol);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    bad |= !(isfinite(zA) && isfinite(zB)) || !(fabs(zA - zB) <= tol);
    loss[b] = -(zA + shifts);                                  // criterion.py:162
    status[b] = bad ? fail : W2L_OK;
  }
}

// loss only: both directions ran, their totals must agree
__global__ void ctc_loss_only_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                     double *loss, int32_t *status, int want, int fail) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  if (status[b] != want) {
    if (want == W2L_OK) loss[b] = CUDART_NAN;   // (a later tier overwrites those it takes)
    return;
  }
  const double zA = w.scal[b * 4 + 0], zB = w.scal[b * 4 + 1], shifts = w.scal[b * 4 + 2];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)em_len[b] / 1600.0));
  loss[b] = -(zA + shifts);                                  // criterion.py:162
  const bool bad = !(isfinite(zA + shifts) && isfinite(zB)) || !(fabs(zA - zB) <= tol);
  status[b] = bad ? fail : W2L_OK;
}

template <class V>
cudaError_t launch_ctc_tier(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                            double *loss, float *grad_em, int32_t *status, cudaStream_t s,
                            Tracer *tr, unsigned phases, int want, int fail) {
  // stream the gradient behind the chains (PDL) when both run in this call
  // and no stage trace separates them; otherwise the chains publish no
  // progress and the gradient CTAs do not wait
  const bool stream = (phases & 1u) && (phases & 2u) && !(phases & 4u) && !tr &&
                      ((phases & 8u) || pdl_enabled());
  CtcFastWs wc = w;
  if (!stream) wc.prog = nullptr;
  cudaError_t err = cudaSuccess;
  if (phases & 5u) {
    const size_t smem = chain_smem_bytes<V>();
    // (the streamed-gradient trigger is compiled only into the streaming
    // variant: its checks cost the recursion loops ~2.5%)
    auto k = wc.prog ? ctc_chain_kernel<V, true> : ctc_chain_kernel<V, false>;
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    // maximum shared-memory carveout: chain CTAs of different criteria (and
    // several per SM) can then be co-resident on one SM configuration
    err = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (err != cudaSuccess) return err;
    // (loss only runs both directions too: their totals are its guard)
    // (a plain launch: launched early, the waiting chain CTAs would hold the
    // shared memory the other stream's kernels need)
    err = launch_maybe_pdl(k, dim3(d.B, 2), dim3(32 * (1 + w.W)), smem, s, false, em, em_len, tgt,
                           tgt_len, blank, d, wc, status, want, fail);
    if (err != cudaSuccess) return err;
  }
  trace(tr, s);  // chain
  if (phases & 4u) {
    return launch_maybe_pdl(ctc_loss_only_kernel, dim3((d.B + 127) / 128), dim3(128), 0, s, true,
                            em_len, d, w, loss, status, want, fail);
  }
  if (!(phases & 2u)) return cudaSuccess;
  switch (w.W) {
#define W2L_CASE(n)                                                                          \
  case n:                                                                                    \
    if constexpr (n <= kMaxLatWarps) {                                                       \
    err = launch_ctc_grad_w<n, V>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status,    \
                                  want, s, stream);                                          \
    } else {                                                                                 \
      return cudaErrorInvalidValue;                                                          \
    }                                                                                        \
    break;
    W2L_CASE(1) W2L_CASE(2) W2L_CASE(3) W2L_CASE(4) W2L_CASE(5) W2L_CASE(6) W2L_CASE(7)
    W2L_CASE(8)
#undef W2L_CASE
    default: return cudaErrorInvalidValue;
  }
  if (err != cudaSuccess) return err;
  trace(tr, s);  // grad
  err = launch_maybe_pdl(ctc_final_kernel, dim3((d.B + 7) / 8), dim3(256), 0, s, true, em_len, d, w,
                         loss, status, want, fail);
  trace(tr, s);  // final
  return err;
}

}  // namespace

int ctc_fast_spl(int Lmax) { return lat_warps(2 * Lmax + 1) <= kMaxLatWarps ? kSpl : 0; }

static size_t ctc_ws_layout(Dims d, void *base, CtcFastWs *w) {
  const int W = lat_warps(2 * d.Lmax + 1);
  const int lpad = W * kLatStates;
  const int nblk = (d.Tmax + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  const size_t BWT = (size_t)d.B * W * d.Tmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? (void *)((char *)base + o) : nullptr;
  };
  CtcFastWs t;
  // rows sized for the double tier (the float tier uses the first half; the
  // tiers run one after the other on the same stream)
  t.a = take(BWT * kLatStates * sizeof(double));
  t.b = take(BWT * kLatStates * sizeof(double));
  t.ea = (int *)take(BWT * 32 * 4);
  t.eb = (int *)take(BWT * 32 * 4);
  t.scal = (double *)take((size_t)d.B * 4 * 8);
  t.part_guard = (double *)take((size_t)d.B * nblk * 2 * 8);
  t.prog = (int *)take((size_t)d.B * 2 * 4);
  t.route = (int *)take(kRouteWords * 4);
  t.perm = (int *)take((size_t)d.B * lpad * 4);
  t.tok_start = (int *)take((size_t)d.B * 33 * 4);
  t.spl = kSpl;
  t.W = W;
  t.lpad = lpad;
  t.nblk = nblk;
  t.logits = 0;
  if (w) *w = t;
  return off;
}

#ifdef W2L_TIMELINE
int tl_read_ctc(unsigned long long *host, int maxn) {
  unsigned n = 0;
  cudaMemcpyFromSymbol(&n, g_tl_n, sizeof(n));
  n = n < (unsigned)maxn ? n : (unsigned)maxn;
  n = n < (unsigned)kTlMax ? n : (unsigned)kTlMax;
  cudaMemcpyFromSymbol(host, g_tl, sizeof(unsigned long long) * 4 * n);
  const unsigned z = 0;
  cudaMemcpyToSymbol(g_tl_n, &z, sizeof(z));
  return (int)n;
}
#endif

size_t ctc_fast_ws_bytes(Dims d) { return ctc_ws_layout(d, nullptr, nullptr); }
void ctc_fast_ws_carve(Dims d, void *ws, CtcFastWs *w) { ctc_ws_layout(d, ws, w); }

cudaError_t launch_ctc_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                            double *loss, float *grad_em, int32_t *status, cudaStream_t s,
                            Tracer *tr, unsigned phases, int tier) {
  if (w.W < 1 || w.W > kMaxLatWarps) return cudaErrorInvalidValue;
  if (tier == 0)
    return launch_ctc_tier<float>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status,
                                  s, tr, phases, W2L_OK, kNeedsF64);
  return launch_ctc_tier<double>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status,
                                 s, tr, phases, kNeedsF64, kNeedsLog);
}

}  // namespace w2l
