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

#include "laneblock.cuh"
#include "lattice.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

template <bool FWD, class V>
__device__ __forceinline__ void ctc_chain_body(ChainSm<V> &sm, const float *em, int T, int L,
                                               const int64_t *y, int blank, Dims d,
                                               const CtcFastWs &w, int b, unsigned tokmask,
                                               int32_t *status, int fail) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = 2 * L + 1;
  const int weff = lat_warps(S);
  if (warp == 0) {
    ProdCtx pc{em + (size_t)b * d.Tmax * d.N, d.N, T, FWD, weff, w.logits, tokmask};
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
    lattice_run<kCtc, FWD, V>(sm, c, f);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    w.scal[b * 4 + (FWD ? 0 : 1)] = lattice_total(sm, weff);
    if (sm.flush) status[b] = fail;
  }
}

// grid (B, 2): blockIdx.y 0 = forward (alpha), 1 = backward (beta)
template <class V>
__global__ void __launch_bounds__(32 * (1 + kMaxLatWarps))
    ctc_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, CtcFastWs w, int32_t *__restrict__ status, int want,
                     int fail) {
  extern __shared__ __align__(128) unsigned char dsm[];
  ChainSm<V> &sm = *reinterpret_cast<ChainSm<V> *>(dsm);
  const int b = blockIdx.x;
  if (status[b] != want) return;
  if (want == W2L_OK && route_to_f64(w.route)) {   // the batch goes to the fp64 tier
    if (threadIdx.x == 0 && blockIdx.y == 0) status[b] = kNeedsF64;
    return;
  }
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
    ctc_chain_body<true, V>(sm, em, T, L, y, blank, d, w, b, s_mask, status, fail);
  else
    ctc_chain_body<false, V>(sm, em, T, L, y, blank, d, w, b, s_mask, status, fail);
}

constexpr int kGradFramesPerBlock = 128;
constexpr int kGradWarps = 8;

// One warp per frame at a time; lane i owns states 128 sw + 4 i + k of every
// lattice warp sw and token i of the gradient row.  Posteriors are scaled
// into range by the lane exponents against the utterance's reference
// exponent and normalised by their own per-frame sum z_t.  Rows of lanes
// past the lattice's last state were never stored and are read as zero.
template <int W, class V>
__global__ void __launch_bounds__(kGradWarps * 32)
    ctc_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    int blank, Dims d, CtcFastWs w, float *__restrict__ grad_em,
                    const int32_t *__restrict__ status, int want) {
  constexpr int LP = W * kLatStates;
  __shared__ __align__(16) float prow[kGradWarps][LP];
  __shared__ int sperm[LP];
  __shared__ float gw[kGradWarps][2];
  const int b = blockIdx.y, blk = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N, T = em_len[b];
  const int t0 = blk * kGradFramesPerBlock;
  const int st = status[b];
  float *ge = grad_em + (size_t)b * d.Tmax * N;
  const int fpw = kGradFramesPerBlock / kGradWarps;
  const int ta = t0 + warp * fpw, tb = min(ta + fpw, d.Tmax);
  if (want == W2L_OK) {
    // the first tier owns the zeros: padding frames and utterances it does
    // not compute (a later tier rewrites the rows of the ones it takes)
    for (int t = st == W2L_OK ? max(ta, T) : ta; t < tb; ++t)
      if (lane < N) ge[(size_t)t * N + lane] = 0.f;
  }
  if (st != want || t0 >= T) return;
  const int L = tgt_len[b], S = 2 * L + 1;
  const int weff = lat_warps(S);
  for (int i = threadIdx.x; i < L; i += blockDim.x) sperm[i] = w.perm[(size_t)b * w.lpad + i];
  __syncthreads();
  const int ts0 = lane < N ? w.tok_start[b * 33 + lane] : 0;
  const int ts1 = lane < N ? w.tok_start[b * 33 + lane + 1] : 0;
  const double ref = w.scal[b * 4 + 0] * 1.4426950408889634;
  const int refi = isfinite(ref) ? (int)floor(ref) : 0;
  const float reff = isfinite(ref) ? (float)(ref - refi) : CUDART_NAN_F;
  float gmin = CUDART_INF_F, gmax = -CUDART_INF_F;
  const size_t seg0 = (size_t)b * w.W * d.Tmax;
  const V *A = reinterpret_cast<const V *>(w.a) + seg0 * kLatStates + lane * kSpl;
  const V *Bv = reinterpret_cast<const V *>(w.b) + seg0 * kLatStates + lane * kSpl;
  const int *EA = w.ea + seg0 * 32 + lane;
  const int *EB = w.eb + seg0 * 32 + lane;
  const size_t segv = (size_t)d.Tmax * kLatStates;
  const size_t sege = (size_t)d.Tmax * 32;
  float *myp = prow[warp];
  const int tend = min(tb, T);
  for (int t = ta; t < tend; ++t) {
    const size_t tq = (size_t)t * kLatStates;
    float zl = 0.f, zb = 0.f;
#pragma unroll
    for (int sw = 0; sw < W; ++sw) {
      float p[kSpl];
#pragma unroll
      for (int k = 0; k < kSpl; ++k) p[k] = 0.f;
      if (sw < weff && sw * kLatStates + lane * kSpl < S) {
        V va[kSpl], vb[kSpl];
        ldv(A + sw * segv + tq, va);
        ldv(Bv + sw * segv + tq, vb);
        const V sc = pow2_clamped<V>(EA[sw * sege + (size_t)t * 32] + EB[sw * sege + (size_t)t * 32] - refi);
#pragma unroll
        for (int k = 0; k < kSpl; ++k) p[k] = (float)(va[k] * vb[k] * sc);
      }
      if (sw < weff) {
        stv(myp + sw * kLatStates + lane * kSpl, p);
#pragma unroll
        for (int k = 0; k < kSpl; k += 2) {
          zl += p[k] + p[k + 1];
          zb += p[k];   // blank states are the even ones
        }
      }
    }
    const float z = warp_sum(zl);
    const float zblank = warp_sum(zb);
    const float inv = 1.f / z;
    const float g = __log2f(z) - reff;
    gmin = fminf(gmin, g);
    gmax = fmaxf(gmax, g);
    __syncwarp();
    float c0 = lane == blank ? zblank : 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    int q = ts0;
    for (; q + 4 <= ts1; q += 4) {
      c0 += myp[sperm[q]];
      c1 += myp[sperm[q + 1]];
      c2 += myp[sperm[q + 2]];
      c3 += myp[sperm[q + 3]];
    }
    for (; q < ts1; ++q) c0 += myp[sperm[q]];
    float sm_k = 0.f;
    if (w.logits) {   // gradient w.r.t. logits: softmax - posterior
      const float x = lane < N ? em[((size_t)b * d.Tmax + t) * N + lane] : -CUDART_INF_F;
      const float mx = warp_max(x);
      const float ex = lane < N ? __expf(x - mx) : 0.f;
      sm_k = ex / warp_sum(ex);
    }
    if (lane < N) ge[(size_t)t * N + lane] = sm_k - ((c0 + c1) + (c2 + c3)) * inv;   // criterion.py:159-161
    __syncwarp();
  }
  if (lane == 0) {
    gw[warp][0] = gmin;
    gw[warp][1] = gmax;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    float g = threadIdx.x ? -CUDART_INF_F : CUDART_INF_F;
    for (int q = 0; q < kGradWarps; ++q)
      g = threadIdx.x ? fmaxf(g, gw[q][1]) : fminf(g, gw[q][0]);
    w.part_guard[((size_t)b * w.nblk + blk) * 2 + threadIdx.x] = g;
  }
}

template <int W, class V>
cudaError_t launch_ctc_grad_w(const float *em, const int32_t *em_len, const int64_t *tgt,
                              const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                              float *grad_em, const int32_t *status, int want, cudaStream_t s) {
  ctc_grad_kernel<W, V><<<dim3(w.nblk, d.B), kGradWarps * 32, 0, s>>>(
      em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, want);
  return cudaGetLastError();
}

// one warp per utterance: loss and guard verdict (partials read in parallel)
__global__ void ctc_final_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                 double *loss, int32_t *status, int want, int fail) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= d.B || status[b] != want) return;
  const int T = em_len[b];
  const double ln2 = 0.6931471805599453;
  const double zA = w.scal[b * 4 + 0], zB = w.scal[b * 4 + 1], shifts = w.scal[b * 4 + 2];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)T / 1600.0));
  const int nb_used = (T + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  int bad = 0;
  for (int q = lane; q < nb_used; q += 32) {
    const float *g = w.part_guard + ((size_t)b * w.nblk + q) * 2;
    bad |= !(fabs((double)g[0]) * ln2 <= tol && fabs((double)g[1]) * ln2 <= tol);
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
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B || status[b] != want) return;
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
  cudaError_t err = cudaSuccess;
  if (phases & 5u) {
    const size_t smem = sizeof(ChainSm<V>);
    auto k = ctc_chain_kernel<V>;
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    // maximum shared-memory carveout: chain CTAs of different criteria (and
    // several per SM) can then be co-resident on one SM configuration
    err = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (err != cudaSuccess) return err;
    // (loss only runs both directions too: their totals are its guard)
    k<<<dim3(d.B, 2), 32 * (1 + w.W), smem, s>>>(em, em_len, tgt, tgt_len, blank, d, w, status,
                                                 want, fail);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  trace(tr, s);  // chain
  if (phases & 4u) {
    ctc_loss_only_kernel<<<(d.B + 127) / 128, 128, 0, s>>>(em_len, d, w, loss, status, want,
                                                           fail);
    return cudaGetLastError();
  }
  if (!(phases & 2u)) return cudaSuccess;
  switch (w.W) {
#define W2L_CASE(n)                                                                          \
  case n:                                                                                    \
    if constexpr (n <= kMaxLatWarps) {                                                       \
    err = launch_ctc_grad_w<n, V>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status,    \
                                  want, s);                                                  \
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
  ctc_final_kernel<<<(d.B + 7) / 8, 256, 0, s>>>(em_len, d, w, loss, status, want, fail);
  err = cudaGetLastError();
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
  t.part_guard = (float *)take((size_t)d.B * nblk * 2 * 4);
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
