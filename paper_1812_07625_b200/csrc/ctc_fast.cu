// fp32 batched CTC loss + gradient (replaces criterion.py:84-162 for the
// batched hot path).
//
// The 2L+1-state blank-augmented lattice (criterion.py:113-120) runs in the
// scaled linear domain on the multi-warp wavefront lattice of lattice.cuh
// (4 states per lane, fp64 with a per-lane power-of-two exponent):
//   alpha_t[s] = Et[lab_s] (alpha[s] + alpha[s-1] + skip_s alpha[s-2])
//   beta'_t[s] = w[s] + w[s+1] + skip_{s+2} w[s+2],  w = Et+1[lab] beta'_{t+1}
// with Et = exp(logp - max_i logp) and the per-frame shifts summed in f64 for
// the loss.  The gradient kernel forms per-frame posteriors with their own
// normaliser Z_t, gathers them by token (blank = even states, labels through
// a token CSR) and checks the per-frame consistency guard; failing utterances
// are recomputed by the float64 log-domain kernel.

#include "laneblock.cuh"
#include "lattice.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kGradFramesPerBlock = 128;
constexpr int kGradWarps = 8;

template <bool FWD>
__device__ __forceinline__ void ctc_chain_body(ChainSm &sm, unsigned char *dsm, int W,
                                               const float *em, int T, int L,
                                               const int64_t *y, int blank, Dims d,
                                               const CtcFastWs &w, int b, unsigned tokmask,
                                               int32_t *status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = 2 * L + 1;
  const int weff = lat_warps(S);
  if (warp == 0) {
    ProdCtx pc{em + (size_t)b * d.Tmax * d.N, d.N, T, FWD, W, w.logits, tokmask};
    producer_run(sm, pc, lane, FWD ? w.scal + b * 4 + 2 : nullptr);
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
    c.rows = (FWD ? w.a : w.b) + ub * kLatStates;
    c.exps = (FWD ? w.ea : w.eb) + ub * 32;
    LatState f;
    lat_init_weights<kCtc, FWD>(f, c, y, L, nullptr, 0.f, blank);
    lattice_run<kCtc, FWD>(sm, c, f);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    w.scal[b * 4 + (FWD ? 0 : 1)] = lattice_total(sm, weff);
    if (sm.flush) status[b] = kNeedsExact;
  }
}

// grid (B, 2): blockIdx.y 0 = forward (alpha), 1 = backward (beta)
__global__ void __launch_bounds__(32 * (1 + kMaxLatWarps))
    ctc_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, CtcFastWs w, int32_t *__restrict__ status) {
  extern __shared__ __align__(128) unsigned char dsm[];
  const int W = w.W;
  ChainSm &sm = *reinterpret_cast<ChainSm *>(dsm);
  const int b = blockIdx.x;
  if (status[b] != W2L_OK) return;
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
    ctc_chain_body<true>(sm, dsm, W, em, T, L, y, blank, d, w, b, s_mask, status);
  else
    ctc_chain_body<false>(sm, dsm, W, em, T, L, y, blank, d, w, b, s_mask, status);
}

size_t ctc_chain_smem(int W) { (void)W; return sizeof(ChainSm); }

// 2^x as a float for integer x clamped to [-127, 127] (0 below)
__device__ __forceinline__ float pow2_clamped(int x) { return pow2f_fast(max(min(x, 127), -127)); }

// One warp per frame at a time; lane i owns states 128 w + 4 i + k of every
// segment w and token i of the gradient row.  Posteriors are scaled into
// range by the lane exponents against the utterance's reference exponent
// and normalised by their own per-frame sum z_t.
template <int W>
__global__ void __launch_bounds__(kGradWarps * 32)
    ctc_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    int blank, Dims d, CtcFastWs w, float *__restrict__ grad_em,
                    const int32_t *__restrict__ status) {
  constexpr int LP = W * kLatStates;
  __shared__ __align__(16) float prow[kGradWarps][LP];
  __shared__ int sperm[LP];
  __shared__ float gw[kGradWarps][2];
  const int b = blockIdx.y, blk = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N, T = em_len[b];
  const int t0 = blk * kGradFramesPerBlock;
  const bool ok = status[b] == W2L_OK;
  float *ge = grad_em + (size_t)b * d.Tmax * N;
  const int fpw = kGradFramesPerBlock / kGradWarps;
  const int ta = t0 + warp * fpw, tb = min(ta + fpw, d.Tmax);
  for (int t = ta; t < tb; ++t)
    if (!ok || t >= T)
      if (lane < N) ge[(size_t)t * N + lane] = 0.f;
  if (!ok) return;
  const int L = tgt_len[b];
  const int weff = lat_warps(2 * L + 1);
  for (int i = threadIdx.x; i < L; i += blockDim.x) sperm[i] = w.perm[(size_t)b * w.lpad + i];
  __syncthreads();
  const int ts0 = lane < N ? w.tok_start[b * 33 + lane] : 0;
  const int ts1 = lane < N ? w.tok_start[b * 33 + lane + 1] : 0;
  const double ref = w.scal[b * 4 + 0] * 1.4426950408889634;
  const int refi = isfinite(ref) ? (int)floor(ref) : 0;
  const float reff = isfinite(ref) ? (float)(ref - refi) : CUDART_NAN_F;
  float gmin = CUDART_INF_F, gmax = -CUDART_INF_F;
  const size_t seg0 = (size_t)b * w.W * d.Tmax;
  const float4 *A4 = reinterpret_cast<const float4 *>(w.a + seg0 * kLatStates) + lane;
  const float4 *B4 = reinterpret_cast<const float4 *>(w.b + seg0 * kLatStates) + lane;
  const int *EA = w.ea + seg0 * 32 + lane;
  const int *EB = w.eb + seg0 * 32 + lane;
  const unsigned segq = (unsigned)d.Tmax * (kLatStates / 4);
  const unsigned sege = (unsigned)d.Tmax * 32;
  float *myp = prow[warp];
  const int tend = min(tb, T);
  for (int t = ta; t < tend; ++t) {
    const unsigned tq = (unsigned)t * 32;
    float zl = 0.f, zb = 0.f;
#pragma unroll
    for (int sw = 0; sw < W; ++sw) {
      if (sw < weff) {
        const float4 va = A4[sw * segq + tq];
        const float4 vb = B4[sw * segq + tq];
        const float sc = pow2_clamped(EA[sw * sege + tq] + EB[sw * sege + tq] - refi);
        float4 p;
        p.x = va.x * vb.x * sc;
        p.y = va.y * vb.y * sc;
        p.z = va.z * vb.z * sc;
        p.w = va.w * vb.w * sc;
        reinterpret_cast<float4 *>(myp + sw * kLatStates)[lane] = p;
        zl += (p.x + p.y) + (p.z + p.w);
        zb += p.x + p.z;   // blank states are the even ones
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
    if (lane < N) ge[(unsigned)t * N + lane] = sm_k - ((c0 + c1) + (c2 + c3)) * inv;   // criterion.py:159-161
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

template <int W>
cudaError_t launch_ctc_grad_w(const float *em, const int32_t *em_len, const int64_t *tgt,
                              const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                              float *grad_em, const int32_t *status, cudaStream_t s) {
  ctc_grad_kernel<W><<<dim3(w.nblk, d.B), kGradWarps * 32, 0, s>>>(em, em_len, tgt, tgt_len,
                                                                   blank, d, w, grad_em, status);
  return cudaGetLastError();
}

// one warp per utterance: loss and guard verdict (partials read in parallel)
__global__ void ctc_final_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                 double *loss, int32_t *status) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= d.B || status[b] != W2L_OK) return;
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
    bad |= !(isfinite(zA) && isfinite(zB)) || fabs(zA - zB) > tol;
    loss[b] = -(zA + shifts);                                  // criterion.py:162
    if (bad) status[b] = kNeedsExact;
  }
}

// loss only: both directions ran, their totals must agree
__global__ void ctc_loss_only_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                     double *loss, int32_t *status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B || status[b] != W2L_OK) return;
  const double zA = w.scal[b * 4 + 0], zB = w.scal[b * 4 + 1], shifts = w.scal[b * 4 + 2];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)em_len[b] / 1600.0));
  loss[b] = -(zA + shifts);                                  // criterion.py:162
  if (!(isfinite(zA + shifts) && isfinite(zB)) || !(fabs(zA - zB) <= tol))
    status[b] = kNeedsExact;
}

}  // namespace

#ifdef W2L_PROF
W2L_PROF_READER(w2l_debug_prof_ctc)
#endif

int ctc_fast_spl(int Lmax) { return lat_warps(2 * Lmax + 1) <= kMaxLatWarps ? kSpl : 0; }

static size_t ctc_ws_layout(Dims d, void *base, CtcFastWs *w) {
  const int W = lat_warps(2 * d.Lmax + 1);
  const int lpad = W * kLatStates;
  const int nblk = (d.Tmax + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  const size_t BT = (size_t)d.B * d.Tmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? (void *)((char *)base + o) : nullptr;
  };
  CtcFastWs t;
  t.a = (float *)take(BT * lpad * 4);
  t.b = (float *)take(BT * lpad * 4);
  t.ea = (int *)take(BT * W * 32 * 4);
  t.eb = (int *)take(BT * W * 32 * 4);
  t.scal = (double *)take((size_t)d.B * 4 * 8);
  t.part_guard = (float *)take((size_t)d.B * nblk * 2 * 4);
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
                            Tracer *tr, unsigned phases) {
  if (w.W < 1 || w.W > kMaxLatWarps) return cudaErrorInvalidValue;
  cudaError_t err = cudaSuccess;
  if (phases & 5u) {
    const size_t smem = ctc_chain_smem(w.W);
    err = cudaFuncSetAttribute(ctc_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (err != cudaSuccess) return err;
    // maximum shared-memory carveout: chain CTAs of different criteria (and
    // several per SM) can then be co-resident on one SM configuration
    err = cudaFuncSetAttribute(ctc_chain_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (err != cudaSuccess) return err;
    // (loss only runs both directions too: their totals are its guard)
    ctc_chain_kernel<<<dim3(d.B, 2), 32 * (1 + w.W), smem, s>>>(
        em, em_len, tgt, tgt_len, blank, d, w, status);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  trace(tr, s);  // chain
  if (phases & 4u) {
    ctc_loss_only_kernel<<<(d.B + 127) / 128, 128, 0, s>>>(em_len, d, w, loss, status);
    return cudaGetLastError();
  }
  if (!(phases & 2u)) return cudaSuccess;
  switch (w.W) {
    case 1: err = launch_ctc_grad_w<1>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 2: err = launch_ctc_grad_w<2>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 3: err = launch_ctc_grad_w<3>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 4: err = launch_ctc_grad_w<4>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 5: err = launch_ctc_grad_w<5>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 6: err = launch_ctc_grad_w<6>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 7: err = launch_ctc_grad_w<7>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    case 8: err = launch_ctc_grad_w<8>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (err != cudaSuccess) return err;
  trace(tr, s);  // grad
  ctc_final_kernel<<<(d.B + 7) / 8, 256, 0, s>>>(em_len, d, w, loss, status);
  err = cudaGetLastError();
  trace(tr, s);  // final
  return err;
}

}  // namespace w2l
