// fp32 batched CTC loss + gradient (replaces criterion.py:84-162 for the
// batched hot path).
//
// The 2L+1-state blank-augmented lattice (criterion.py:113-120) runs in the
// scaled linear domain, SPL states per lane with a per-lane power-of-two
// exponent, exactly like the ASG fac chain:
//   alpha_t[s] = Et[lab_s] (alpha[s] + alpha[s-1] + skip_s alpha[s-2])
//   beta'_t[s] = w[s] + w[s+1] + skip_{s+2} w[s+2],  w = Et+1[lab] beta'_{t+1}
// with Et = exp(logp - max_i logp) and the per-frame shifts summed in f64 for
// the loss.  The gradient kernel forms per-frame posteriors with their own
// normaliser Z_t, gathers them by token (blank = even states, labels through
// a token CSR) and checks the per-frame consistency guard; failing utterances
// are recomputed by the float64 log-domain kernel.

#include "chunk.cuh"
#include "lane64.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kGradFramesPerBlock = 64;
constexpr int kGradWarps = 8;

template <int SPL, class R>
__device__ __forceinline__ void ctc_lattice_lane(const int64_t *y, int L, int blank, int N,
                                                 int lane, int *lab, R *sk, R *sk2) {
  const int S = 2 * L + 1;
  auto skip_of = [&](int s) -> bool {
    return (s & 1) && s >= 3 && s < S && y[s >> 1] != y[(s >> 1) - 1];
  };
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    const int s = lane * SPL + k;
    lab[k] = s < S ? ((s & 1) ? (int)y[s >> 1] : blank) : N;
    sk[k] = skip_of(s) ? R(1) : R(0);
    sk2[k] = skip_of(s + 2) ? R(1) : R(0);
  }
}

template <int SPL>
struct CtcState {
  int lab[SPL];
  double sk[SPL], sk2[SPL], v[SPL];
  int ex, blank;
};

// alpha_t[s] = Et[lab_s] (alpha[s] + alpha[s-1] + skip_s alpha[s-2])  (:126-134), fp64 lanes
template <int SPL>
__device__ __forceinline__ void ctc_alpha_step(CtcState<SPL> &f, const double *row, bool renorm,
                                               bool check, float *out, int *oute, int lane,
                                               int t) {
  // even states are blanks (SPL is even): one shared emission, no skip edge
  double E[SPL];
  const double Eb = row[f.blank];
#pragma unroll
  for (int k = 1; k < SPL; k += 2) E[k] = row[f.lab[k]];
  double nb1 = __shfl_up_sync(0xffffffffu, f.v[SPL - 1], 1);
  double nb2 = __shfl_up_sync(0xffffffffu, f.v[SPL - 2], 1);
  int nbe = __shfl_up_sync(0xffffffffu, f.ex, 1);
  if (lane == 0) {
    nb1 = nb2 = 0.0;
    nbe = kNegExp;
  }
  const double n1 = align_neighbour_d<SPL>(nb1, nbe, f.v, f.ex, check);
  const double n2 = nb2 * pow2d_fast(min(nbe - f.ex, 1000));
#pragma unroll
  for (int k = SPL - 1; k >= 2; --k)
    f.v[k] = (k & 1) ? E[k] * fma(f.sk[k], f.v[k - 2], f.v[k] + f.v[k - 1])
                     : Eb * (f.v[k] + f.v[k - 1]);
  const double v1 = E[1] * fma(f.sk[1], n1, f.v[1] + f.v[0]);
  f.v[0] = Eb * (f.v[0] + n1);
  f.v[1] = v1;
  (void)n2;
  if (renorm) lane_renorm_d<SPL>(f.v, f.ex);
  lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, t);
}

// beta'_{u-1}[s] = w[s] + w[s+1] + skip_{s+2} w[s+2],  w = Et_u[lab] beta'_u  (:147-155)
template <int SPL>
__device__ __forceinline__ void ctc_beta_step(CtcState<SPL> &f, const double *row, bool renorm,
                                              bool check, float *out, int *oute, int lane,
                                              int t_out) {
  double wv[SPL];
  const double Eb = row[f.blank];
#pragma unroll
  for (int k = 0; k < SPL; ++k) wv[k] = ((k & 1) ? row[f.lab[k]] : Eb) * f.v[k];
  double nb1 = __shfl_down_sync(0xffffffffu, wv[0], 1);
  double nb2 = __shfl_down_sync(0xffffffffu, wv[1], 1);
  int nbe = __shfl_down_sync(0xffffffffu, f.ex, 1);
  if (lane == 31) {
    nb1 = nb2 = 0.0;
    nbe = kNegExp;
  }
  const double n1 = align_neighbour_d<SPL>(nb1, nbe, wv, f.ex, check);
  const double n2 = nb2 * pow2d_fast(min(nbe - f.ex, 1000));
#pragma unroll
  for (int k = 0; k < SPL - 2; ++k)
    f.v[k] = (k & 1) ? fma(f.sk2[k], wv[k + 2], wv[k] + wv[k + 1]) : wv[k] + wv[k + 1];
  f.v[SPL - 2] = wv[SPL - 2] + wv[SPL - 1];
  f.v[SPL - 1] = fma(f.sk2[SPL - 1], n2, wv[SPL - 1] + n1);
  if (renorm) lane_renorm_d<SPL>(f.v, f.ex);
  lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, t_out);
}

// One warp per CTA, grid (B, 2): blockIdx.y 0 = alpha, 1 = beta.
template <int SPL>
__global__ void __launch_bounds__(32)
    ctc_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, CtcFastWs w, const int32_t *__restrict__ status) {
  __shared__ __align__(16) float chunk[2][kChunk * kStride];
  __shared__ __align__(16) double dchunk[2][kChunk * kStride];
  extern __shared__ __align__(128) unsigned char dsm[];  // row staging (dynamic)
  RowStage<SPL * 32, 32> &st = *reinterpret_cast<RowStage<SPL * 32, 32> *>(dsm);
  const int b = blockIdx.x, lane = threadIdx.x;
  if (status[b] != W2L_OK) return;
  int gi = 0;
  ChainCtx c;
  c.trans = nullptr;
  c.e = em + (size_t)b * d.Tmax * d.N;
  c.N = d.N;
  c.T = em_len[b];
  c.lane = lane;
  c.amax = 0.f;
  const int T = c.T, L = tgt_len[b], S = 2 * L + 1;
  const bool fwd = blockIdx.y == 0;
  const size_t row0 = (size_t)b * d.Tmax;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  CtcState<SPL> f;
  ctc_lattice_lane<SPL, double>(y, L, blank, d.N, lane, f.lab, f.sk, f.sk2);
  f.blank = blank;
  float *out = (fwd ? w.a : w.b) + row0 * (SPL * 32);
  int *oute = (fwd ? w.ea : w.eb) + row0 * 32;
  const double ln2 = 0.6931471805599453;
  const int nch = (T + kChunk - 1) / kChunk;
  f.ex = 0;

  if (fwd) {
    double shifts = 0.0;
    stage_issue(chunk[0], c, 0);
    for (int ch = 0; ch < nch; ++ch) {
      const double *buf = dchunk[ch & 1];
      const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
      stage_convert_d(chunk[ch & 1], dchunk[ch & 1], c, rows, &shifts);
      if (ch + 1 < nch) stage_issue(chunk[(ch + 1) & 1], c, t0 + kChunk);
      if (ch > 0 && rows == kChunk) {
#pragma unroll 1
        for (int g = 0; g < kChunk; g += kUnroll, ++gi) {
          const int tb = t0 + g;
          const int slot = gi & 1;
          stage_acquire(gi, lane);
#pragma unroll
          for (int q = 0; q < kUnroll; ++q)
            ctc_alpha_step<SPL>(f, buf + (g + q) * kStride, (q % kRenormD) == 0,
                                (q % kRenormD) == 1, st.v[slot], st.e[slot], lane, q);
          stage_release(st, slot, out + (size_t)tb * (SPL * 32), oute + tb * 32, lane);
        }
      } else {
        int r = 0;
        if (ch == 0) {  // criterion.py:123-125
#pragma unroll
          for (int k = 0; k < SPL; ++k) f.v[k] = 0.0;
          if (lane == 0) {
            f.v[0] = buf[f.lab[0]];
            if (S > 1) f.v[1] = buf[f.lab[1]];
          }
          lane_renorm_d<SPL>(f.v, f.ex);
          lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, 0);
          r = 1;
        }
        for (; r < rows; ++r) {
          const int t = t0 + r;
          ctc_alpha_step<SPL>(f, buf + r * kStride, (t % kRenormD) == 0 || t == T - 1, true,
                              out, oute, lane, t);
        }
      }
    }
    stage_drain(lane);
    // log Z = logadd(alpha[S-1], alpha[S-2]) (criterion.py:136-139), in f64
    double part = 0.0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const int s = lane * SPL + k;
      if (s == S - 1 || s == S - 2) part += f.v[k];
    }
    const double lp_ = part > 0.0 ? log(part) + (double)f.ex * ln2 : -CUDART_INF;
    const double m = warp_max(lp_);
    const double sum = warp_sum(lp_ > -CUDART_INF ? exp(lp_ - m) : 0.0);
    shifts = warp_sum(shifts);
    if (lane == 0) {
      w.scal[b * 4 + 0] = isfinite(m) ? m + log(sum) : -CUDART_INF;
      w.scal[b * 4 + 2] = shifts;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const int s = lane * SPL + k;
      f.v[k] = (s == S - 1 || s == S - 2) ? 1.0 : 0.0;
    }
    lane_renorm_d<SPL>(f.v, f.ex);
    lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, T - 1);
    stage_issue(chunk[(nch - 1) & 1], c, (nch - 1) * kChunk);
    double z0 = 0.0;
    for (int ch = nch - 1; ch >= 0; --ch) {
      const double *buf = dchunk[ch & 1];
      const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
      stage_convert_d(chunk[ch & 1], dchunk[ch & 1], c, rows);
      if (ch > 0) stage_issue(chunk[(ch - 1) & 1], c, t0 - kChunk);
      if (ch > 0 && rows == kChunk) {
#pragma unroll 1
        for (int g = kChunk - kUnroll; g >= 0; g -= kUnroll, ++gi) {
          const int ub = t0 + g;
          const int slot = gi & 1;
          stage_acquire(gi, lane);
#pragma unroll
          for (int q = kUnroll - 1; q >= 0; --q)
            ctc_beta_step<SPL>(f, buf + (g + q) * kStride, ((q + kUnroll - 1) % kRenormD) == 0,
                               (q % kRenormD) == 0, st.v[slot], st.e[slot], lane, q);
          stage_release(st, slot, out + (size_t)(ub - 1) * (SPL * 32), oute + (ub - 1) * 32,
                        lane);
        }
      } else {
        for (int r = rows - 1; r >= (ch == 0 ? 1 : 0); --r) {
          const int u = t0 + r;
          ctc_beta_step<SPL>(f, buf + r * kStride, ((u - 1) % kRenormD) == 0 || u == 1, true,
                             out, oute, lane, u - 1);
        }
      }
      if (ch == 0 && lane == 0) {
        z0 = buf[f.lab[0]] * f.v[0];
        if (S > 1) z0 += buf[f.lab[1]] * f.v[1];
      }
    }
    stage_drain(lane);
    if (lane == 0) w.scal[b * 4 + 1] = log(z0) + (double)f.ex * ln2;
  }
}

template <int SPL>
__global__ void __launch_bounds__(kGradWarps * 32)
    ctc_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    int blank, Dims d, CtcFastWs w, float *__restrict__ grad_em,
                    const int32_t *__restrict__ status) {
  constexpr int LP = SPL * 32;
  __shared__ float prow[kGradWarps][LP];
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
  const int L = tgt_len[b], S = 2 * L + 1;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  int lab[SPL];
  float sk[SPL], sk2[SPL];
  ctc_lattice_lane<SPL, float>(y, L, blank, N, lane, lab, sk, sk2);
  (void)S;
  const int *perm = w.perm + (size_t)b * w.lpad;
  const int ts0 = lane < N ? w.tok_start[b * 33 + lane] : 0;
  const int ts1 = lane < N ? w.tok_start[b * 33 + lane + 1] : 0;
  const double ref = w.scal[b * 4 + 0] * 1.4426950408889634;
  float gmin = CUDART_INF_F, gmax = -CUDART_INF_F;
  const size_t row0 = (size_t)b * d.Tmax;
  float *myp = prow[warp];
  const int tend = min(tb, T);
  for (int t = ta; t < tend; ++t) {
    int va[SPL], vb[SPL];   // high words of fp64 lane values (lane64.cuh)
    lane_load_int<SPL>(va, w.a + (row0 + t) * LP, lane);
    lane_load_int<SPL>(vb, w.b + (row0 + t) * LP, lane);
    const int ea = w.ea[(row0 + t) * 32 + lane];
    const int eb = w.eb[(row0 + t) * 32 + lane];
    double pd[SPL];
    const int es = lane_products<SPL>(va, vb, ea, eb, pd);
    const int estar = warp_max(es);
    const double sc = pow2d_fast(max(ea + eb - estar, -1100));
    float zl = 0.f, zb = 0.f;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const float p = (float)(pd[k] * sc);
      myp[lane * SPL + k] = p;
      zl += p;
      if ((k & 1) == 0) zb += p;   // blank states (SPL is even)
    }
    const float z = warp_sum(zl);
    const float zblank = warp_sum(zb);
    const float inv = 1.f / z;
    const float g = (float)((double)__log2f(z) + (double)estar - ref);
    gmin = fminf(gmin, g);
    gmax = fmaxf(gmax, g);
    __syncwarp();
    float acc = lane == blank ? zblank : 0.f;
    for (int q = ts0; q < ts1; ++q) acc += myp[perm[q]];
    if (lane < N) ge[(size_t)t * N + lane] = -acc * inv;   // criterion.py:159-161
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

__global__ void ctc_final_kernel(const int32_t *__restrict__ em_len, Dims d, CtcFastWs w,
                                 double *loss, int32_t *status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B || status[b] != W2L_OK) return;
  const int T = em_len[b];
  const double ln2 = 0.6931471805599453;
  const double zA = w.scal[b * 4 + 0], zB = w.scal[b * 4 + 1], shifts = w.scal[b * 4 + 2];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)T / 1600.0));
  bool bad = !(isfinite(zA) && isfinite(zB)) || fabs(zA - zB) > tol;
  const int nb_used = (T + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  for (int q = 0; q < nb_used && !bad; ++q) {
    const float *g = w.part_guard + ((size_t)b * w.nblk + q) * 2;
    bad |= !(fabs((double)g[0]) * ln2 <= tol && fabs((double)g[1]) * ln2 <= tol);
  }
  loss[b] = -(zA + shifts);                                  // criterion.py:162
  if (bad) status[b] = kNeedsExact;
}

template <int SPL>
cudaError_t launch_spl(const float *em, const int32_t *em_len, const int64_t *tgt,
                       const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                       float *grad_em, const int32_t *status, cudaStream_t s, Tracer *tr) {
  const size_t stage_bytes = sizeof(RowStage<SPL * 32, 32>);
  auto kc = ctc_chain_kernel<SPL>;
  cudaError_t err0 =
      cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_bytes);
  if (err0 != cudaSuccess) return err0;
  kc<<<dim3(d.B, 2), 32, stage_bytes, s>>>(em, em_len, tgt, tgt_len, blank, d, w, status);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  trace(tr, s);  // chain
  ctc_grad_kernel<SPL><<<dim3(w.nblk, d.B), kGradWarps * 32, 0, s>>>(em, em_len, tgt, tgt_len,
                                                                      blank, d, w, grad_em,
                                                                      status);
  return cudaGetLastError();
}

}  // namespace

int ctc_fast_spl(int Lmax) {
  static const int opts[] = {2, 4, 8, 10, 12, 16, 20, 24, 32};
  const int S = 2 * Lmax + 1;
  for (int o : opts)
    if (32 * o >= S) return o;
  return 0;
}

static size_t ctc_ws_layout(Dims d, void *base, CtcFastWs *w) {
  const int spl = ctc_fast_spl(d.Lmax);
  const int lpad = spl * 32;
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
  t.ea = (int *)take(BT * 32 * 4);
  t.eb = (int *)take(BT * 32 * 4);
  t.scal = (double *)take((size_t)d.B * 4 * 8);
  t.part_guard = (float *)take((size_t)d.B * nblk * 2 * 4);
  t.perm = (int *)take((size_t)d.B * lpad * 4);
  t.tok_start = (int *)take((size_t)d.B * 33 * 4);
  t.spl = spl;
  t.lpad = lpad;
  t.nblk = nblk;
  if (w) *w = t;
  return off;
}

size_t ctc_fast_ws_bytes(Dims d) { return ctc_ws_layout(d, nullptr, nullptr); }
void ctc_fast_ws_carve(Dims d, void *ws, CtcFastWs *w) { ctc_ws_layout(d, ws, w); }

cudaError_t launch_ctc_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                            double *loss, float *grad_em, int32_t *status, cudaStream_t s,
                            Tracer *tr) {
  cudaError_t err = cudaSuccess;
  switch (w.spl) {
    case 2: err = launch_spl<2>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 4: err = launch_spl<4>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 8: err = launch_spl<8>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 10: err = launch_spl<10>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 12: err = launch_spl<12>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 16: err = launch_spl<16>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 20: err = launch_spl<20>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 24: err = launch_spl<24>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    case 32: err = launch_spl<32>(em, em_len, tgt, tgt_len, blank, d, w, grad_em, status, s, tr); break;
    default: return cudaErrorInvalidValue;
  }
  if (err != cudaSuccess) return err;
  trace(tr, s);  // grad
  ctc_final_kernel<<<(d.B + 127) / 128, 128, 0, s>>>(em_len, d, w, loss, status);
  err = cudaGetLastError();
  trace(tr, s);  // final
  return err;
}

}  // namespace w2l
