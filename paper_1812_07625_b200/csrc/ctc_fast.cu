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
    double va[SPL], vb[SPL];   // high words of fp64 lane values (lane64.cuh)
    lane_load_hi<SPL>(va, w.a + (row0 + t) * LP, lane);
    lane_load_hi<SPL>(vb, w.b + (row0 + t) * LP, lane);
    const int ea = w.ea[(row0 + t) * 32 + lane];
    const int eb = w.eb[(row0 + t) * 32 + lane];
    const int es = lane_pair_exponent_d<SPL>(va, vb, ea, eb);
    const int estar = warp_max(es);
    const double sc = es > kNegExp / 2 ? pow2d_fast(ea + eb - estar) : 0.0;
    float zl = 0.f, zb = 0.f;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const float p = (float)(va[k] * vb[k] * sc);
      myp[lane * SPL + k] = p;
      zl += p;
      if (((lane * SPL + k) & 1) == 0) zb += p;   // blank states
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

// ------------------------------------------------------------- fused kernel --
// One CTA per utterance: warp 0 = alpha chain, warp 1 = beta chain, then
// H helper warps for alpha and H for beta.  Meet in the middle at row S (a
// multiple of 32, ~T/2):
//   phase 1  alpha computes rows [0, S), beta rows [S, T); each stores its rows
//            with TMA bulk stores out of a shared-memory ring;
//   barrier  bulk writes complete and published (named barrier, all warps);
//   phase 2  alpha computes rows [S, T), beta rows [0, S); each hands its rows
//            through the same ring to its helper warps (mbarrier "full" per
//            slot, per-helper "consumed" counters back), which bulk-prefetch the
//            partner's stored rows (TMA, mbarrier complete_tx) and emit every
//            frame's posteriors, gradient row and guard value.
// Every row is stored once, every posterior is computed once, and the
// gradient work overlaps the serial recursions (no separate gradient pass).
template <int SPL>
struct CtcCfg {
  static constexpr int kUnroll = 4;                   // rows per unrolled block (I-cache)
  static constexpr int kRenorm = 4;                   // rows between lane renormalisations
  static constexpr int kSlot = 2;                     // rows per ring slot
  static constexpr int kRing = 4;                     // slots per chain
  static constexpr int kHelpers = SPL <= 24 ? 3 : 2;  // helper warps per chain
  static constexpr int kWarps = 2 + 2 * kHelpers;
};

template <int SPL>
struct CtcSmem {
  using C = CtcCfg<SPL>;
  static constexpr int kRowI = SPL * 32;
  float raw[2][2][kChunk * kStride];                  // [chain][buffer] raw emission chunks
  double dch[2][2][kChunk * kStride];                 // converted Et (fp64)
  int rv[2][C::kRing][C::kSlot * kRowI];              // ring rows (fp64 high words)
  int re[2][C::kRing][C::kSlot * 32];                 // ring lane exponents
  int pf[2 * C::kHelpers][2][C::kSlot * kRowI];       // partner rows (TMA prefetch)
  int pfe[2 * C::kHelpers][2][C::kSlot * 32];
  uint64_t full[2][C::kRing];                         // chain -> helper
  uint64_t pfbar[2 * C::kHelpers][2];                 // prefetch completion
  volatile int consumed[2 * C::kHelpers];             // helper -> chain (slots released)
  float prow[2 * C::kHelpers][kRowI];                 // helper posterior rows
  double gmin[2 * C::kHelpers], gmax[2 * C::kHelpers];
  int perm[SPL * 16];                                 // label states grouped by token
  double lnz[2], shifts;
};

__device__ __forceinline__ int split_row(int T) { return (T / 64) * 32; }

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void *sdst, const void *gsrc, uint32_t bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// A chain's row sink: phase 1 -> bulk stores to its global rows, phase 2 ->
// the helpers.  Slots are aligned to kSlot in row space; a slot holds the rows
// of one phase only.  Phase-2 slot q goes to helper q % H.
template <int SPL>
struct Emitter {
  using C = CtcCfg<SPL>;
  CtcSmem<SPL> *sm;
  int chain;       // 0 alpha (rows ascending), 1 beta (descending)
  float *grow;     // this chain's rows in the workspace (utterance base)
  int *gexp;
  int S, T;
  bool phase2, met;
  int seq1, seq2;  // slots issued in phase 1 / phase 2
  int seen[C::kHelpers];  // cached consumed counters

  __device__ __forceinline__ int ring() const { return (phase2 ? seq2 : seq1) % C::kRing; }
  __device__ __forceinline__ float *rows() {
    return reinterpret_cast<float *>(sm->rv[chain][ring()]);
  }
  __device__ __forceinline__ int *exps() { return sm->re[chain][ring()]; }
  __device__ __forceinline__ int lo_phase() const { return chain == 0 ? (phase2 ? S : 0) : (phase2 ? 0 : S); }
  __device__ __forceinline__ int hi_phase() const { return chain == 0 ? (phase2 ? T : S) : (phase2 ? S : T); }

  __device__ __forceinline__ void meet(int lane) {
    if (!met) {
      if (lane == 0) bulk_publish();
      __syncwarp();
      named_barrier(1, C::kWarps * 32);
      met = true;
    }
  }
  __device__ __forceinline__ void enter_phase2(int lane) {
    meet(lane);
    phase2 = true;
  }
  __device__ __forceinline__ void acquire(int lane) {
    if (!phase2) {
      if (seq1 >= C::kRing && lane == 0) bulk_wait_read_n<C::kRing - 1>();
    } else if (seq2 >= C::kRing) {
      // slot seq2 - kRing (same ring position) must have been released by its helper
      const int prev = seq2 - C::kRing;
      const int hh = prev % C::kHelpers, need = prev / C::kHelpers + 1;
#pragma unroll
      for (int x = 0; x < C::kHelpers; ++x)
        if (x == hh) {
          while (seen[x] < need) seen[x] = sm->consumed[chain * C::kHelpers + x];
        }
      __threadfence_block();
    }
    __syncwarp();
  }
  // close the open slot, which holds rows [lo, lo + n) at positions lo % kSlot ..
  __device__ __forceinline__ void release(int lo, int n, int lane) {
    if (!phase2) {
      bulk_fence();
      __syncwarp();
      if (lane == 0) {
        constexpr int LP = SPL * 32;
        bulk_store(grow + (size_t)lo * LP, rows() + (lo % C::kSlot) * LP,
                   n * LP * sizeof(int));
        bulk_store(gexp + lo * 32, exps() + (lo % C::kSlot) * 32, n * 32 * sizeof(int));
        bulk_commit();
      }
      ++seq1;
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->full[chain][seq2 % C::kRing]);
      ++seq2;
    }
  }
  // generic per-row protocol around the step that produces row r
  __device__ __forceinline__ void begin(int r, int lane) {
    if (!phase2 && (chain == 0 ? r >= S : r < S)) enter_phase2(lane);
    const int k = r / C::kSlot;
    const int first = chain == 0 ? max(k * C::kSlot, lo_phase())
                                 : min(k * C::kSlot + C::kSlot, hi_phase()) - 1;
    if (r == first) acquire(lane);
  }
  __device__ __forceinline__ void end(int r, int lane) {
    const int k = r / C::kSlot;
    const int lo = max(k * C::kSlot, lo_phase()), hi = min(k * C::kSlot + C::kSlot, hi_phase());
    const int last = chain == 0 ? hi - 1 : lo;
    if (r == last) release(lo, hi - lo, lane);
  }
};

// ---- alpha chain (rows ascending)
template <int SPL>
__device__ void ctc_alpha_chain(CtcSmem<SPL> &sm, const ChainCtx &c, CtcState<SPL> &f,
                                Emitter<SPL> &o, int S_len) {
  constexpr int SLOT = CtcCfg<SPL>::kSlot, UNR = CtcCfg<SPL>::kUnroll, RN = CtcCfg<SPL>::kRenorm;
  const int lane = c.lane, T = c.T, S = o.S;
  const int nch = (T + kChunk - 1) / kChunk;
  double shifts = 0.0;
  f.ex = 0;
  stage_issue(sm.raw[0][0], c, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
    const double *buf = sm.dch[0][ch & 1];
    stage_convert_d(sm.raw[0][ch & 1], sm.dch[0][ch & 1], c, rows, &shifts);
    if (ch + 1 < nch) stage_issue(sm.raw[0][(ch + 1) & 1], c, t0 + kChunk);
    if (ch > 0 && rows == kChunk) {
      if (!o.phase2 && t0 >= S) o.enter_phase2(lane);
#pragma unroll 1
      for (int g = 0; g < kChunk; g += UNR) {
#pragma unroll
        for (int sl = 0; sl < UNR / SLOT; ++sl) {
          o.acquire(lane);
          float *rw = o.rows();
          int *re = o.exps();
#pragma unroll
          for (int q = 0; q < SLOT; ++q) {
            const int qq = sl * SLOT + q;   // position in the unrolled block
            ctc_alpha_step<SPL>(f, buf + (g + qq) * kStride, (qq % RN) == 0, (qq % RN) == 1, rw,
                                re, lane, q);
          }
          o.release(t0 + g + sl * SLOT, SLOT, lane);
        }
      }
    } else {
      for (int r = 0; r < rows; ++r) {
        const int t = t0 + r;
        o.begin(t, lane);
        if (t == 0) {   // criterion.py:123-125
#pragma unroll
          for (int k = 0; k < SPL; ++k) f.v[k] = 0.0;
          if (lane == 0) {
            f.v[0] = buf[f.lab[0]];
            if (S_len > 1) f.v[1] = buf[f.lab[1]];
          }
          lane_renorm_d<SPL>(f.v, f.ex);
          lane_store_hi<SPL>(f.v, f.ex, o.rows(), o.exps(), lane, t % SLOT);
        } else {
          ctc_alpha_step<SPL>(f, buf + r * kStride, (t % RN) == 0 || t == T - 1, true,
                              o.rows(), o.exps(), lane, t % SLOT);
        }
        o.end(t, lane);
      }
    }
  }
  o.meet(lane);
  // log Z = logadd(alpha[S-1], alpha[S-2]) (criterion.py:136-139), in f64
  double part = 0.0;
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    const int s = lane * SPL + k;
    if (s == S_len - 1 || s == S_len - 2) part += f.v[k];
  }
  const double lp_ = part > 0.0 ? log(part) + (double)f.ex * 0.6931471805599453 : -CUDART_INF;
  const double m = warp_max(lp_);
  const double sum = warp_sum(lp_ > -CUDART_INF ? exp(lp_ - m) : 0.0);
  shifts = warp_sum(shifts);
  if (lane == 0) {
    sm.lnz[0] = isfinite(m) ? m + log(sum) : -CUDART_INF;
    sm.shifts = shifts;
  }
  (void)S;
}

// ---- beta chain (rows descending; row r consumes frame r+1).  Chunks are in
// ROW space: chunk c holds rows [32c, 32c+32) = frames 32c+1 .. 32c+32.
template <int SPL>
__device__ void ctc_beta_chain(CtcSmem<SPL> &sm, const ChainCtx &c, CtcState<SPL> &f,
                               Emitter<SPL> &o, int S_len) {
  constexpr int SLOT = CtcCfg<SPL>::kSlot, UNR = CtcCfg<SPL>::kUnroll, RN = CtcCfg<SPL>::kRenorm;
  const int lane = c.lane, T = c.T;
  ChainCtx cf = c;
  cf.e = c.e + c.N;   // frame r+1 for row r
  cf.T = T - 1;       // rows 0 .. T-2 have a step
#pragma unroll
  for (int k = 0; k < SPL; ++k) {   // row T-1: beta' = 1 on the last two states
    const int s = lane * SPL + k;
    f.v[k] = (s == S_len - 1 || s == S_len - 2) ? 1.0 : 0.0;
  }
  f.ex = 0;
  lane_renorm_d<SPL>(f.v, f.ex);
  o.begin(T - 1, lane);
  lane_store_hi<SPL>(f.v, f.ex, o.rows(), o.exps(), lane, (T - 1) % SLOT);
  o.end(T - 1, lane);
  const int nch = (T - 1 + kChunk - 1) / kChunk;   // row chunks with a step
  if (nch > 0) stage_issue(sm.raw[1][(nch - 1) & 1], cf, (nch - 1) * kChunk);
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int r0 = ch * kChunk, rows = min(kChunk, T - 1 - r0);
    const double *buf = sm.dch[1][ch & 1];
    stage_convert_d(sm.raw[1][ch & 1], sm.dch[1][ch & 1], cf, rows);
    if (ch > 0) stage_issue(sm.raw[1][(ch - 1) & 1], cf, r0 - kChunk);
    // full chunk below the top, inside one phase (S is a multiple of kChunk)
    const bool uniform = rows == kChunk && r0 + kChunk <= T - 1 &&
                         (r0 + kChunk <= o.S || r0 >= o.S);
    if (uniform) {
      if (!o.phase2 && r0 + kChunk <= o.S) o.enter_phase2(lane);
#pragma unroll 1
      for (int g = kChunk - UNR; g >= 0; g -= UNR) {
#pragma unroll
        for (int sl = UNR / SLOT - 1; sl >= 0; --sl) {
          o.acquire(lane);
          float *rw = o.rows();
          int *re = o.exps();
#pragma unroll
          for (int q = SLOT - 1; q >= 0; --q) {
            const int qq = sl * SLOT + q;   // row offset in the unrolled block
            ctc_beta_step<SPL>(f, buf + (g + qq) * kStride, (qq % RN) == 0, (qq % RN) == RN - 1,
                               rw, re, lane, q);
          }
          o.release(r0 + g + sl * SLOT, SLOT, lane);
        }
      }
    } else {
      for (int j = rows - 1; j >= 0; --j) {
        const int r = r0 + j;   // produces beta'_r from frame r+1
        o.begin(r, lane);
        ctc_beta_step<SPL>(f, buf + j * kStride, (r % RN) == 0, true, o.rows(), o.exps(),
                           lane, r % SLOT);
        o.end(r, lane);
      }
    }
  }
  o.meet(lane);
  // Z_beta = sum over the two start states of Et_0[lab_s] beta'_0[s]
  const float x = lane < c.N ? c.e[lane] : -CUDART_INF_F;
  const float m0 = warp_max(x);
  const float et = lane < c.N ? expf(x - m0) : 0.f;
  const float el0 = __shfl_sync(0xffffffffu, et, f.lab[0] & 31);
  const float el1 = __shfl_sync(0xffffffffu, et, f.lab[1] & 31);
  if (lane == 0) {
    double z0 = (double)el0 * f.v[0];
    if (S_len > 1) z0 += (double)el1 * f.v[1];
    sm.lnz[1] = log(z0) + (double)f.ex * 0.6931471805599453;
  }
}

// ---- helper: posteriors and gradient rows for the phase-2 slots of a chain
template <int SPL>
__device__ void ctc_helper(CtcSmem<SPL> &sm, int chain, int h, int lane, const CtcFastWs &w,
                           size_t row0, int T, int S, int N, int blank, const int *ts,
                           float *ge) {
  using C = CtcCfg<SPL>;
  constexpr int LP = SPL * 32, SLOT = C::kSlot, H = C::kHelpers;
  const int hid = chain * H + h;
  float *myp = sm.prow[hid];
  const int *prow_g = reinterpret_cast<const int *>(chain == 0 ? w.b : w.a);   // partner rows
  const int *pexp_g = chain == 0 ? w.eb : w.ea;
  const int ts0 = lane < N ? ts[lane] : 0, ts1 = lane < N ? ts[lane + 1] : 0;
  double gmin = CUDART_INF, gmax = -CUDART_INF;
  const int Q = chain == 0 ? (T - S + SLOT - 1) / SLOT : S / SLOT;
  auto rows_of = [&](int q, int &lo, int &hi) {
    const int k = chain == 0 ? S / SLOT + q : S / SLOT - 1 - q;
    lo = k * SLOT;
    hi = min(lo + SLOT, T);
  };
  auto prefetch = [&](int q, int buf) {
    if (lane == 0 && q < Q) {
      int lo, hi;
      rows_of(q, lo, hi);
      const uint32_t bv = (hi - lo) * LP * sizeof(int), be = (hi - lo) * 32 * sizeof(int);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(&sm.pfbar[hid][buf], bv + be);
      bulk_load(sm.pf[hid][buf], prow_g + (row0 + lo) * LP, bv, &sm.pfbar[hid][buf]);
      bulk_load(sm.pfe[hid][buf], pexp_g + (row0 + lo) * 32, be, &sm.pfbar[hid][buf]);
    }
  };
  named_barrier(1, C::kWarps * 32);   // phase 1 finished: partner rows are in memory
  prefetch(h, 0);
  prefetch(h + H, 1);
  int i = 0;
  for (int q = h; q < Q; q += H, ++i) {
    const int buf = i & 1, ring = q % C::kRing;
    int lo, hi;
    rows_of(q, lo, hi);
    mbar_wait(&sm.pfbar[hid][buf], (i >> 1) & 1);
    mbar_wait(&sm.full[chain][ring], (q / C::kRing) & 1);
    for (int r = lo; r < hi; ++r) {
      const int2 *own2 = reinterpret_cast<const int2 *>(sm.rv[chain][ring] + (r % SLOT) * LP + lane * SPL);
      const int2 *oth2 = reinterpret_cast<const int2 *>(sm.pf[hid][buf] + (r - lo) * LP + lane * SPL);
      int oh[SPL], ph[SPL];
#pragma unroll
      for (int k = 0; k < SPL / 2; ++k) {
        const int2 a = own2[k], bq = oth2[k];
        oh[2 * k] = a.x;
        oh[2 * k + 1] = a.y;
        ph[2 * k] = bq.x;
        ph[2 * k + 1] = bq.y;
      }
      const int eo = sm.re[chain][ring][(r % SLOT) * 32 + lane];
      const int ep = sm.pfe[hid][buf][(r - lo) * 32 + lane];
      // largest product exponent of the lane from the stored high words
      // (positive doubles: biased exponent = hi >> 20; zero -> excluded)
      int pe = -(1 << 20);
#pragma unroll
      for (int k = 0; k < SPL; ++k)
        pe = max(pe, (oh[k] && ph[k]) ? (oh[k] >> 20) + (ph[k] >> 20) : -(1 << 20));
      const bool alive = pe > 0 && eo > kNegExp / 2 && ep > kNegExp / 2;
      const int es = alive ? eo + ep + pe - 2046 : kNegExp;
      const int estar = warp_max(es);
      const double sc = alive ? pow2d_fast(max(eo + ep - estar, -1100)) : 0.0;
      float zl = 0.f, zb = 0.f;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const float p = (float)(from_hi(oh[k]) * from_hi(ph[k]) * sc);
        myp[lane * SPL + k] = p;
        zl += p;
        if ((k & 1) == 0) zb += p;   // even states are blanks (SPL is even)
      }
      const float z = warp_sum(zl);
      const float zblank = warp_sum(zb);
      const double g = (double)__log2f(z) + (double)estar;
      gmin = fmin(gmin, g);
      gmax = fmax(gmax, g);
      __syncwarp();
      float acc = lane == blank ? zblank : 0.f;
      for (int qq = ts0; qq < ts1; ++qq) acc += myp[sm.perm[qq]];
      if (lane < N) ge[(size_t)r * N + lane] = -acc / z;   // criterion.py:159-161
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      sm.consumed[hid] = i + 1;   // releases ring slot q back to the chain
    }
    prefetch(q + 2 * H, buf);
  }
  if (lane == 0) {
    sm.gmin[hid] = gmin;
    sm.gmax[hid] = gmax;
  }
}

template <int SPL>
__global__ void __launch_bounds__(CtcCfg<SPL>::kWarps * 32)
    ctc_fused_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     int blank, Dims d, CtcFastWs w, double *loss, float *grad_em,
                     int32_t *status) {
  using C = CtcCfg<SPL>;
  extern __shared__ __align__(128) unsigned char dsm[];
  CtcSmem<SPL> &sm = *reinterpret_cast<CtcSmem<SPL> *>(dsm);
  const int b = blockIdx.x, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N, T = em_len[b];
  float *ge = grad_em + (size_t)b * d.Tmax * N;
  if (status[b] != W2L_OK) {
    for (int i = threadIdx.x; i < d.Tmax * N; i += blockDim.x) ge[i] = 0.f;
    return;
  }
  for (int i = T * N + threadIdx.x; i < d.Tmax * N; i += blockDim.x) ge[i] = 0.f;
  const int L = tgt_len[b], S_len = 2 * L + 1;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  const size_t row0 = (size_t)b * d.Tmax;
  const int S = split_row(T);
  for (int i = threadIdx.x; i < L; i += blockDim.x) sm.perm[i] = w.perm[(size_t)b * w.lpad + i];
  if (threadIdx.x < 2 * C::kHelpers) {
    sm.consumed[threadIdx.x] = 0;
    sm.gmin[threadIdx.x] = CUDART_INF;
    sm.gmax[threadIdx.x] = -CUDART_INF;
  }
  if (threadIdx.x == 0) {
    for (int c2 = 0; c2 < 2; ++c2)
      for (int r = 0; r < C::kRing; ++r) mbar_init(&sm.full[c2][r], 1);
    for (int hh = 0; hh < 2 * C::kHelpers; ++hh) {
      mbar_init(&sm.pfbar[hh][0], 1);
      mbar_init(&sm.pfbar[hh][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (wid < 2) {
    ChainCtx c;
    c.trans = nullptr;
    c.e = em + row0 * N;
    c.N = N;
    c.T = T;
    c.lane = lane;
    c.amax = 0.f;
    CtcState<SPL> f;
    ctc_lattice_lane<SPL, double>(y, L, blank, N, lane, f.lab, f.sk, f.sk2);
    f.blank = blank;
    Emitter<SPL> o;
    o.sm = &sm;
    o.chain = wid;
    o.grow = (wid == 0 ? w.a : w.b) + row0 * (SPL * 32);
    o.gexp = (wid == 0 ? w.ea : w.eb) + row0 * 32;
    o.S = S;
    o.T = T;
    o.phase2 = false;
    o.met = false;
    o.seq1 = 0;
    o.seq2 = 0;
#pragma unroll
    for (int x = 0; x < C::kHelpers; ++x) o.seen[x] = 0;
    if (wid == 0) ctc_alpha_chain<SPL>(sm, c, f, o, S_len);
    else ctc_beta_chain<SPL>(sm, c, f, o, S_len);
    if (lane == 0) bulk_wait_all();
  } else {
    const int hw = wid - 2;
    ctc_helper<SPL>(sm, hw / C::kHelpers, hw % C::kHelpers, lane, w, row0, T, S, N, blank,
                    w.tok_start + b * 33, ge);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double zA = sm.lnz[0], zB = sm.lnz[1];
    const double tol = 1e-4 * fmax(1.0, sqrt((double)T / 1600.0));
    const double ln2 = 0.6931471805599453;
    bool bad = !(isfinite(zA) && isfinite(zB)) || fabs(zA - zB) > tol;
    for (int q = 0; q < 2 * C::kHelpers; ++q) {
      if (sm.gmin[q] <= sm.gmax[q])   // helpers that saw frames
        bad |= !(fabs(sm.gmin[q] * ln2 - zA) <= tol && fabs(sm.gmax[q] * ln2 - zA) <= tol);
    }
    loss[b] = -(zA + sm.shifts);                                 // criterion.py:162
    if (bad) status[b] = kNeedsExact;
  }
}

template <int SPL>
cudaError_t launch_spl(const float *em, const int32_t *em_len, const int64_t *tgt,
                       const int32_t *tgt_len, int blank, Dims d, const CtcFastWs &w,
                       double *loss, float *grad_em, int32_t *status, cudaStream_t s,
                       Tracer *tr) {
  const size_t smem = sizeof(CtcSmem<SPL>);
  auto k = ctc_fused_kernel<SPL>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  k<<<d.B, CtcCfg<SPL>::kWarps * 32, smem, s>>>(em, em_len, tgt, tgt_len, blank, d, w, loss,
                                                 grad_em, status);
  err = cudaGetLastError();
  trace(tr, s);  // chain (fused chains + gradient)
  trace(tr, s);  // grad (inside the fused kernel)
  trace(tr, s);  // final (inside the fused kernel)
  return err;
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
    case 2: err = launch_spl<2>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 4: err = launch_spl<4>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 8: err = launch_spl<8>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 10: err = launch_spl<10>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 12: err = launch_spl<12>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 16: err = launch_spl<16>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 20: err = launch_spl<20>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 24: err = launch_spl<24>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    case 32: err = launch_spl<32>(em, em_len, tgt, tgt_len, blank, d, w, loss, grad_em, status, s, tr); break;
    default: return cudaErrorInvalidValue;
  }
  return err;
}

}  // namespace w2l
