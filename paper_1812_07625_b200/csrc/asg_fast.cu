// fp32 batched ASG loss + gradient (replaces criterion.py:167-247 for the
// batched hot path).
//
// Algorithm: the four ASG recursions are run in the SCALED LINEAR domain,
// the standard exact reformulation of log-space forward-backward
//     alpha_t = Et (.) (M alpha_{t-1}) * 2^-k_t ,   M = exp(A - max A),
//     Et[i]   = exp(e[t][i] - max_i e[t][i]),
// with exact power-of-two rescaling (only integer exponents accumulate, no
// rounding in the scale factors).  The fcc (fully connected, N x N) graph is
// a 32-lane mat-vec per frame with the previous vector broadcast through
// shared memory; the fac (forced alignment, L-state chain) graph keeps SPL
// states per lane in registers with a per-lane power-of-two exponent
// (block floating point) and a single shuffle per frame to the neighbour.
// No transcendental sits on the recursion's critical path.
//
// Kernels (one stream, in order):
//   asg_csr      per utterance: states grouped by token (for the emissions
//                gradient scatter), written to the workspace.
//   asg_chain    grid (B, 4): fcc-alpha, fcc-beta, fac-alpha, fac-beta; one
//                warp each; rows of alpha/beta and exponents to workspace.
//   asg_grad     grid (frame blocks, B): 8 warps, one frame per warp at a time:
//                posteriors (per-frame normaliser Z_t), grad_e, partial
//                transition gradients, and the consistency guard G_t.
//   asg_final    per utterance: loss, grad_A_b, guard verdict -> either OK or
//                kNeedsExact (then the float64 kernel recomputes it).
// Reference correspondence: fac alpha/beta = criterion.py:193-212, fac
// posteriors = :214-224, fcc = :227-241, combine = :243-247.

#include "chunk.cuh"
#include "lane64.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kGradFramesPerBlock = 64;
constexpr int kGradWarps = 8;

__device__ __forceinline__ float trans_max(const float *trans, int N) {
  float m = -CUDART_INF_F;
  for (int p = threadIdx.x & 31; p < N * N; p += 32) m = fmaxf(m, trans[p]);
  return warp_max(m);
}

// ---------------------------------------------------------- chain kernel --
// One warp per (utterance, role).  Loops are chunk-major: a chunk of kChunk
// frames is staged (cp.async, one chunk in flight) and converted to Et once;
// full chunks are then walked in fully unrolled blocks of kUnroll frames, so
// every shared-memory row offset, store offset, buffer parity and
// renormalisation decision is a compile-time constant (no per-frame address
// arithmetic or branches on the critical path).  The first/last partial
// chunks take a generic per-frame path.
// Rescaling is lazy and exact (powers of two):
//   fcc: the exponent of sum(vector read this step) arrives through a spare
//        lane (row of ones in M) after the step's own scale is chosen; the
//        scale is predicted from the last two observed log-masses
//        (LaggedScale) -- off the critical path (for N = 32 every lane sums);
//   fac: each lane renormalises its block every kRenorm frames.
// Growth between rescales is bounded; whatever the bounds cannot cover (huge
// transition ranges, emissions that underflow) trips the guard.

// Power-of-two scale for a recursion whose vector sum is only known one
// step late.  At step t the exponent e_{t-1} of the vector consumed by step t
// becomes available after step t's own scale k_t is chosen, so k_t is
// predicted from the true (unscaled) log-masses X_s = e_s + K_s:
// K_t = X_{t-2} + (X_{t-2} - X_{t-3}).  The scaled log-mass is then
// x_t = (X_t - X_{t-2}) - (X_{t-2} - X_{t-3}), bounded by the per-step growth
// of the recursion -- unlike k_t = e_{t-2} directly, whose
// x_t = g + x_{t-1} - x_{t-2} is only marginally stable and drifts.
struct LaggedScale {
  int K1 = 0;                    // cumulative exponent of the newest vector
  int X2 = 0, X3 = 0, seen = 0;  // log-masses of the last two observed vectors
  int pending_K = 0;             // K of the vector whose exponent arrives next
  __device__ __forceinline__ int next() {
    int Kt = K1;
    if (seen >= 2) Kt = X2 + (X2 - X3);
    else if (seen == 1) Kt = X2;
    const int k = max(-120, min(120, Kt - K1));
    pending_K = K1;
    K1 += k;
    return k;
  }
  __device__ __forceinline__ void observe(int e) {
    X3 = X2;
    X2 = e + pending_K;
    ++seen;
  }
};

// ---- fcc: one frame of the 32-lane mat-vec recursion.  `vin` is the vector
// of the previous step (alpha_{t-1}, or w_u = Et_u * beta'_u), m the lane's
// row (alpha) or column (beta) of M; returns the unscaled product.
__device__ __forceinline__ float fcc_matvec(const float (&m)[32], const float *vin, bool spare,
                                            int N, int &e_sum) {
  const float4 *pv = reinterpret_cast<const float4 *>(vin);
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 x = pv[q];
    acc[q] = m[4 * q] * x.x;
    acc[q] = fmaf(m[4 * q + 1], x.y, acc[q]);
    acc[q] = fmaf(m[4 * q + 2], x.z, acc[q]);
    acc[q] = fmaf(m[4 * q + 3], x.w, acc[q]);
  }
  const float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  if (spare) {
    e_sum = exponent_of(__shfl_sync(0xffffffffu, s, N));   // lane N: row of ones
  } else {
    float tot = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) tot += (pv[q].x + pv[q].y) + (pv[q].z + pv[q].w);
    e_sum = exponent_of(tot);
  }
  return s;
}

struct FccState {
  float m[32];
  float v;       // this lane's current alpha_t / beta'_t
  int K;
  LaggedScale sc;
  bool spare;
};

// fcc alpha step t (criterion.py:230): alpha_t = Et (.) (M alpha_{t-1}) 2^-k
__device__ __forceinline__ void fcc_alpha_step(FccState &f, const float *row, float (*vec)[32],
                                               int par, float *out_row, int *outk_t, int lane,
                                               int N) {
  const float et = row[lane];
  __syncwarp();
  int e1;
  const float s = fcc_matvec(f.m, vec[par ^ 1], f.spare, N, e1);
  const int k = f.sc.next();
  f.K += k;
  f.v = et * (s * pow2f(-k));
  f.sc.observe(e1);
  vec[par][lane] = f.v;
  out_row[lane] = f.v;
  if (lane == 0) *outk_t = f.K;
}

// fcc beta' step consuming frame u (criterion.py:236): beta'_{u-1} = M^T (Et_u beta'_u) 2^-k
__device__ __forceinline__ void fcc_beta_step(FccState &f, const float *row, float (*vec)[32],
                                              int par, float *out_row, int *outk_t, int lane,
                                              int N) {
  vec[par][lane] = row[lane] * f.v;
  __syncwarp();
  int e1;
  const float s = fcc_matvec(f.m, vec[par], f.spare, N, e1);
  const int k = f.sc.next();
  f.K += k;
  f.v = lane < N ? s * pow2f(-k) : 0.f;
  f.sc.observe(e1);
  out_row[lane] = f.v;
  if (lane == 0) *outk_t = f.K;
}

__device__ __forceinline__ void fcc_alpha(const ChainCtx &c, float (*chunk)[kChunk * kStride],
                                          float (*vec)[32], RowStage<32, 1> &st, float *out,
                                          int *outk, double *lnz) {
  int gi = 0;
  const int lane = c.lane, N = c.N, T = c.T;
  FccState f;
  f.spare = N < 32;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    f.m[j] = (lane < N && j < N) ? expf(c.trans[lane * N + j] - c.amax)
                                 : ((f.spare && lane == N && j < N) ? 1.f : 0.f);
  f.K = 0;
  const int nch = (T + kChunk - 1) / kChunk;
  stage_issue(chunk[0], c, 0);
  for (int ch = 0; ch < nch; ++ch) {
    float *buf = chunk[ch & 1];
    const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
    stage_convert(buf, c, rows);
    if (ch + 1 < nch) stage_issue(chunk[(ch + 1) & 1], c, t0 + kChunk);
    if (ch > 0 && rows == kChunk) {
#pragma unroll 1
      for (int g = 0; g < kChunk; g += kUnroll, ++gi) {
        const int tb = t0 + g;   // multiple of kUnroll: parities are static
        const int slot = gi & 1;
        stage_acquire(gi, lane);
#pragma unroll
        for (int q = 0; q < kUnroll; ++q)
          fcc_alpha_step(f, buf + (g + q) * kStride, vec, q & 1, st.v[slot] + q * 32,
                         st.e[slot] + q, lane, N);
        stage_release(st, slot, out + tb * 32, outk + tb, lane);
      }
    } else {
      int r = 0;
      if (ch == 0) {
        f.v = buf[lane];               // alpha_0 = Et_0 (criterion.py:228)
        vec[0][lane] = f.v;
        out[lane] = f.v;
        if (lane == 0) outk[0] = 0;
        r = 1;
      }
      for (; r < rows; ++r) {
        const int t = t0 + r;
        fcc_alpha_step(f, buf + r * kStride, vec, t & 1, out + t * 32, outk + t, lane, N);
      }
    }
  }
  stage_drain(lane);
  const float z = warp_sum(lane < N ? f.v : 0.f);
  if (lane == 0) *lnz = log((double)z) + (double)f.K * 0.6931471805599453;
}

__device__ __forceinline__ void fcc_beta(const ChainCtx &c, float (*chunk)[kChunk * kStride],
                                         float (*vec)[32], RowStage<32, 1> &st, float *out,
                                         int *outk, double *lnz) {
  int gi = 0;
  const int lane = c.lane, N = c.N, T = c.T;
  FccState f;
  f.spare = N < 32;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    f.m[i] = (lane < N && i < N) ? expf(c.trans[i * N + lane] - c.amax)
                                 : ((f.spare && lane == N && i < N) ? 1.f : 0.f);
  f.K = 0;
  f.v = lane < N ? 1.f : 0.f;
  out[(T - 1) * 32 + lane] = f.v;
  if (lane == 0) outk[T - 1] = 0;
  const int nch = (T + kChunk - 1) / kChunk;
  stage_issue(chunk[(nch - 1) & 1], c, (nch - 1) * kChunk);
  float e0 = 0.f;
  for (int ch = nch - 1; ch >= 0; --ch) {
    float *buf = chunk[ch & 1];
    const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
    stage_convert(buf, c, rows);
    if (ch > 0) stage_issue(chunk[(ch - 1) & 1], c, t0 - kChunk);
    if (ch > 0 && rows == kChunk) {
#pragma unroll 1
      for (int g = kChunk - kUnroll; g >= 0; g -= kUnroll, ++gi) {
        const int ub = t0 + g;
        const int slot = gi & 1;
        stage_acquire(gi, lane);
#pragma unroll
        for (int q = kUnroll - 1; q >= 0; --q)
          fcc_beta_step(f, buf + (g + q) * kStride, vec, q & 1, st.v[slot] + q * 32,
                        st.e[slot] + q, lane, N);
        stage_release(st, slot, out + (ub - 1) * 32, outk + ub - 1, lane);
      }
    } else {
      for (int r = rows - 1; r >= (ch == 0 ? 1 : 0); --r) {
        const int u = t0 + r;   // consumes frame u, produces beta'_{u-1}
        fcc_beta_step(f, buf + r * kStride, vec, u & 1, out + (u - 1) * 32, outk + u - 1,
                      lane, N);
      }
    }
    if (ch == 0) e0 = buf[lane];
  }
  stage_drain(lane);
  const float z = warp_sum(e0 * f.v);
  if (lane == 0) *lnz = log((double)z) + (double)f.K * 0.6931471805599453;
}

// fac chain weights for this lane's states l = lane*SPL + k: token, stay
// weight M[y_l][y_l] and the step weight (alpha: INTO l from l-1; beta: from
// l INTO l+1).  Padding states read the zero emission column N.
template <int SPL>
__device__ __forceinline__ void fac_weights(const ChainCtx &c, const int64_t *y, int L,
                                            bool is_alpha, int (&tok)[SPL], double (&S)[SPL],
                                            double (&P)[SPL]) {
  const int N = c.N;
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    const int l = c.lane * SPL + k;
    if (l < L) {
      const int yl = (int)y[l];
      tok[k] = yl;
      S[k] = (double)expf(c.trans[yl * N + yl] - c.amax);
      if (is_alpha)
        P[k] = l > 0 ? (double)expf(c.trans[yl * N + (int)y[l - 1]] - c.amax) : 0.0;
      else
        P[k] = l + 1 < L ? (double)expf(c.trans[(int)y[l + 1] * N + yl] - c.amax) : 0.0;
    } else {
      tok[k] = N;
      S[k] = 0.0;
      P[k] = 0.0;
    }
  }
}

template <int SPL>
struct FacState {
  int tok[SPL];
  double S[SPL], P[SPL], v[SPL];
  int ex;
};

// fac alpha step t (criterion.py:197-202), fp64 lane block
template <int SPL>
__device__ __forceinline__ void fac_alpha_step(FacState<SPL> &f, const double *row, bool renorm,
                                               bool check, float *out, int *oute, int lane,
                                               int t) {
  double E[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) E[k] = row[f.tok[k]];
  double nb = __shfl_up_sync(0xffffffffu, f.v[SPL - 1], 1);
  int nbe = __shfl_up_sync(0xffffffffu, f.ex, 1);
  if (lane == 0) {
    nb = 0.0;
    nbe = kNegExp;
  }
  const double nbs = align_neighbour_d<SPL>(nb, nbe, f.v, f.ex, check);
#pragma unroll
  for (int k = SPL - 1; k >= 1; --k) f.v[k] = E[k] * fma(f.S[k], f.v[k], f.P[k] * f.v[k - 1]);
  f.v[0] = E[0] * fma(f.S[0], f.v[0], f.P[0] * nbs);
  if (renorm) lane_renorm_d<SPL>(f.v, f.ex);
  lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, t);
}

// fac beta' step consuming frame u (criterion.py:207-212)
template <int SPL>
__device__ __forceinline__ void fac_beta_step(FacState<SPL> &f, const double *row, bool renorm,
                                              bool check, float *out, int *oute, int lane,
                                              int t_out) {
  double wv[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) wv[k] = row[f.tok[k]] * f.v[k];
  double nb = __shfl_down_sync(0xffffffffu, wv[0], 1);
  int nbe = __shfl_down_sync(0xffffffffu, f.ex, 1);
  if (lane == 31) {
    nb = 0.0;
    nbe = kNegExp;
  }
  const double nbs = align_neighbour_d<SPL>(nb, nbe, wv, f.ex, check);
#pragma unroll
  for (int k = 0; k < SPL - 1; ++k) f.v[k] = fma(f.S[k], wv[k], f.P[k] * wv[k + 1]);
  f.v[SPL - 1] = fma(f.S[SPL - 1], wv[SPL - 1], f.P[SPL - 1] * nbs);
  if (renorm) lane_renorm_d<SPL>(f.v, f.ex);
  lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, t_out);
}

template <int SPL>
__device__ __forceinline__ void fac_alpha(const ChainCtx &c, float (*chunk)[kChunk * kStride],
                                          double (*dchunk)[kChunk * kStride],
                                          RowStage<SPL * 32, 32> &st, const int64_t *y, int L,
                                          float *out, int *oute, double *lnz) {
  int gi = 0;
  const int lane = c.lane, T = c.T;
  FacState<SPL> f;
  fac_weights<SPL>(c, y, L, true, f.tok, f.S, f.P);
  f.ex = 0;
  const int nch = (T + kChunk - 1) / kChunk;
  stage_issue(chunk[0], c, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const double *buf = dchunk[ch & 1];
    const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
    stage_convert_d(chunk[ch & 1], dchunk[ch & 1], c, rows);
    if (ch + 1 < nch) stage_issue(chunk[(ch + 1) & 1], c, t0 + kChunk);
    if (ch > 0 && rows == kChunk) {
#pragma unroll 1
      for (int g = 0; g < kChunk; g += kUnroll, ++gi) {
        const int tb = t0 + g;
        const int slot = gi & 1;
        stage_acquire(gi, lane);
#pragma unroll
        for (int q = 0; q < kUnroll; ++q)
          fac_alpha_step<SPL>(f, buf + (g + q) * kStride, (q % kRenormD) == 0,
                              (q % kRenormD) == 1, st.v[slot], st.e[slot], lane, q);
        stage_release(st, slot, out + (size_t)tb * (SPL * 32), oute + tb * 32, lane);
      }
    } else {
      int r = 0;
      if (ch == 0) {   // t = 0: only the first target state is reachable (:194)
#pragma unroll
        for (int k = 0; k < SPL; ++k) f.v[k] = 0.0;
        if (lane == 0) f.v[0] = buf[f.tok[0]];
        lane_renorm_d<SPL>(f.v, f.ex);
        lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, 0);
        r = 1;
      }
      for (; r < rows; ++r) {
        const int t = t0 + r;
        fac_alpha_step<SPL>(f, buf + r * kStride, (t % kRenormD) == 0 || t == T - 1, true, out,
                            oute, lane, t);
      }
    }
  }
  stage_drain(lane);
  // fac score = alpha_{T-1}[L-1] (:203)
  const int lastl = L - 1;
  double vl = 0.0;
#pragma unroll
  for (int k = 0; k < SPL; ++k) vl = (lane * SPL + k == lastl) ? f.v[k] : vl;
  if (lane == lastl / SPL) *lnz = log(vl) + (double)f.ex * 0.6931471805599453;
}

template <int SPL>
__device__ __forceinline__ void fac_beta(const ChainCtx &c, float (*chunk)[kChunk * kStride],
                                         double (*dchunk)[kChunk * kStride],
                                         RowStage<SPL * 32, 32> &st, const int64_t *y, int L,
                                         float *out, int *oute, double *lnz) {
  int gi = 0;
  const int lane = c.lane, T = c.T;
  FacState<SPL> f;
  fac_weights<SPL>(c, y, L, false, f.tok, f.S, f.P);
  const int lastl = L - 1;
#pragma unroll
  for (int k = 0; k < SPL; ++k) f.v[k] = (lane * SPL + k == lastl) ? 1.0 : 0.0;
  f.ex = (lane == lastl / SPL) ? 0 : kNegExp;
  lane_store_hi<SPL>(f.v, f.ex, out, oute, lane, T - 1);
  const int nch = (T + kChunk - 1) / kChunk;
  stage_issue(chunk[(nch - 1) & 1], c, (nch - 1) * kChunk);
  double e0 = 0.0;
  for (int ch = nch - 1; ch >= 0; --ch) {
    const double *buf = dchunk[ch & 1];
    const int t0 = ch * kChunk, rows = min(kChunk, T - t0);
    stage_convert_d(chunk[ch & 1], dchunk[ch & 1], c, rows);
    if (ch > 0) stage_issue(chunk[(ch - 1) & 1], c, t0 - kChunk);
    if (ch > 0 && rows == kChunk) {
#pragma unroll 1
      for (int g = kChunk - kUnroll; g >= 0; g -= kUnroll, ++gi) {
        const int ub = t0 + g;   // frames ub .. ub+7 produce beta' at ub-1 .. ub+6
        const int slot = gi & 1;
        stage_acquire(gi, lane);
#pragma unroll
        for (int q = kUnroll - 1; q >= 0; --q)
          fac_beta_step<SPL>(f, buf + (g + q) * kStride, ((q + kUnroll - 1) % kRenormD) == 0,
                             (q % kRenormD) == 0, st.v[slot], st.e[slot], lane, q);
        stage_release(st, slot, out + (size_t)(ub - 1) * (SPL * 32), oute + (ub - 1) * 32, lane);
      }
    } else {
      for (int r = rows - 1; r >= (ch == 0 ? 1 : 0); --r) {
        const int u = t0 + r;
        fac_beta_step<SPL>(f, buf + r * kStride, ((u - 1) % kRenormD) == 0 || u == 1, true,
                           out, oute, lane, u - 1);
      }
    }
    if (ch == 0) e0 = buf[f.tok[0]];
  }
  stage_drain(lane);
  if (lane == 0) *lnz = log(e0 * f.v[0]) + (double)f.ex * 0.6931471805599453;
}

// One warp per CTA, grid (B, 4 roles): the CTA scheduler spreads the
// serial recursions over the SMs (measured faster than packing several
// recursions per SM, which contend for the load/store path).
template <int SPL>
__global__ void __launch_bounds__(32)
    asg_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     const float *__restrict__ trans, Dims d, AsgFastWs w,
                     const int32_t *__restrict__ status) {
  __shared__ __align__(16) float chunk[2][kChunk * kStride];
  __shared__ __align__(16) double dchunk[2][kChunk * kStride];
  __shared__ __align__(16) float vec[2][32];
  extern __shared__ __align__(128) unsigned char dsm[];  // row staging (dynamic)
  union Stage {
    RowStage<32, 1> fcc;
    RowStage<SPL * 32, 32> fac;
  };
  Stage &st = *reinterpret_cast<Stage *>(dsm);
  const int b = blockIdx.x, role = blockIdx.y;
  if (status[b] != W2L_OK) return;
  ChainCtx c;
  c.trans = trans;
  c.e = em + (size_t)b * d.Tmax * d.N;
  c.N = d.N;
  c.T = em_len[b];
  c.lane = threadIdx.x & 31;
  c.amax = trans_max(trans, d.N);
  const size_t row0 = (size_t)b * d.Tmax;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  if (role == 0) {
    fcc_alpha(c, chunk, vec, st.fcc, w.fcc_a + row0 * 32, w.fcc_ka + (size_t)b * w.tpad,
              w.scal + b * 4 + 0);
  } else if (role == 1) {
    fcc_beta(c, chunk, vec, st.fcc, w.fcc_b + row0 * 32, w.fcc_kb + (size_t)b * w.tpad + 1,
             w.scal + b * 4 + 1);
  } else if (role == 2) {
    fac_alpha<SPL>(c, chunk, dchunk, st.fac, y, tgt_len[b], w.fac_a + row0 * (SPL * 32),
                   w.fac_ea + row0 * 32, w.scal + b * 4 + 2);
  } else {
    fac_beta<SPL>(c, chunk, dchunk, st.fac, y, tgt_len[b], w.fac_b + row0 * (SPL * 32),
                  w.fac_eb + row0 * 32, w.scal + b * 4 + 3);
  }
}

// ----------------------------------------------------------- grad kernel --
template <int SPL>
__global__ void __launch_bounds__(kGradWarps * 32)
    asg_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    const float *__restrict__ trans, Dims d, AsgFastWs w,
                    float *__restrict__ grad_em, const int32_t *__restrict__ status) {
  constexpr int LP = SPL * 32;
  extern __shared__ __align__(16) float gsm[];
  float *red = gsm;                              // [kGradWarps][32*32] fullA partials
  float *redE = red + kGradWarps * 1024;         // [kGradWarps][2][LP] edge partials
  float *prow = redE + kGradWarps * 2 * LP;      // [kGradWarps][LP] posterior row
  float *erow = prow + kGradWarps * LP;          // [kGradWarps][64] Et row (+ zero col)
  float *vrow = erow + kGradWarps * 64;          // [kGradWarps][32] alpha_{t-1} fcc row
  float *gwarp = vrow + kGradWarps * 32;         // [kGradWarps][4] guard

  const int b = blockIdx.y, blk = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N;
  const int T = em_len[b];
  const int t0 = blk * kGradFramesPerBlock;
  const bool ok = status[b] == W2L_OK;
  float *ge = grad_em + (size_t)b * d.Tmax * N;
  const int fpw = kGradFramesPerBlock / kGradWarps;
  const int ta = t0 + warp * fpw, tb = min(ta + fpw, d.Tmax);

  // rows outside the utterance (or a failed utterance) get zero gradient
  for (int t = ta; t < tb; ++t)
    if (!ok || t >= T)
      if (lane < N) ge[(size_t)t * N + lane] = 0.f;
  if (!ok) return;
  if (t0 >= T) {
    // keep the partial buffers well-defined for the final reduction
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
      w.part_fullA[((size_t)b * w.nblk + blk) * 1024 + i] = 0.f;
    for (int i = threadIdx.x; i < 2 * LP; i += blockDim.x)
      w.part_edge[((size_t)b * w.nblk + blk) * 2 * LP + i] = 0.f;
    if (threadIdx.x < 4)
      w.part_guard[((size_t)b * w.nblk + blk) * 4 + threadIdx.x] =
          (threadIdx.x & 1) ? -CUDART_INF_F : CUDART_INF_F;
    return;
  }

  const int L = tgt_len[b];
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  const float amax = trans_max(trans, N);
  int tok[SPL];
  float S[SPL], P[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    const int l = lane * SPL + k;
    if (l < L) {
      const int yl = (int)y[l];
      tok[k] = yl;
      S[k] = expf(trans[yl * N + yl] - amax);
      P[k] = l > 0 ? expf(trans[yl * N + (int)y[l - 1]] - amax) : 0.f;
    } else {
      tok[k] = N;
      S[k] = 0.f;
      P[k] = 0.f;
    }
  }
  // token CSR of this utterance, staged once per block (the gather reads it
  // every frame)
  int *sperm = reinterpret_cast<int *>(gwarp + kGradWarps * 4);
  for (int i = threadIdx.x; i < L; i += blockDim.x) sperm[i] = w.perm[(size_t)b * w.lpad + i];
  __syncthreads();
  const int ts0 = lane < N ? w.tok_start[b * 33 + lane] : 0;
  const int ts1 = lane < N ? w.tok_start[b * 33 + lane + 1] : 0;

  float accA[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) accA[j] = 0.f;
  float accS[SPL], accP[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) accS[k] = accP[k] = 0.f;
  // guard: deviation (log2 units) of every frame's normaliser from the
  // forward totals the chain kernel produced
  const double refF = w.scal[b * 4 + 0] * 1.4426950408889634;
  const double refC = w.scal[b * 4 + 2] * 1.4426950408889634;
  float gminF = CUDART_INF_F, gmaxF = -CUDART_INF_F, gminC = CUDART_INF_F,
        gmaxC = -CUDART_INF_F;

  float *myp = prow + warp * LP;
  float *mye = erow + warp * 64;
  float *myv = vrow + warp * 32;
  const size_t row0 = (size_t)b * d.Tmax;
  const int *ka_row = w.fcc_ka + (size_t)b * w.tpad;
  const int *kb_row = w.fcc_kb + (size_t)b * w.tpad + 1;
  const int tend = min(tb, T);

  // one frame's inputs; the next frame's are loaded while this one is used
  struct Frame {   // fac rows hold the high words of fp64 values (lane64.cuh)
    float e, fa, fb, va[SPL], vb[SPL];
    int ka, kb, ea, eb;
  };
  auto load = [&](Frame &f, int t) {
    f.e = lane < N ? em[(row0 + t) * N + lane] : -CUDART_INF_F;
    f.fa = w.fcc_a[(row0 + t) * 32 + lane];
    f.fb = w.fcc_b[(row0 + t) * 32 + lane];
    f.ka = ka_row[t];
    f.kb = kb_row[t];
    lane_load<SPL>(f.va, w.fac_a + (row0 + t) * LP, lane);
    lane_load<SPL>(f.vb, w.fac_b + (row0 + t) * LP, lane);
    f.ea = w.fac_ea[(row0 + t) * 32 + lane];
    f.eb = w.fac_eb[(row0 + t) * 32 + lane];
  };

  // fac alpha at t-1 (high words and lane exponent) carried across frames
  int pa[SPL];
  int pea = kNegExp;
  float pfa = 0.f;  // fcc alpha_{t-1}[lane]
  int pka = 0;
  if (ta >= 1 && ta < tend) {
    lane_load_int<SPL>(pa, w.fac_a + (row0 + ta - 1) * LP, lane);
    pea = w.fac_ea[(row0 + ta - 1) * 32 + lane];
    pfa = w.fcc_a[(row0 + ta - 1) * 32 + lane];
    pka = ka_row[ta - 1];
  }
  Frame cur, nxt;
  if (ta < tend) load(cur, ta);

  for (int t = ta; t < tend; ++t) {
    if (t + 1 < tend) load(nxt, t + 1);
    // ---- emissions of frame t, shifted and exponentiated (same as the chain)
    const float m = warp_max(cur.e);
    const float et = lane < N ? expf(cur.e - m) : 0.f;
    mye[lane] = et;
    if (lane == 0) mye[32] = 0.f;
    // ---- fcc node posteriors (:238)
    const float gam = cur.fa * cur.fb;
    const float zf = warp_sum(gam);
    const float inv_zf = 1.f / zf;
    const float gF = (float)((double)__log2f(zf) + (double)(cur.ka + cur.kb) - refF);
    gminF = fminf(gminF, gF);
    gmaxF = fmaxf(gmaxF, gF);
    const float full_e = gam * inv_zf;
    // ---- fcc edge posteriors (:240-241): u_t[i] alpha_{t-1}[j], times M later
    if (t >= 1) {
      myv[lane] = pfa;
      __syncwarp();
      const float u = et * cur.fb * pow2f(pka - cur.ka) * inv_zf;
      const float4 *pv = reinterpret_cast<const float4 *>(myv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x = pv[q];
        accA[4 * q] = fmaf(u, x.x, accA[4 * q]);
        accA[4 * q + 1] = fmaf(u, x.y, accA[4 * q + 1]);
        accA[4 * q + 2] = fmaf(u, x.z, accA[4 * q + 2]);
        accA[4 * q + 3] = fmaf(u, x.w, accA[4 * q + 3]);
      }
    }
    // ---- fac node posteriors (:214-217) from the fp64 high words (lane64.cuh);
    // the frame reference exponent comes from the actual magnitudes
    int vah[SPL], vbh[SPL];
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      vah[k] = __float_as_int(cur.va[k]);
      vbh[k] = __float_as_int(cur.vb[k]);
    }
    double pd[SPL];
    const int es = lane_products<SPL>(vah, vbh, cur.ea, cur.eb, pd);
    const int estar = warp_max(es);
    const double sc = pow2d_fast(max(cur.ea + cur.eb - estar, -1100));
    float zl = 0.f;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const float p = (float)(pd[k] * sc);
      myp[lane * SPL + k] = p;
      zl += p;
    }
    const float zc = warp_sum(zl);
    const float inv_zc = 1.f / zc;
    const float gC = (float)((double)__log2f(zc) + (double)estar - refC);
    gminC = fminf(gminC, gC);
    gmaxC = fmaxf(gmaxC, gC);
    __syncwarp();
    // token gather: lane k sums the posteriors of the states labelled k
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    int q = ts0;
    for (; q + 4 <= ts1; q += 4) {
      c0 += myp[sperm[q]];
      c1 += myp[sperm[q + 1]];
      c2 += myp[sperm[q + 2]];
      c3 += myp[sperm[q + 3]];
    }
    for (; q < ts1; ++q) c0 += myp[sperm[q]];
    const float con = (c0 + c1) + (c2 + c3);
    if (lane < N) ge[(size_t)t * N + lane] = full_e - con * inv_zc;
    // ---- fac edge posteriors (:218-224).  The lane scale 2^d is bounded by
    // 2^127 and the mantissa products are tiny whenever d is large (a
    // posterior is <= 1), so x * 2^d * (1/Z) cannot overflow.
    if (t >= 1) {
      // stay/step edge posteriors: (alpha_{t-1} beta'_t) products in fp64 scaled
      // to the frame reference, then the float weights S|P * Et
      const int nbh = __shfl_up_sync(0xffffffffu, pa[SPL - 1], 1);
      const int nbe = __shfl_up_sync(0xffffffffu, pea, 1);
      const double s_own = pow2d_fast(max(pea + cur.eb - estar, -1100));
      const double s_nb = lane > 0 ? pow2d_fast(max(nbe + cur.eb - estar, -1100)) : 0.0;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const double bk = hi_to_d(vbh[k]);
        const float ek = mye[tok[k]] * inv_zc;
        const float stay = (float)(hi_to_d(pa[k]) * bk * s_own);
        const float prev = k > 0 ? (float)(hi_to_d(pa[k - 1]) * bk * s_own)
                                 : (float)(hi_to_d(nbh) * bk * s_nb);
        accS[k] = fmaf(stay * S[k], ek, accS[k]);
        accP[k] = fmaf(prev * P[k], ek, accP[k]);
      }
    }
    // carry alpha_t as alpha_{t-1} for the next frame
#pragma unroll
    for (int k = 0; k < SPL; ++k) pa[k] = vah[k];
    pea = cur.ea;
    pfa = cur.fa;
    pka = cur.ka;
    cur = nxt;
    __syncwarp();
  }

  // ---- block reduction of the partials in fixed warp order (deterministic)
  float *rA = red + warp * 1024;
#pragma unroll
  for (int j = 0; j < 32; ++j) rA[lane * 32 + j] = accA[j];
  float *rE = redE + warp * 2 * LP;
#pragma unroll
  for (int k = 0; k < SPL; ++k) {
    rE[lane * SPL + k] = accS[k];
    rE[LP + lane * SPL + k] = accP[k];
  }
  if (lane == 0) {
    gwarp[warp * 4 + 0] = gminF;
    gwarp[warp * 4 + 1] = gmaxF;
    gwarp[warp * 4 + 2] = gminC;
    gwarp[warp * 4 + 3] = gmaxC;
  }
  __syncthreads();
  float *dstA = w.part_fullA + ((size_t)b * w.nblk + blk) * 1024;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < kGradWarps; ++q) s += red[q * 1024 + i];
    dstA[i] = s;
  }
  float *dstE = w.part_edge + ((size_t)b * w.nblk + blk) * 2 * LP;
  for (int i = threadIdx.x; i < 2 * LP; i += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < kGradWarps; ++q) s += redE[q * 2 * LP + i];
    dstE[i] = s;
  }
  if (threadIdx.x < 4) {
    float g = (threadIdx.x & 1) ? -CUDART_INF_F : CUDART_INF_F;
    for (int q = 0; q < kGradWarps; ++q) {
      const float v = gwarp[q * 4 + threadIdx.x];
      g = (threadIdx.x & 1) ? fmaxf(g, v) : fminf(g, v);
    }
    w.part_guard[((size_t)b * w.nblk + blk) * 4 + threadIdx.x] = g;
  }
}

// ---------------------------------------------------------- final kernel --
// per utterance: dA_b = M (.) sum_blocks(fullA partials) - scatter(fac edge
// sums) (criterion.py:239-246), the loss (:244) and the guard verdict.
__global__ void __launch_bounds__(1024)
    asg_final_kernel(const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     const int32_t *__restrict__ em_len, const float *__restrict__ trans, Dims d,
                     AsgFastWs w, double *loss, float *ga_utt, int32_t *status) {
  const int b = blockIdx.x;
  __shared__ float sEdge[2 * 1024];
  __shared__ float sA[1024];
  __shared__ float s_red[32];
  __shared__ int s_bad;
  const int N = d.N, NN = N * N;
  if (status[b] != W2L_OK) {
    for (int p = threadIdx.x; p < NN; p += blockDim.x) ga_utt[(size_t)b * NN + p] = 0.f;
    return;
  }
  const int L = tgt_len[b], T = em_len[b], LP = w.lpad;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float am = -CUDART_INF_F;
  for (int p = threadIdx.x; p < NN; p += blockDim.x) am = fmaxf(am, trans[p]);
  am = warp_max(am);
  if (lane == 0) s_red[warp] = am;
  if (threadIdx.x == 0) s_bad = 0;
  // fixed-order sums of the per-frame-block partials; 4 independent
  // accumulators keep several loads in flight per thread
  const int nb_used = (T + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  auto sum_parts = [&](const float *base, size_t stride) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int q = 0;
    for (; q + 4 <= nb_used; q += 4) {
      a0 += base[(size_t)q * stride];
      a1 += base[(size_t)(q + 1) * stride];
      a2 += base[(size_t)(q + 2) * stride];
      a3 += base[(size_t)(q + 3) * stride];
    }
    for (; q < nb_used; ++q) a0 += base[(size_t)q * stride];
    return (a0 + a1) + (a2 + a3);
  };
  for (int i = threadIdx.x; i < 2 * LP; i += blockDim.x)
    sEdge[i] = sum_parts(w.part_edge + (size_t)b * w.nblk * 2 * LP + i, 2 * LP);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    sA[i] = sum_parts(w.part_fullA + (size_t)b * w.nblk * 1024 + i, 1024);
  __syncthreads();
  float amax = s_red[0];
  for (int q = 1; q < (int)(blockDim.x >> 5); ++q) amax = fmaxf(amax, s_red[q]);
  const int *perm = w.perm + (size_t)b * w.lpad;
  const int *ts = w.tok_start + b * 33;
  for (int p = threadIdx.x; p < NN; p += blockDim.x) {
    const int i = p / N, j = p % N;
    const float full = sA[i * 32 + j] * expf(trans[p] - amax);
    float con = 0.f;  // states labelled i: stay edges (i,i), step edges (i, y_{l-1})
    for (int q = ts[i]; q < ts[i + 1]; ++q) {
      const int l = perm[q];
      if (i == j) con += sEdge[l];
      if (l > 0 && (int)y[l - 1] == j) con += sEdge[LP + l];
    }
    ga_utt[(size_t)b * NN + p] = full - con;
    if (!isfinite(full - con)) atomicOr(&s_bad, 1);
  }
  // guard: every frame's normaliser must reproduce the forward totals
  const double ln2 = 0.6931471805599453;
  const double zF = w.scal[b * 4 + 0], zFb = w.scal[b * 4 + 1];
  const double zC = w.scal[b * 4 + 2], zCb = w.scal[b * 4 + 3];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)T / 1600.0));
  int bad = !(isfinite(zF) && isfinite(zFb) && isfinite(zC) && isfinite(zCb));
  bad |= fabs(zF - zFb) > tol || fabs(zC - zCb) > tol;
  for (int q = threadIdx.x; q < nb_used; q += blockDim.x) {
    const float *g = w.part_guard + ((size_t)b * w.nblk + q) * 4;
    bad |= !(fabs((double)g[0]) * ln2 <= tol && fabs((double)g[1]) * ln2 <= tol);
    bad |= !(fabs((double)g[2]) * ln2 <= tol && fabs((double)g[3]) * ln2 <= tol);
  }
  (void)L;
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    loss[b] = zF - zC;
    if (s_bad) status[b] = kNeedsExact;
  }
}

template <int SPL>
cudaError_t launch_spl(const float *em, const int32_t *em_len, const int64_t *tgt,
                       const int32_t *tgt_len, const float *trans, Dims d, const AsgFastWs &w,
                       float *grad_em, const int32_t *status, cudaStream_t s, Tracer *tr) {
  const size_t stage_bytes = sizeof(RowStage<SPL * 32, 32>);
  auto kc = asg_chain_kernel<SPL>;
  cudaError_t err0 =
      cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_bytes);
  if (err0 != cudaSuccess) return err0;
  kc<<<dim3(d.B, 4), 32, stage_bytes, s>>>(em, em_len, tgt, tgt_len, trans, d, w, status);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  trace(tr, s);  // chain
  constexpr int LP = SPL * 32;
  const size_t smem = sizeof(float) * (kGradWarps * (1024 + 2 * LP + LP + 64 + 32 + 4) + LP);
  auto k = asg_grad_kernel<SPL>;
  err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  k<<<dim3(w.nblk, d.B), kGradWarps * 32, smem, s>>>(em, em_len, tgt, tgt_len, trans, d, w,
                                                      grad_em, status);
  return cudaGetLastError();
}

}  // namespace

int asg_fast_spl(int Lmax) {
  static const int opts[] = {2, 4, 8, 10, 12, 16, 20, 24, 32};
  for (int o : opts)
    if (32 * o >= Lmax) return o;
  return 0;
}

static size_t asg_ws_layout(Dims d, void *base, AsgFastWs *w) {
  const int spl = asg_fast_spl(d.Lmax);
  const int lpad = spl * 32;
  const int nblk = (d.Tmax + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  const size_t BT = (size_t)d.B * d.Tmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? (void *)((char *)base + o) : nullptr;
  };
  AsgFastWs t;
  t.fcc_a = (float *)take(BT * 32 * 4);
  t.fcc_b = (float *)take(BT * 32 * 4);
  const int tpad = round_up(d.Tmax + 1, 8);
  t.fcc_ka = (int *)take((size_t)d.B * tpad * 4);
  t.fcc_kb = (int *)take((size_t)d.B * tpad * 4);
  t.fac_a = (float *)take(BT * lpad * 4);
  t.fac_b = (float *)take(BT * lpad * 4);
  t.fac_ea = (int *)take(BT * 32 * 4);
  t.fac_eb = (int *)take(BT * 32 * 4);
  t.scal = (double *)take((size_t)d.B * 4 * 8);
  t.part_fullA = (float *)take((size_t)d.B * nblk * 1024 * 4);
  t.part_edge = (float *)take((size_t)d.B * nblk * 2 * lpad * 4);
  t.part_guard = (float *)take((size_t)d.B * nblk * 4 * 4);
  t.perm = (int *)take((size_t)d.B * lpad * 4);
  t.tok_start = (int *)take((size_t)d.B * 33 * 4);
  t.spl = spl;
  t.lpad = lpad;
  t.nblk = nblk;
  t.tpad = tpad;
  if (w) *w = t;
  return off;
}

size_t asg_fast_ws_bytes(Dims d) { return asg_ws_layout(d, nullptr, nullptr); }
void asg_fast_ws_carve(Dims d, void *ws, AsgFastWs *w) { asg_ws_layout(d, ws, w); }

cudaError_t launch_asg_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, const float *trans, Dims d,
                            const AsgFastWs &w, double *loss, float *grad_em, float *ga_utt,
                            int32_t *status, cudaStream_t s, Tracer *tr) {
  cudaError_t err = cudaSuccess;
  switch (w.spl) {
    case 2: err = launch_spl<2>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 4: err = launch_spl<4>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 8: err = launch_spl<8>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 10: err = launch_spl<10>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 12: err = launch_spl<12>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 16: err = launch_spl<16>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 20: err = launch_spl<20>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 24: err = launch_spl<24>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    case 32: err = launch_spl<32>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, s, tr); break;
    default: return cudaErrorInvalidValue;
  }
  if (err != cudaSuccess) return err;
  trace(tr, s);  // grad
  asg_final_kernel<<<d.B, 1024, 0, s>>>(tgt, tgt_len, em_len, trans, d, w, loss, ga_utt, status);
  err = cudaGetLastError();
  trace(tr, s);  // final
  return err;
}

// --------------------------------------------------- batch reduction of dA --
// one warp per transition pair: fixed-order float64 sum over utterances
// (trainer.py:442-447 sums in float64), deterministic run to run
__global__ void reduce_grad_trans_kernel(const float *ga_utt, const int32_t *status, Dims d,
                                         float *grad_trans) {
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= d.N * d.N) return;
  double s = 0.0;
  for (int b = lane; b < d.B; b += 32)
    if (status[b] == W2L_OK) s += (double)ga_utt[(size_t)b * d.N * d.N + p];
  s = warp_sum(s);
  if (lane == 0) grad_trans[p] = (float)s;
}

cudaError_t launch_reduce_grad_trans(const float *ga_utt, const int32_t *status, Dims d,
                                     float *grad_trans, cudaStream_t s) {
  const int n = d.N * d.N;
  reduce_grad_trans_kernel<<<(n + 7) / 8, 256, 0, s>>>(ga_utt, status, d, grad_trans);
  return cudaGetLastError();
}

}  // namespace w2l
