// Batched ASG loss + gradient (replaces criterion.py:167-247 for the batched
// hot path), in two precision tiers of one algorithm.
//
// Algorithm: the four ASG recursions are run in the SCALED LINEAR domain,
// the standard exact reformulation of log-space forward-backward
//     alpha_t = Et (.) (M alpha_{t-1}) * 2^-k_t ,   M = exp(A - max A),
//     Et[i]   = exp(e[t][i] - max_i e[t][i]),
// with exact power-of-two rescaling (only integer exponents accumulate, no
// rounding in the scale factors).  The fcc (fully connected, N x N) graph is
// a 32-lane mat-vec per frame with the previous vector broadcast through
// shared memory; the fac (forced alignment, L-state chain) graph is a
// multi-warp wavefront lattice (lattice.cuh): 4 states per lane with one
// power-of-two exponent per lane.  No transcendental sits on the recursion's
// critical path.  V (the lane type) is float for the fast tier and double
// for the wide-range tier that takes the utterances failing the fp32 guard.
//
// Kernels (one stream, in order):
//   asg_chain    grid (B, 2 directions), one CTA per (utterance, direction):
//                producer warp (Et ring), fcc warp, W fac lattice warps;
//                rows of alpha/beta and exponents to the workspace.
//   asg_grad     two CTA bodies in one launch, 128 frames each:
//                fac   per-frame fac posteriors (normaliser Z_t), the whole
//                      gradient row (fcc node posteriors minus the fac node
//                      posteriors gathered by token), state occupancies and
//                      the fac guard;
//                fcc   fcc edge outer products and the fcc guard.
//   asg_final    per utterance: loss, grad_A_b, guard verdict -> OK, or the
//                next tier.
// Reference correspondence: fac alpha/beta = criterion.py:193-212, fac
// posteriors = :214-224, fcc = :227-241, combine = :243-247.

#include <algorithm>

#include "band.cuh"
#include "laneblock.cuh"
#include "lattice.cuh"
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

#ifndef W2L_ASG_GRAD_FRAMES
#define W2L_ASG_GRAD_FRAMES 128
#endif
constexpr int kGradFramesPerBlock = W2L_ASG_GRAD_FRAMES;   // frames per gradient CTA (both bodies)
constexpr int kFccFrames = kGradFramesPerBlock;
constexpr int kGradWarps = 8;
// asg_final: one CTA per utterance (launched as a programmatic dependent
// during the gradient grid's last wave, it stages its inputs before the
// gradient completes); 512 threads, each with the partials of up to 4
// entries in flight (kFinalChunk frame blocks each): ASG alone 0.327 ->
// 0.321 ms.  16 blocks per entry (111 registers) was no better in the
// two-criteria step, where the early-launched CTAs hold their registers.
constexpr int kFinalThreads = 512;
#ifndef W2L_FINAL_CHUNK
#define W2L_FINAL_CHUNK 4
#endif
constexpr int kFinalChunk = W2L_FINAL_CHUNK;   // frame-block partials in flight per entry
constexpr int kFinalEnt =   // entries (L occupancies + N^2 edge sums) per thread
    (W2L_MAX_ASG_LABELS + W2L_MAX_TOKENS * W2L_MAX_TOKENS + kFinalThreads - 1) / kFinalThreads;

__device__ __forceinline__ float trans_max(const float *trans, int N) {
  float m = -CUDART_INF_F;
  for (int p = threadIdx.x & 31; p < N * N; p += 32) m = fmaxf(m, trans[p]);
  return warp_max(m);
}

// ---------------------------------------------------------- fcc steps --
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
    const int Kt = seen >= 2 ? X2 + (X2 - X3) : (seen == 1 ? X2 : K1);
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

// packed fp32x2 arithmetic (FFMA2): two lanes of a 64-bit register
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ unsigned long long f2_dup(float x) { return f2_pack(x, x); }
__device__ __forceinline__ float f2_lo(unsigned long long x) { return __uint_as_float((unsigned)x); }
__device__ __forceinline__ float f2_hi(unsigned long long x) {
  return __uint_as_float((unsigned)(x >> 32));
}

// m: the lane's row of M (alpha) or column (beta); vin: the 32-vector (16B
// aligned); 8 independent accumulators of depth 4 (scalar FMA measured
// faster than FFMA2 on this latency-bound chain).  SUM: also return the
// exponent of the vector's sum (lane N's row of ones, or a direct sum).
template <bool SUM, class V>
__device__ __forceinline__ V fcc_matvec(const V (&m)[32], const V *vin, bool spare, int N,
                                        int &e_sum) {
  V acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    V x[4];
    ld4(vin + 4 * q, x);
    acc[q] = m[4 * q] * x[0];
    acc[q] = fma(m[4 * q + 1], x[1], acc[q]);
    acc[q] = fma(m[4 * q + 2], x[2], acc[q]);
    acc[q] = fma(m[4 * q + 3], x[3], acc[q]);
  }
  const V s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  if (SUM) {
    if (spare) {
      e_sum = Pow2<V>::expo(__shfl_sync(0xffffffffu, s, N));   // lane N: row of ones
    } else {
      V tot = (V)0;
#pragma unroll
      for (int q = 0; q < 32; ++q) tot += vin[q];
      e_sum = Pow2<V>::expo(tot);
    }
  }
  return s;
}

template <class V>
struct FccState {
  V m[32];
  V v;           // this lane's current alpha_t / beta'_t
  int K;
  int knext;     // scale exponent of the next step (chosen one step ahead)
  LaggedScale sc;
  bool spare;
};

// The power-of-two rescaling runs on every kFccRescale-th step only (RS):
// between rescales the vector's magnitude moves by at most a few steps of
// growth, far inside the type's range.  The scale bookkeeping (the sum's
// exponent arrives through a shuffle) runs after the step's vector is stored,
// so the next step's mat-vec does not wait behind it.
constexpr int kFccRescale = 4;

// fcc alpha step t (criterion.py:230): alpha_t = Et (.) (M alpha_{t-1}) 2^-k
template <bool RS, class V>
__device__ __forceinline__ void fcc_alpha_step(FccState<V> &f, V et, V (*vec)[32], int par,
                                               V *out_row, int *outk_t, int lane, int N) {
  const int k = RS ? f.knext : 0;
  const V sc = RS ? et * Pow2<V>::p2(-k) : et;   // |k| <= 120: exact
  __syncwarp();
  int e1 = 0;
  const V s = fcc_matvec<RS, V>(f.m, vec[par ^ 1], f.spare, N, e1);
  f.K += k;
  f.v = s * sc;
  vec[par][lane] = f.v;
#ifndef W2L_NO_ROW_STORES
  out_row[lane] = f.v;
#endif
  if (lane == 0) *outk_t = f.K;
  if (RS) {
    f.sc.observe(e1);
    f.knext = f.sc.next();
  }
}

// fcc beta' step consuming frame u (criterion.py:236): beta'_{u-1} = M^T (Et_u beta'_u) 2^-k
template <bool RS, class V>
__device__ __forceinline__ void fcc_beta_step(FccState<V> &f, V et, V (*vec)[32], int par,
                                              V *out_row, int *outk_t, int lane, int N) {
  const int k = RS ? f.knext : 0;
  const V sc = lane < N ? (RS ? Pow2<V>::p2(-k) : (V)1) : (V)0;
  vec[par][lane] = et * f.v;
  __syncwarp();
  int e1 = 0;
  const V s = fcc_matvec<RS, V>(f.m, vec[par], f.spare, N, e1);
  f.K += k;
  f.v = s * sc;
#ifndef W2L_NO_ROW_STORES
  out_row[lane] = f.v;
#endif
  if (lane == 0) *outk_t = f.K;
  if (RS) {
    f.sc.observe(e1);
    f.knext = f.sc.next();
  }
}

template <class V>
struct FccCtx {
  const float *trans;
  float amax;
  int N, T, lane, cons_idx;
  V *rows;      // [Tmax][32] this utterance
  int *ks;      // cumulative exponents, indexed by frame
};

// fcc recursion over the shared Et ring (criterion.py:227-236); the same
// step schedule as the lattice warps (lattice.cuh)
template <bool FWD, class V, bool STREAM>
__device__ void fcc_run(ChainSm<V> &sm, const FccCtx<V> &c, double *lnz) {
  constexpr int kRing = Ring<V>::n;
  const int lane = c.lane, N = c.N, T = c.T;
  FccState<V> f;
  f.spare = N < 32;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // forward: row `lane` of M; backward: column `lane`; lane N of a spare
    // lane is a row of ones (its product is the sum of the vector)
    const int p = FWD ? lane * N + j : j * N + lane;
    f.m[j] = (lane < N && j < N) ? Pow2<V>::ex((V)c.trans[p] - (V)c.amax)
                                 : ((f.spare && lane == N && j < N) ? (V)1 : (V)0);
  }
  f.K = 0;
  f.knext = f.sc.next();
  int *mycons = &sm.cons[c.cons_idx];
  if (FWD) {
    wait_ge(&sm.prod, 1);
    f.v = sm.ering[ring_slot<V>(true, 0)][lane];   // alpha_0 = Et_0 (criterion.py:228)
    sm.vec[0][lane] = f.v;
    c.rows[lane] = f.v;
    if (lane == 0) c.ks[0] = 0;
  } else {
    f.v = lane < N ? (V)1 : (V)0;
    c.rows[(size_t)(T - 1) * 32 + lane] = f.v;
    if (lane == 0) c.ks[T - 1] = 0;
  }
  publish(mycons, 1, lane);
  auto generic = [&](int j) {
    wait_ge(&sm.prod, eidx_of(FWD, j) + 1);
    const V et = sm.ering[j & (kRing - 1)][lane];
    const int t = frame_of(FWD, T, j);
    if (FWD)
      fcc_alpha_step<true, V>(f, et, sm.vec, j & 1, c.rows + (size_t)t * 32, c.ks + t, lane, N);
    else
      fcc_beta_step<true, V>(f, et, sm.vec, j & 1, c.rows + (size_t)t * 32, c.ks + t, lane, N);
    publish(mycons, j + 1, lane);
  };
  const int pro_end = min(T, kBlk);
  for (int j = 1; j < pro_end; ++j) generic(j);
  const int nfull = T > kBlk ? (T - kBlk) / kBlk : 0;
  const int mtrig = STREAM ? stream_trigger_block<kFac>(T) : -1;   // (see lattice_run)
#pragma unroll 1
  for (int m = 1; m <= nfull; ++m) {
    const int j0 = m * kBlk;
    if (STREAM && m == mtrig) pdl_launch_dependents();
    wait3(&sm.prod, eidx_of(FWD, j0 + kBlk - 1) + 1, &sm.prod, 0, &sm.prod, 0);
    const V *eb = sm.ering[j0 & (kRing - 1)];
    const int tb = frame_of(FWD, T, j0);
    V *sv = c.rows + (size_t)tb * 32;
    V etq[kBlk];
#pragma unroll
    for (int q = 0; q < kBlk; ++q) etq[q] = eb[q * kStride + lane];
#pragma unroll
    for (int q = 0; q < kBlk; ++q) {
      const int dq = FWD ? q : -q;
      if ((q % kFccRescale) == kFccRescale - 1) {
        if (FWD)
          fcc_alpha_step<true, V>(f, etq[q], sm.vec, q & 1, sv + dq * 32, c.ks + tb + dq, lane, N);
        else
          fcc_beta_step<true, V>(f, etq[q], sm.vec, q & 1, sv + dq * 32, c.ks + tb + dq, lane, N);
      } else {
        if (FWD)
          fcc_alpha_step<false, V>(f, etq[q], sm.vec, q & 1, sv + dq * 32, c.ks + tb + dq, lane,
                                   N);
        else
          fcc_beta_step<false, V>(f, etq[q], sm.vec, q & 1, sv + dq * 32, c.ks + tb + dq, lane,
                                  N);
      }
    }
    publish(mycons, j0 + kBlk, lane);
  }
  for (int j = max(pro_end, (nfull + 1) * kBlk); j < T; ++j) generic(j);
  if (STREAM && mtrig > nfull) pdl_launch_dependents();
  publish(mycons, kDone, lane);
  V z;
  if (FWD) {
    z = warp_sum(lane < N ? f.v : (V)0);
  } else {
    wait_ge(&sm.prod, T);   // frame 0's Et (the last step only waited for T - 1)
    const V e0 = sm.ering[ring_slot<V>(false, T - 1)][lane];   // frame 0
    z = warp_sum(e0 * f.v);
  }
  if (lane == 0) *lnz = log((double)z) + (double)f.K * 0.6931471805599453;
}

template <bool FWD, class V, bool STREAM>
__device__ __forceinline__ void asg_chain_body(ChainSm<V> &sm, const float *em, int T, int L,
                                               const int64_t *y, const float *trans, Dims d,
                                               const AsgFastWs &w, int b, int32_t *status,
                                               int fail) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float amax = trans_max(trans, d.N);
  const int weff = lat_warps(L);
  if (warp == 0) {
    // the fcc uses every token
    ProdCtx pc{em + (size_t)b * d.Tmax * d.N, d.N, T, FWD, 1 + weff, 0,
               d.N >= 32 ? 0xffffffffu : (1u << d.N) - 1u};
    pc.gprog = w.prog ? w.prog + 2 * b + (FWD ? 0 : 1) : nullptr;
    pc.trig = stream_trigger_step<kFac>(T);
    producer_run<V>(sm, pc, lane, nullptr);
  } else if (warp == 1) {
    FccCtx<V> fc;
    fc.trans = trans;
    fc.amax = amax;
    fc.N = d.N;
    fc.T = T;
    fc.lane = lane;
    fc.cons_idx = 0;
    fc.rows = reinterpret_cast<V *>(FWD ? w.fcc_a : w.fcc_b) + (size_t)b * d.Tmax * 32;
    fc.ks = FWD ? w.fcc_ka + (size_t)b * w.tpad : w.fcc_kb + (size_t)b * w.tpad + 1;
    fcc_run<FWD, V, STREAM>(sm, fc, w.scal + b * 4 + (FWD ? 0 : 1));
  } else if (warp - 2 < weff) {
    LatCtx c;
    c.w = warp - 2;
    c.W = weff;
    c.lane = lane;
    c.T = T;
    c.N = d.N;
    c.nstates = L;
    c.cons_idx = 1;
    c.Tmax = d.Tmax;
    const size_t ub = (size_t)b * w.W * d.Tmax;
    c.rows = reinterpret_cast<V *>(FWD ? w.fac_a : w.fac_b) + ub * kLatStates;
    c.exps = (FWD ? w.fac_ea : w.fac_eb) + ub * 32;
    LatState<V> f;
    lat_init_weights<kFac, FWD, V>(f, c.w, lane, d.N, L, y, L, trans, amax, 0);
    lattice_run<kFac, FWD, V, STREAM>(sm, c, f);
  } else if (STREAM) {   // a warp without a role: its share of the trigger, at
    wait_ge(&sm.cons[1], stream_trigger_step<kFac>(T));   // lattice warp 0's midpoint
    pdl_launch_dependents();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    w.scal[b * 4 + (FWD ? 2 : 3)] = lattice_total(sm, weff);
    if (sm.flush) status[b] = fail;
    if (w.prog) st_release_gpu(w.prog + 2 * b + (FWD ? 0 : 1), T);   // last write of the CTA
  }
}

// grid (B, 2): blockIdx.y 0 = forward (alpha), 1 = backward (beta);
// STREAM: publish progress and trigger the streamed gradient (w.prog set)
template <class V, bool STREAM>
__global__ void __launch_bounds__(32 * (2 + kMaxLatWarps))
    asg_chain_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                     const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     const float *__restrict__ trans, Dims d, AsgFastWs w,
                     int32_t *__restrict__ status, int want, int fail) {
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
  const int weff = lat_warps(L);
  if (threadIdx.x == 0) sm.prod = 0, sm.flush = 0;
  // counters: 0 = fcc, 1 + w = lattice warp w (absent warps are done)
  if (threadIdx.x < kCounters) sm.cons[threadIdx.x] = threadIdx.x <= weff ? 0 : kDone;
  __syncthreads();
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  if (blockIdx.y == 0)
    asg_chain_body<true, V, STREAM>(sm, em, T, L, y, trans, d, w, b, status, fail);
  else
    asg_chain_body<false, V, STREAM>(sm, em, T, L, y, trans, d, w, b, status, fail);
  W2L_TL(if (threadIdx.x == 0) tl_rec(3000000ull + b * 10 + blockIdx.y, tl0, gtimer(), smid() | (hw_warpid() << 16)));
}

// ----------------------------------------------------------- grad kernel --
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// Per-warp staging area of the fcc body: the warp's frames' fcc rows (alpha
// including frame ta-1, beta), exponents and emission rows come in with one
// cp.async batch.  Reused for the block reduction.
constexpr int kFccFpw = kFccFrames / kGradWarps;            // 16 frames per warp
constexpr int kRedStride = 33;   // padded row of the fcc body's per-warp [32][32] partial
template <class V>
__host__ __device__ constexpr size_t fcc_stage_bytes() {
  const size_t stage = (((size_t)(kFccFpw + 1) * 32 + (size_t)kFccFpw * 32) * sizeof(V) +
                        (size_t)kFccFpw * 32 * 4 + (size_t)(2 * kFccFpw + 1) * 4 + 15) &
                       ~(size_t)15;
  const size_t red = (32 * kRedStride * sizeof(float) + 15) & ~(size_t)15;
  return stage > red ? stage : red;
}
static_assert(fcc_stage_bytes<float>() >= 32 * kRedStride * sizeof(float),
              "the staging area doubles as the reduction buffer");

// fcc edge posteriors and the fcc guard (the fcc node posteriors are formed
// by the fac body, which writes the whole gradient row)
template <class V>
__device__ __forceinline__ void asg_fcc_grad_body(const float *__restrict__ em,
                                                  const int32_t *__restrict__ em_len, Dims d,
                                                  const AsgFastWs &w, int ust, int want, int b,
                                                  int blk, unsigned char *smem) {
  __shared__ double gwarp[kGradWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N;
  const int T = em_len[b];
  const int t0 = blk * kFccFrames;
  if (ust != want || t0 >= T) return;
  const int ta = t0 + warp * kFccFpw, tb = min(ta + kFccFpw, d.Tmax);
  double gmin = CUDART_INF, gmax = -CUDART_INF;
  const int tend = min(tb, T);

  // ---- stage this warp's frames: row r of sfa/ska is frame ta-1+r, row r of
  // sfb/skb/se is frame ta+r
  unsigned char *st = smem + warp * fcc_stage_bytes<V>();
  V *sfa = reinterpret_cast<V *>(st);                // [kFccFpw+1][32]
  V *sfb = sfa + (kFccFpw + 1) * 32;                 // [kFccFpw][32]
  float *se = reinterpret_cast<float *>(sfb + kFccFpw * 32);   // [kFccFpw][N] (flat)
  int *ska = reinterpret_cast<int *>(se + kFccFpw * 32);       // [kFccFpw+1]
  int *skb = ska + kFccFpw + 1;                      // [kFccFpw]
  constexpr int kRowChunks = 32 * sizeof(V) / 16;    // 16-byte chunks per row
  if (ta < tend) {
    const int f0 = max(ta - 1, 0), nf = tend - ta;
    const V *fa_g = reinterpret_cast<const V *>(w.fcc_a) + (size_t)b * d.Tmax * 32;
    const V *fb_g = reinterpret_cast<const V *>(w.fcc_b) + (size_t)b * d.Tmax * 32;
    const int nfa = (tend - f0) * kRowChunks;
    V *dfa = sfa + (f0 - (ta - 1)) * 32;
    for (int i = lane; i < nfa; i += 32)
      cp_async16(reinterpret_cast<char *>(dfa) + 16 * i,
                 reinterpret_cast<const char *>(fa_g + (size_t)f0 * 32) + 16 * i);
    for (int i = lane; i < nf * kRowChunks; i += 32)
      cp_async16(reinterpret_cast<char *>(sfb) + 16 * i,
                 reinterpret_cast<const char *>(fb_g + (size_t)ta * 32) + 16 * i);
    const float *e_g = em + ((size_t)b * d.Tmax + ta) * N;
    for (int i = lane; i < nf * N; i += 32) cp_async4(se + i, e_g + i);
    const int *ka_g = w.fcc_ka + (size_t)b * w.tpad;
    const int *kb_g = w.fcc_kb + (size_t)b * w.tpad + 1;
    // (L2 loads: these words share cache lines with frames a concurrently
    // running chain may not have written yet)
    if (lane < tend - f0) ska[(f0 - (ta - 1)) + lane] = __ldcg(ka_g + f0 + lane);
    if (lane < nf) skb[lane] = __ldcg(kb_g + ta + lane);
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncwarp();

  // edge accumulators: acc[lane][j] = sum_t u_t[lane] alpha_{t-1}[j]
  unsigned long long accA[16];   // float: (row lane, columns 2jj, 2jj+1) packed
  double accD[sizeof(V) == 8 ? 32 : 1];
#pragma unroll
  for (int j = 0; j < 16; ++j) accA[j] = 0ull;
#pragma unroll
  for (int j = 0; j < (int)(sizeof(accD) / sizeof(double)); ++j) accD[j] = 0.0;
#pragma unroll 2
  for (int t = ta; t < tend; ++t) {
    const int r = t - ta;
    const float e = lane < N ? se[r * N + lane] : -CUDART_INF_F;
    const V fa = sfa[(r + 1) * 32 + lane], fb = sfb[r * 32 + lane];
    const int ka = ska[r + 1], kb = skb[r];
    const float m = warp_max(e);
    const V et = lane < N ? et_of<V>(e, m) : (V)0;
    // the frame's fcc normaliser (the node posteriors themselves, :238, are
    // formed in the fac body)
    const V zf = warp_sum(fa * fb);
    const V izf = (V)1 / zf;
    float lz;
    if constexpr (sizeof(V) == 4) lz = __log2f(zf);
    else lz = (float)log2(zf);
    // the frame's log2-normaliser
    const double g = (double)lz + (double)(ka + kb);
    gmin = fmin(gmin, g);
    gmax = fmax(gmax, g);
    if (t >= 1) {
      // fcc edge posteriors (:240-241): u_t[i] alpha_{t-1}[j] (times M later)
      const V u = et * fb * Pow2<V>::p2(ska[r] - ka) * izf;
      if constexpr (sizeof(V) == 4) {
        const unsigned long long u2 = f2_dup((float)u);
        const ulonglong2 *pv = reinterpret_cast<const ulonglong2 *>(sfa + r * 32);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          const ulonglong2 x = pv[qq];
          accA[2 * qq] = ffma2(u2, x.x, accA[2 * qq]);
          accA[2 * qq + 1] = ffma2(u2, x.y, accA[2 * qq + 1]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) accD[j] = fma((double)u, (double)sfa[r * 32 + j], accD[j]);
      }
    }
  }
  __syncwarp();
  // this warp's partial [32][32], rows padded to kRedStride floats so that the
  // 32 lanes' stores of one column hit 32 different banks (an unpadded row of
  // 32 floats put every lane on the same bank)
  float *red = reinterpret_cast<float *>(st);
  if constexpr (sizeof(V) == 4) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      red[lane * kRedStride + 2 * j] = f2_lo(accA[j]);
      red[lane * kRedStride + 2 * j + 1] = f2_hi(accA[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) red[lane * kRedStride + j] = (float)accD[j];
  }
  if (lane == 0) {
    gwarp[warp][0] = gmin;
    gwarp[warp][1] = gmax;
  }
  __syncthreads();
  float *dstA = w.part_fullA + ((size_t)b * w.nblk + blk) * 1024;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    float s = 0.f;
    const int ri = (i >> 5) * kRedStride + (i & 31);
    for (int q = 0; q < kGradWarps; ++q)
      s += reinterpret_cast<const float *>(smem + q * fcc_stage_bytes<V>())[ri];
    dstA[i] = s;
  }
  if (threadIdx.x < 2) {
    double g = threadIdx.x ? -CUDART_INF : CUDART_INF;
    for (int q = 0; q < kGradWarps; ++q)
      g = threadIdx.x ? fmax(g, gwarp[q][1]) : fmin(g, gwarp[q][0]);
    w.part_guard[((size_t)b * w.nblk + blk) * 4 + threadIdx.x] = g;
  }
}

// one shared-memory float at an absolute shared-window address
__device__ __forceinline__ float lds_f32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
template <int W>
constexpr size_t fac_grad_smem() {
  // per warp: posterior row + occupancy row (floats), guard (2 doubles),
  // token bins, a band word; the CTA's lane-block tokens, 2 band words
  return sizeof(float) * (kGradWarps * (2 * (size_t)W * kLatStates + 4 + 32 + 1) +
                          (size_t)W * kLatStates / 4 + 2);
}

// The whole gradient row: fcc node posteriors (full part, :238) minus the
// fac node posteriors gathered by token (:214-217), plus the fac occupancy.
// A warp walks consecutive frames with the band-limited reads of band.cuh
// (fac posterior mass moves by 0 or 1 state per frame).
//
// Fac edge sums need no edge products: a forced alignment enters every state
// l >= 1 exactly once and stays in state l (n_l - 1) times, n_l its frame
// count, so the summed posteriors of the stay and step edges (:218-224) are
// occ(l) - 1 and 1, occ(l) = sum_t of the node posterior.  Only occ is
// accumulated here (per warp, in shared memory: a lane's blocks move with
// the window); asg_final applies the identity.
template <int W, class V>
__device__ __forceinline__ void asg_fac_grad_body(const int32_t *__restrict__ em_len,
                                                  const int64_t *__restrict__ tgt,
                                                  const int32_t *__restrict__ tgt_len, Dims d,
                                                  const AsgFastWs &w, float *__restrict__ grad_em,
                                                  int st, int want, int b, int blk,
                                                  unsigned char *smem) {
  constexpr int LP = W * kLatStates;
  static_assert(W <= kGradWarps, "cta_first_band: one lane block per thread");
  float *prow = reinterpret_cast<float *>(smem);       // [kGradWarps][LP] wide-window posteriors
  float *occ = prow + kGradWarps * LP;                 // [kGradWarps][LP] occupancy
  double *gwarp = reinterpret_cast<double *>(occ + kGradWarps * LP);   // [kGradWarps][2]
  unsigned *bins = reinterpret_cast<unsigned *>(gwarp + kGradWarps * 2);   // [kGradWarps][32]
  unsigned *stok = bins + kGradWarps * 32;             // [LP / 4] tokens, 4 states per word

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = d.N;
  const int T = em_len[b];
  const int t0 = blk * kGradFramesPerBlock;
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

  const int L = tgt_len[b];
  float *myp = prow + warp * LP;
  float *myo = occ + warp * LP;
  unsigned *mybins = bins + warp * 32;
  for (int i = lane; i < LP; i += 32) myo[i] = 0.f;
  mybins[lane] = 0u;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  for (int m = threadIdx.x; m < (L + 3) / 4; m += blockDim.x) {
    unsigned v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= (m * 4 + k < L ? (unsigned)y[m * 4 + k] : 0xffu) << (8 * k);
    stok[m] = v;
  }
  __syncthreads();
  const size_t seg0 = (size_t)b * w.W * d.Tmax;
  const int tend = min(tb, T);

  // the fcc rows of the next frame (full-part node posteriors) are loaded one
  // frame ahead
  const V *fca = reinterpret_cast<const V *>(w.fcc_a) + (size_t)b * d.Tmax * 32 + lane;
  const V *fcb = reinterpret_cast<const V *>(w.fcc_b) + (size_t)b * d.Tmax * 32 + lane;
  V ca_nx = (V)0, cb_nx = (V)0;
  if (ta < tend) {
    ca_nx = __ldcg(fca + (size_t)ta * 32);
    cb_nx = __ldcg(fcb + (size_t)ta * 32);
  }
  BandRows<V> br;
  br.A = reinterpret_cast<const V *>(w.fac_a) + seg0 * kLatStates;
  br.B = reinterpret_cast<const V *>(w.fac_b) + seg0 * kLatStates;
  br.EA = w.fac_ea + seg0 * 32;
  br.EB = w.fac_eb + seg0 * 32;
  br.segv = (uint32_t)d.Tmax * kLatStates;
  br.sege = (uint32_t)d.Tmax * 32;
  br.S = L;
  br.nblk = (L + kSpl - 1) / kSpl;
  // the CTA's reference exponent and the band of its first frame t0
  int *sband = reinterpret_cast<int *>(stok + LP / 4);   // [kGradWarps + 2]
  int ref, blo, bhi;
  br.cta_first_band(t0, kGradWarps, sband, ref, blo, bhi);
  float l2min = CUDART_INF_F, l2max = -CUDART_INF_F;   // log2 z_t (the guard adds ref)
  // the two-frame prefetch ring (band.cuh): this warp's first two frames from
  // the CTA's band, widened by the frames in between (fac mass moves by at
  // most one state per frame)
  BandPf<V> pf;
  pf.init(smem + align_up(fac_grad_smem<W>(), 16) + warp * band_pf_bytes<V>());
  int clo, chi, nlo, nhi;   // lane-block windows of frames t and t + 1
  br.window(blo, bhi, ta - t0, clo, chi);
  br.window(blo, bhi, ta + 1 - t0, nlo, nhi);
  if (ta < tend) pf.issue(br, br.frame(ta), clo + lane, clo + lane <= chi, 0, lane);
  cp_async_commit();
  if (ta + 1 < tend) pf.issue(br, br.frame(ta + 1), nlo + lane, nlo + lane <= nhi, 1, lane);
  cp_async_commit();
  int slot = 0;   // ring slot of frame t
  for (int t = ta; t < tend; ++t) {
    const float gam = (float)(ca_nx * cb_nx);   // fcc node posterior, unnormalised
    if (t + 1 < tend) {
      ca_nx = __ldcg(fca + (size_t)(t + 1) * 32);
      cb_nx = __ldcg(fcb + (size_t)(t + 1) * 32);
    }
    // fac node posteriors (:214-217)
    float zl = 0.f;
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
      for (int k = 0; k < kSpl; ++k) zl += q[k];
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
    br.next_window(lo, hi, 2, lo2, hi2);
    if (t + 2 < tend)
      pf.issue(br, br.frame(t + 2), lo2 + lane, lo2 + lane <= hi2, slot == 0 ? 2 : slot - 1,
               lane);
    cp_async_commit();
    const float zc = warp_sum(zl);
    const float izc = 1.f / zc;
    const float izf = 1.f / warp_sum(gam);
    const float l2 = __log2f(zc);
    l2min = fminf(l2min, l2);
    l2max = fmaxf(l2max, l2);
    // token bins and state occupancies of this frame's window (a lane owns
    // its blocks: plain shared read-modify-write for the occupancy)
    auto settle = [&](const float (&q)[kSpl], int m) {
      band_scatter(q, izc, stok + m * kTokWords, mybins);
      float o[kSpl];
      ldv(myo + m * kSpl, o);
#pragma unroll
      for (int k = 0; k < kSpl; ++k) o[k] = fmaf(q[k], izc, o[k]);
      stv(myo + m * kSpl, o);
    };
    if (clo + lane <= chi && clo + lane < br.nblk) settle(q0, clo + lane);
    for (int m = clo + lane + 32; m <= chi; m += 32) {
      if (m < br.nblk) {
        float q[kSpl];
        ldv(myp + m * kSpl, q);
        settle(q, m);
      }
    }
    __syncwarp();
    const float con = (float)mybins[lane] * kFixInv;
    mybins[lane] = 0u;
    if (lane < N) ge[(size_t)t * N + lane] = gam * izf - con;
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

  // ---- block reduction of the occupancy partials in fixed warp order
  // (deterministic)
  if (lane == 0) {
    gwarp[warp * 2 + 0] = gmin;
    gwarp[warp * 2 + 1] = gmax;
  }
  __syncthreads();
  float *dstE = w.part_edge + ((size_t)b * w.nblk + blk) * LP;
  for (int i = threadIdx.x; i < LP; i += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < kGradWarps; ++q) s += occ[q * LP + i];
    dstE[i] = s;
  }
  if (threadIdx.x < 2) {
    double g2 = threadIdx.x ? -CUDART_INF : CUDART_INF;
    for (int q = 0; q < kGradWarps; ++q) {
      const double v = gwarp[q * 2 + threadIdx.x];
      g2 = threadIdx.x ? fmax(g2, v) : fmin(g2, v);
    }
    w.part_guard[((size_t)b * w.nblk + blk) * 4 + 2 + threadIdx.x] = g2;
  }
}

// ---------------------------------------------------------- final kernel --
// per utterance: dA_b = M (.) sum_blocks(fullA partials) - scatter(fac edge
// sums) (criterion.py:239-246), the loss (:244) and the guard verdict.
__global__ void __launch_bounds__(kFinalThreads)
    asg_final_kernel(const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                     const int32_t *__restrict__ em_len, const float *__restrict__ trans, Dims d,
                     AsgFastWs w, double *loss, float *ga_utt, int32_t *status, int want,
                     int fail) {
  pdl_launch_dependents();
  const int b = blockIdx.x;
  __shared__ float sEdge[W2L_MAX_ASG_LABELS];
  __shared__ float sA[1024];
  __shared__ float s_red[32];
  __shared__ int s_bad;
  __shared__ int sy[W2L_MAX_ASG_LABELS];      // targets (int), staged once
  __shared__ int sperm[W2L_MAX_ASG_LABELS];   // token CSR
  __shared__ int sts[33];
  const int N = d.N, NN = N * N;
  // ---- inputs first (the gradient writes none of them: they load while the
  // gradient grid finishes); the token CSR only exists for valid utterances
  const int L = min(max(tgt_len[b], 0), d.Lmax), T = em_len[b], LP = w.lpad;
  const int64_t *y = tgt + (size_t)b * d.Lmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float am = -CUDART_INF_F;
  for (int p = threadIdx.x; p < NN; p += blockDim.x) am = fmaxf(am, trans[p]);
  am = warp_max(am);
  if (lane == 0) s_red[warp] = am;
  if (threadIdx.x == 0) s_bad = 0;
  for (int l = threadIdx.x; l < L; l += blockDim.x) sy[l] = (int)y[l];
  pdl_wait();
  if (threadIdx.x < 2 && w.prog) w.prog[2 * b + threadIdx.x] = 0;   // next tier / call
  const int st = status[b];
  if (st != want) {
    // the first tier owns the zeros (NaN loss) of the utterances it does not
    // compute; a later tier overwrites those it takes
    if (want == W2L_OK) {
      for (int p = threadIdx.x; p < NN; p += blockDim.x) ga_utt[(size_t)b * NN + p] = 0.f;
      if (threadIdx.x == 0) loss[b] = CUDART_NAN;
    }
    return;
  }
  for (int l = threadIdx.x; l < L; l += blockDim.x) sperm[l] = w.perm[(size_t)b * w.lpad + l];
  if (threadIdx.x <= N) sts[threadIdx.x] = w.tok_start[b * 33 + threadIdx.x];   // N+1 written
  // ---- fixed-order sums of the per-frame-block partials: the fac
  // occupancies of the L states and the fcc edge sums of the N x N
  // transitions; each thread owns up to kFinalEnt of these entries and has
  // every partial of a 16-block chunk in flight at once
  const int nb_used = (T + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  const int nent = L + NN;
  const float *pe = w.part_edge + (size_t)b * w.nblk * LP;
  const float *pa = w.part_fullA + (size_t)b * w.nblk * 1024;
  float acc[kFinalEnt];
  const float *src[kFinalEnt];
  size_t stride[kFinalEnt];
#pragma unroll
  for (int k = 0; k < kFinalEnt; ++k) {
    const int e = threadIdx.x + k * kFinalThreads;
    acc[k] = 0.f;
    if (e < L) {
      src[k] = pe + e;
      stride[k] = LP;
    } else {
      const int p = min(e - L, NN - 1);
      src[k] = pa + (p / N) * 32 + p % N;
      stride[k] = 1024;
    }
  }
  for (int q0 = 0; q0 < nb_used; q0 += kFinalChunk) {
    float v[kFinalEnt][kFinalChunk];
#pragma unroll
    for (int k = 0; k < kFinalEnt; ++k) {
      const bool on = threadIdx.x + k * kFinalThreads < nent;
#pragma unroll
      for (int q = 0; q < kFinalChunk; ++q)
        v[k][q] = on && q0 + q < nb_used ? src[k][(size_t)(q0 + q) * stride[k]] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kFinalEnt; ++k) {   // fixed pairwise order
#pragma unroll
      for (int h = 1; h < kFinalChunk; h *= 2)
#pragma unroll
        for (int q = 0; q < kFinalChunk; q += 2 * h) v[k][q] += v[k][q + h];
      acc[k] += v[k][0];
    }
  }
#pragma unroll
  for (int k = 0; k < kFinalEnt; ++k) {
    const int e = threadIdx.x + k * kFinalThreads;
    if (e < L) {
      sEdge[e] = acc[k];
    } else if (e < nent) {
      const int p = e - L;
      sA[(p / N) * 32 + p % N] = acc[k];
    }
  }
  __syncthreads();
  float amax = s_red[0];
  for (int q = 1; q < (int)(blockDim.x >> 5); ++q) amax = fmaxf(amax, s_red[q]);
  for (int p = threadIdx.x; p < NN; p += blockDim.x) {
    const int i = p / N, j = p % N;
    const float full = sA[i * 32 + j] * expf(trans[p] - amax);
    // states labelled i: stay edges (i,i) sum to occ(l) - 1, step edges
    // (i, y_{l-1}) to 1 (see asg_fac_grad_body)
    float con = 0.f;
    for (int q = sts[i]; q < sts[i + 1]; ++q) {
      const int l = sperm[q];
      if (i == j) con += sEdge[l] - 1.f;
      if (l > 0 && sy[l - 1] == j) con += 1.f;
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
  bad |= !(fabs(zF - zFb) <= tol) || !(fabs(zC - zCb) <= tol);
  for (int q = threadIdx.x; q < nb_used; q += blockDim.x) {
    // every frame's log-normaliser (log2 units) must reproduce the totals
    const double *g = w.part_guard + ((size_t)b * w.nblk + q) * 4;
    bad |= !(fabs(g[0] * ln2 - zF) <= tol && fabs(g[1] * ln2 - zF) <= tol);
    bad |= !(fabs(g[2] * ln2 - zC) <= tol && fabs(g[3] * ln2 - zC) <= tol);
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    loss[b] = zF - zC;
    status[b] = s_bad ? fail : W2L_OK;
  }
}

// Both directions ran: their totals must agree (the per-frame guard of the
// gradient path needs the posteriors, which loss-only mode does not form).
__global__ void asg_loss_only_kernel(const int32_t *__restrict__ em_len, Dims d, AsgFastWs w,
                                     double *loss, int32_t *status, int want, int fail) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  if (status[b] != want) {
    if (want == W2L_OK) loss[b] = CUDART_NAN;   // (a later tier overwrites those it takes)
    return;
  }
  const double zF = w.scal[b * 4 + 0], zFb = w.scal[b * 4 + 1];
  const double zC = w.scal[b * 4 + 2], zCb = w.scal[b * 4 + 3];
  const double tol = 1e-4 * fmax(1.0, sqrt((double)em_len[b] / 1600.0));
  loss[b] = zF - zC;                                         // criterion.py:244
  const bool bad = !(isfinite(zF) && isfinite(zFb) && isfinite(zC) && isfinite(zCb)) ||
                   !(fabs(zF - zFb) <= tol && fabs(zC - zCb) <= tol);
  status[b] = bad ? fail : W2L_OK;
}

// One launch for both gradient bodies; they are independent, so their CTAs
// run side by side.  The kinds alternate in x (even: fac + gradient row,
// odd: fcc edges; 128 frames each), so both are dispatched from the start of
// the launch.  With the kinds in blockIdx.z instead every fac CTA was
// dispatched before any fcc CTA (slower).  Grid (2B, nblk): y is the frame
// block's completion rank (block_of_rank), so with PDL the CTAs run in the
// order the two chains complete their frames; prog (null: the chains have
// finished) gates them.
// fp32 gradient CTAs per SM the registers must allow (W <= 3): 4 (64
// registers, no spills) against 3 (79): asg grad 100 -> 96 us, two-criteria
// step 0.426 -> 0.418 ms (5 of 5 A/B pairs)
#ifndef W2L_ASG_GRAD_MINB
#define W2L_ASG_GRAD_MINB 4
#endif
template <int W, class V>
__global__ void __launch_bounds__(kGradWarps * 32,
                                  W <= 3 ? (sizeof(V) == 4 ? W2L_ASG_GRAD_MINB : 2) : 1)
    asg_grad_kernel(const float *__restrict__ em, const int32_t *__restrict__ em_len,
                    const int64_t *__restrict__ tgt, const int32_t *__restrict__ tgt_len,
                    const float *__restrict__ trans, Dims d, AsgFastWs w,
                    float *__restrict__ grad_em, const int32_t *__restrict__ status, int want,
                    const int *prog) {
  extern __shared__ __align__(16) unsigned char gsm[];
  pdl_launch_dependents();
  if (!prog) pdl_wait();   // not streamed: the chain grid must have completed
  const int b = blockIdx.x >> 1, blk = block_of_rank(blockIdx.y, w.nblk);
  const int T = em_len[b], t0 = blk * kGradFramesPerBlock;
  W2L_TL(const unsigned long long tl0 = gtimer());
  if (t0 < T) wait_chain_progress(prog, b, min(t0 + kGradFramesPerBlock, T), T - t0);
  W2L_TL(const unsigned long long tl1 = gtimer());
  const int st = *(volatile const int32_t *)(status + b);
  if (blockIdx.x & 1)
    asg_fcc_grad_body<V>(em, em_len, d, w, st, want, b, blk, gsm);
  else
    asg_fac_grad_body<W, V>(em_len, tgt, tgt_len, d, w, grad_em, st, want, b, blk, gsm);
  W2L_TL(if (threadIdx.x == 0 && t0 < T) tl_rec(4000000ull + (blockIdx.x & 1) * 500000ull + b * 1000 + blk, tl0, tl1, gtimer()));
}

template <int W, class V>
cudaError_t launch_grad_w(const float *em, const int32_t *em_len, const int64_t *tgt,
                          const int32_t *tgt_len, const float *trans, Dims d, const AsgFastWs &w,
                          float *grad_em, const int32_t *status, int want, cudaStream_t s,
                          bool stream) {
  const size_t smem = std::max(align_up(fac_grad_smem<W>(), 16) + kGradWarps * band_pf_bytes<V>(),
                               kGradWarps * fcc_stage_bytes<V>());
  auto k = asg_grad_kernel<W, V>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return launch_maybe_pdl(k, dim3(2 * d.B, w.nblk), dim3(kGradWarps * 32), smem, s, true, em,
                          em_len, tgt, tgt_len, trans, d, w, grad_em, status, want,
                          (const int *)(stream ? w.prog : nullptr));
}

template <class V>
cudaError_t launch_asg_tier(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, const float *trans, Dims d,
                            const AsgFastWs &w, double *loss, float *grad_em, float *ga_utt,
                            int32_t *status, cudaStream_t s, Tracer *tr, unsigned phases,
                            int want, int fail) {
  // stream the gradient behind the chains (PDL) when both run in this call
  // and no stage trace separates them; otherwise the chains publish no
  // progress and the gradient CTAs do not wait
  const bool stream = (phases & 1u) && (phases & 2u) && !(phases & 4u) && !tr &&
                      ((phases & 8u) || pdl_enabled());
  AsgFastWs wc = w;
  if (!stream) wc.prog = nullptr;
  cudaError_t err = cudaSuccess;
  if (phases & 5u) {
    const size_t smem = chain_smem_bytes<V>();
    // (the streamed-gradient trigger is compiled only into the streaming
    // variant: its checks cost the recursion loops ~2.5%)
    auto k = wc.prog ? asg_chain_kernel<V, true> : asg_chain_kernel<V, false>;
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
    err = launch_maybe_pdl(k, dim3(d.B, 2), dim3(32 * (2 + w.W)), smem, s, false, em, em_len, tgt,
                           tgt_len, trans, d, wc, status, want, fail);
    if (err != cudaSuccess) return err;
  }
  trace(tr, s);  // chain
  if (phases & 4u) {
    return launch_maybe_pdl(asg_loss_only_kernel, dim3((d.B + 127) / 128), dim3(128), 0, s, true,
                            em_len, d, w, loss, status, want, fail);
  }
  if (!(phases & 2u)) return cudaSuccess;
  switch (w.W) {
#define W2L_CASE(n)                                                                          \
  case n:                                                                                    \
    if constexpr (n <= kMaxLatWarps) {                                                       \
    err = launch_grad_w<n, V>(em, em_len, tgt, tgt_len, trans, d, w, grad_em, status, want,  \
                              s, stream);                                                    \
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
  err = launch_maybe_pdl(asg_final_kernel, dim3(d.B), dim3(kFinalThreads), 0, s, true, tgt, tgt_len, em_len,
                         trans, d, w, loss, ga_utt, status, want, fail);
  trace(tr, s);  // final
  return err;
}

}  // namespace

int asg_fast_spl(int Lmax) { return lat_warps(Lmax) <= kMaxLatWarps ? kSpl : 0; }

static size_t asg_ws_layout(Dims d, void *base, AsgFastWs *w) {
  const int W = lat_warps(d.Lmax);
  const int lpad = W * kLatStates;
  const int nblk = (d.Tmax + kGradFramesPerBlock - 1) / kGradFramesPerBlock;
  const size_t BT = (size_t)d.B * d.Tmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? (void *)((char *)base + o) : nullptr;
  };
  AsgFastWs t;
  // rows sized for the double tier (the float tier uses the first half; the
  // tiers run one after the other on the same stream)
  t.fcc_a = take(BT * 32 * sizeof(double));
  t.fcc_b = take(BT * 32 * sizeof(double));
  const int tpad = round_up(d.Tmax + 1, 8);
  t.fcc_ka = (int *)take((size_t)d.B * tpad * 4);
  t.fcc_kb = (int *)take((size_t)d.B * tpad * 4);
  t.fac_a = take(BT * lpad * sizeof(double));
  t.fac_b = take(BT * lpad * sizeof(double));
  t.fac_ea = (int *)take(BT * W * 32 * 4);
  t.fac_eb = (int *)take(BT * W * 32 * 4);
  t.scal = (double *)take((size_t)d.B * 4 * 8);
  t.part_fullA = (float *)take((size_t)d.B * nblk * 1024 * 4);
  t.part_edge = (float *)take((size_t)d.B * nblk * lpad * 4);
  t.part_guard = (double *)take((size_t)d.B * nblk * 4 * 8);
  t.prog = (int *)take((size_t)d.B * 2 * 4);
  t.route = (int *)take(kRouteWords * 4);
  t.perm = (int *)take((size_t)d.B * lpad * 4);
  t.tok_start = (int *)take((size_t)d.B * 33 * 4);
  t.spl = kSpl;
  t.W = W;
  t.lpad = lpad;
  t.nblk = nblk;
  t.tpad = tpad;
  if (w) *w = t;
  return off;
}

#ifdef W2L_TIMELINE
int tl_read_asg(unsigned long long *host, int maxn) {
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

size_t asg_fast_ws_bytes(Dims d) { return asg_ws_layout(d, nullptr, nullptr); }
void asg_fast_ws_carve(Dims d, void *ws, AsgFastWs *w) { asg_ws_layout(d, ws, w); }

cudaError_t launch_asg_fast(const float *em, const int32_t *em_len, const int64_t *tgt,
                            const int32_t *tgt_len, const float *trans, Dims d,
                            const AsgFastWs &w, double *loss, float *grad_em, float *ga_utt,
                            int32_t *status, cudaStream_t s, Tracer *tr, unsigned phases,
                            int tier) {
  if (w.W < 1 || w.W > kMaxLatWarps) return cudaErrorInvalidValue;
  if (tier == 0)
    return launch_asg_tier<float>(em, em_len, tgt, tgt_len, trans, d, w, loss, grad_em, ga_utt,
                                  status, s, tr, phases, W2L_OK, kNeedsF64);
  return launch_asg_tier<double>(em, em_len, tgt, tgt_len, trans, d, w, loss, grad_em, ga_utt,
                                 status, s, tr, phases, kNeedsF64, kNeedsLog);
}

// --------------------------------------------------- batch reduction of dA --
// one warp per transition pair: fixed-order float64 sum over utterances
// (trainer.py:442-447 sums in float64), deterministic run to run
__global__ void reduce_grad_trans_kernel(const float *ga_utt, const int32_t *status, Dims d,
                                         float *grad_trans) {
  pdl_enter();
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= d.N * d.N) return;
  double s = 0.0;
  for (int b = lane; b < d.B; b += 32)
    if (status[b] == W2L_OK) s += (double)ga_utt[(size_t)b * d.N * d.N + p];
  s = warp_sum(s);
  if (lane == 0) grad_trans[p] = (float)s;
}

// SGD with classical momentum on the transitions (autodiff.py:429-433) after
// the /B of trainer.py:447; float32 arithmetic without contraction, as numpy
__global__ void transitions_sgd_kernel(float *w, float *v, const float *gsum, int nn, double batch,
                                       float lr, float momentum) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nn) return;
  const float g = (float)((double)gsum[p] / batch);   // (total / batch.size).astype(f32)
  const float vv = __fadd_rn(__fmul_rn(v[p], momentum), g);
  v[p] = vv;
  w[p] = __fsub_rn(w[p], __fmul_rn(lr, vv));
}

cudaError_t launch_transitions_sgd(float *w, float *v, const float *gsum, int N, int batch,
                                   float lr, float momentum, cudaStream_t s) {
  const int nn = N * N;
  transitions_sgd_kernel<<<(nn + 255) / 256, 256, 0, s>>>(w, v, gsum, nn, (double)batch, lr,
                                                          momentum);
  return cudaGetLastError();
}

cudaError_t launch_reduce_grad_trans(const float *ga_utt, const int32_t *status, Dims d,
                                     float *grad_trans, cudaStream_t s) {
  const int n = d.N * d.N;
  return launch_maybe_pdl(reduce_grad_trans_kernel, dim3((n + 7) / 8), dim3(256), 0, s, true, ga_utt,
                          status, d, grad_trans);
}

}  // namespace w2l
