// Multi-warp wavefront chains for the serial forward/backward recursions.
//
// CHAIN CTA: one CTA runs one (utterance, direction).  Its warps:
//   warp 0          producer: stages emission chunks with cp.async and writes
//                   Et[t][i] = exp(e[t][i] - max_i e[t][i]) into a ring in
//                   shared memory, once for the whole CTA;
//   warp 1 (ASG)    the fcc recursion (fully connected N x N graph, 32-lane
//                   mat-vec per frame, asg_fast.cu);
//   lattice warps   W warps over a linear lattice (ASG fac: L states; CTC:
//                   2L+1 states).  Lattice warp w owns states
//                   [128 w, 128 (w+1)), kSpl = 4 consecutive states per lane
//                   in registers of type V with one power-of-two exponent per
//                   lane (block floating point, renormalised every kRenormF
//                   steps).
//
// V is the precision tier: float (the fast path) or double (the wide-range
// tier for inputs whose dynamic range exceeds fp32's; same algorithm).
//
// A lattice state at step j depends only on its own lane and the previous
// lane's states at step j-1 (criterion.py:126-134,147-155 for CTC,
// :197-202,207-212 for the fac graph), so the warps form a WAVEFRONT: warp w
// runs a few steps behind its upstream neighbour (w-1 forward, w+1 backward)
// and reads the neighbour's boundary states of step j-1 from a small ring in
// shared memory.  Progress is published every kBlk = 8 steps through
// release/acquire counters, so the warps never meet at a barrier.
//
// ROWS.  Every step's lane values and exponents go to the workspace
// (warp-major [W][Tmax][128] values, [W][Tmax][32] exponents; lanes wholly
// past the lattice's last state store nothing and the gradient kernels do
// not read them).  A checkpointed variant that recomputed alpha and beta per
// 16-frame segment inside the gradient kernels moved ~10x less HBM data but
// executed 2.3x the instructions and ran 2x slower.
//
// The processing index j counts steps in the direction of the recursion
// (forward: frame t = j; backward: frame t = T-1-j).  Forward step j consumes
// Et at frame j; backward step j consumes frame u = T-j and produces beta' at
// frame T-1-j.  Ring slots are assigned so that step j reads slot j mod kRing.
#pragma once

#include <type_traits>

#include "laneblock.cuh"

namespace w2l {

#ifndef W2L_SPL
#define W2L_SPL 4
#endif
constexpr int kSpl = W2L_SPL;              // lattice states per lane (even, multiple of 4)
static_assert(kSpl % 4 == 0, "lane blocks are moved as 4-wide vectors");
constexpr int kLatStates = 32 * kSpl;      // states per lattice warp
constexpr int kMaxLatWarps = 32 / kSpl;    // 1024 states
constexpr int kBndRing = 128;              // boundary ring (steps): decouples neighbouring warps
constexpr int kCounters = kMaxLatWarps + 2;  // lattice warps + fcc warp (+ spare)
constexpr int kDone = 1 << 30;             // progress of a finished consumer

constexpr int kRenormF = 4;                // steps between lane renormalisations
constexpr int kBlk = 8;                    // steps per unrolled block (one publish / wait per block)

// Streamed gradient: a chain warp triggers the dependent launch once its
// steps reach stream_trigger_step(T) = ceil(T NUM / DIV), i.e. after the
// block of kBlk steps stream_trigger_block(T).  Per lattice kind (A/B builds:
// W2L_TRIG_{FAC,CTC}_{NUM,DIV}; the fac fraction also serves ASG's fcc warp):
// ASG at 3T/5, CTC at 2T/3.  In the two-criteria step ASG's gradient grid
// must launch before CTC's (its CTAs then queue first): ASG at 2T/3 with CTC
// at T/2 ran 0.445 vs 0.420 ms.  3T/5 + 2T/3 against T/2 + T/2: device step
// -1%, e2e +0.7% (4 A/B pairs; ASG 3T/5 alone: 8 of 8 pairs faster).
#ifndef W2L_TRIG_FAC_NUM
#define W2L_TRIG_FAC_NUM 3
#endif
#ifndef W2L_TRIG_FAC_DIV
#define W2L_TRIG_FAC_DIV 5
#endif
#ifndef W2L_TRIG_CTC_NUM
#define W2L_TRIG_CTC_NUM 2
#endif
#ifndef W2L_TRIG_CTC_DIV
#define W2L_TRIG_CTC_DIV 3
#endif
template <int KIND>   // 0: fac (ASG), 1: CTC
__host__ __device__ __forceinline__ int stream_trigger_step(int T) {
  return KIND == 0 ? (T * W2L_TRIG_FAC_NUM + W2L_TRIG_FAC_DIV - 1) / W2L_TRIG_FAC_DIV
                   : (T * W2L_TRIG_CTC_NUM + W2L_TRIG_CTC_DIV - 1) / W2L_TRIG_CTC_DIV;
}
template <int KIND>
__device__ __forceinline__ int stream_trigger_block(int T) {
  return max(1, (stream_trigger_step<KIND>(T) + kBlk - 1) / kBlk - 1);
}

constexpr int kProdStages = 4;             // emission chunks in flight (hides HBM latency)
// The producer runs up to a ring ahead of the recursions and then polls for
// free slots; each poll takes issue slots from the recursion warps of the
// (up to two) chain CTAs on the SM, so it sleeps between polls.
#ifndef W2L_PROD_SLEEP_NS
#define W2L_PROD_SLEEP_NS 256
#endif

// Et ring depth (frames): > wavefront spread + producer stages
template <class V>
struct Ring {
  static constexpr int n = sizeof(V) == 4 ? 256 : 128;
};

template <class V>
struct __align__(sizeof(V) == 4 ? 16 : 8) BndT {
  V v0, v1;
  int ex, pad;
};

// shared-memory layout of a chain CTA (dynamic shared memory)
template <class V>
struct ChainSm {
  V ering[Ring<V>::n][kStride];
  float raw[kProdStages][kChunk * 32];
  BndT<V> bnd[kMaxLatWarps][kBndRing];
  __align__(16) V vec[2][32];
  double fin[kMaxLatWarps + 1];
  int prod;
  int cons[kCounters];
  int flush;   // a used token's Et fell below exp(-kFlush) (set by the producer)
};

// Dynamic shared memory of a chain CTA.  Requested above a third of the SM's
// shared memory so that at most TWO chain CTAs (of either criterion) are
// resident per SM: with the default placement a third chain CTA on an SM
// ran its three recursions at about half speed, and the slowest chain of
// the batch gates the gradient phase (two-stream timeline: chains ending
// between 153 and 330 us instead of ~180).  W2L_CHAIN_SMEM_KB overrides
// (A/B measurements).
template <class V>
inline size_t chain_smem_bytes() {
  static const size_t kb = [] {
    const char *e = getenv("W2L_CHAIN_SMEM_KB");
    return e ? (size_t)atoi(e) : (size_t)80;
  }();
  return sizeof(ChainSm<V>) > kb * 1024 ? sizeof(ChainSm<V>) : kb * 1024;
}

// ---- 4-wide vector load/store of lane values (float4 / 2 x double2)
__device__ __forceinline__ void ld4(const float *p, float (&v)[4]) {
  const float4 x = *reinterpret_cast<const float4 *>(p);
  v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
__device__ __forceinline__ void ld4(const double *p, double (&v)[4]) {
  const double2 x = reinterpret_cast<const double2 *>(p)[0];
  const double2 y = reinterpret_cast<const double2 *>(p)[1];
  v[0] = x.x, v[1] = x.y, v[2] = y.x, v[3] = y.y;
}
__device__ __forceinline__ void st4(float *p, const float (&v)[4]) {
  *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void st4(double *p, const double (&v)[4]) {
  reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
}
// L2-only loads (rows written by a concurrently running chain grid)
__device__ __forceinline__ void ld4_cg(const float *p, float (&v)[4]) {
  const float4 x = __ldcg(reinterpret_cast<const float4 *>(p));
  v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
__device__ __forceinline__ void ld4_cg(const double *p, double (&v)[4]) {
  const double2 x = __ldcg(reinterpret_cast<const double2 *>(p));
  const double2 y = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
  v[0] = x.x, v[1] = x.y, v[2] = y.x, v[3] = y.y;
}
template <class V, int K>
__device__ __forceinline__ void ldv_cg(const V *p, V (&v)[K]) {
#pragma unroll
  for (int q = 0; q < K; q += 4) ld4_cg(p + q, *reinterpret_cast<V(*)[4]>(v + q));
}
// a whole lane block (kSpl values) as 4-wide vectors
template <class V, int K>
__device__ __forceinline__ void ldv(const V *p, V (&v)[K]) {
#pragma unroll
  for (int q = 0; q < K; q += 4) ld4(p + q, *reinterpret_cast<V(*)[4]>(v + q));
}
template <class V, int K>
__device__ __forceinline__ void stv(V *p, const V (&v)[K]) {
#pragma unroll
  for (int q = 0; q < K; q += 4) st4(p + q, *reinterpret_cast<const V(*)[4]>(v + q));
}

// ---- release/acquire progress counters (CTA scope, shared memory)
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.cta.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_cta() {
  asm volatile("fence.acq_rel.cta;\n" ::: "memory");
}
// Polls of the recursion warps.  W2L_SPIN_NS > 0 sleeps between polls (a
// poll takes issue slots from the other chain CTA on the SM).
#ifndef W2L_SPIN_NS
#define W2L_SPIN_NS 32
#endif
__device__ __forceinline__ void spin_pause() {
  if (W2L_SPIN_NS > 0) __nanosleep(W2L_SPIN_NS);
}
// every lane spins on the same word (a broadcast load, no divergence)
__device__ __forceinline__ void wait_ge(const int *p, int need) {
  while (ld_acquire(p) < need) spin_pause();
}
// wait for up to three counters with relaxed polls issued together, then one
// acquire fence (cheaper than three acquire loads when they are satisfied)
__device__ __forceinline__ void wait3(const int *p0, int n0, const int *p1, int n1, const int *p2,
                                      int n2) {
  while (true) {
    const int a = ld_relaxed(p0), b = ld_relaxed(p1), c = ld_relaxed(p2);
    if (a >= n0 && b >= n1 && c >= n2) break;
    spin_pause();
  }
  fence_acq_rel_cta();
}
// all lanes' shared-memory writes are ordered before lane 0's release
__device__ __forceinline__ void publish(int *p, int v, int lane) {
  __syncwarp();
  if (lane == 0) st_release(p, v);
  __syncwarp();
}

struct ProdCtx {
  const float *e;  // &em[b][0][0]
  int N, T;
  bool fwd;
  int nconsumers;  // counters cons[0 .. nconsumers) gate ring reuse
  int logits;      // shift term: 0 = max_i e (log-probs), 1 = -log sum_i Et (logits)
  unsigned tokmask;  // tokens whose Et enter the recursions (flush check)
  int *gprog = nullptr;  // global progress word of this (utterance, direction), or null
  int trig = 0;          // streamed gradient: the step at which to trigger the launch
};

// Publish the CTA's progress (steps whose rows every row-writing warp has
// stored) to the global word, capped at T - 1: the final value T is
// published by the CTA epilogue after the totals are written.  The
// acquire of the warps' CTA-scope counters followed by the gpu-scope
// release makes their row stores visible to a gradient CTA that acquires
// the word (release is cumulative).  Lane 0 only.
template <class V>
__device__ __forceinline__ void prod_publish(ChainSm<V> &sm, const ProdCtx &c, int &last) {
  int mn = c.T - 1;
  for (int q = 0; q < c.nconsumers; ++q) mn = min(mn, ld_acquire(&sm.cons[q]));
  if (mn > last) {
    st_release_gpu(c.gprog, mn);
    last = mn;
  }
}

// frame of processing index p
__device__ __forceinline__ int frame_of(bool fwd, int T, int p) { return fwd ? p : T - 1 - p; }
// ring slot of processing index p: step j reads slot j (forward reads index
// j, backward index j-1)
template <class V>
__device__ __forceinline__ int ring_slot(bool fwd, int p) {
  return (p + (fwd ? 0 : 1)) & (Ring<V>::n - 1);
}
__device__ __forceinline__ int eidx_of(bool fwd, int j) { return fwd ? j : j - 1; }

// Stage chunk p0 (up to 32 frames, processing order) linearly: the frames of
// a chunk are contiguous in the emissions (ascending for the forward
// direction, descending for the backward one), so lane l copies elements
// l, l+32, ... of that range (coalesced 4-byte cp.async).
template <class V>
__device__ __forceinline__ void prod_issue(ChainSm<V> &sm, const ProdCtx &c, int p0, int buf,
                                           int lane) {
  const int rows = min(kChunk, c.T - p0);
  const int f0 = c.fwd ? p0 : c.T - p0 - rows;   // lowest frame of the chunk
  const float *src = c.e + (size_t)f0 * c.N;
  float *dst = sm.raw[buf];
  const int n = rows * c.N;
  for (int e = lane; e < n; e += 32) cp_async4(dst + e, src + e);
  cp_async_commit();
}

// Et of one emission value (the gradient kernels recompute it identically)
template <class V>
__device__ __forceinline__ V et_of(float e, float m) {
  if (sizeof(V) == 4) return (V)__expf(e - m);
  return (V)exp((double)e - (double)m);
}

// The producer warp: converts every frame once for the whole CTA (lane r
// owns processing row r of a 32-frame chunk).  The row maxima are summed
// into *shift_sum (CTC loss offset) when requested.
template <class V>
__device__ __forceinline__ void producer_run(ChainSm<V> &sm, const ProdCtx &c, int lane,
                                             double *shift_sum) {
  constexpr int kRing = Ring<V>::n;
  double shifts = 0.0;
  bool flush = false;
  int published = 0;
  bool trig = false;   // streamed gradient: this warp's share of the dependent launch
  const int nch = (c.T + kChunk - 1) / kChunk;
  // kProdStages - 1 chunks in flight ahead of the one being converted (an
  // empty commit group keeps the wait count uniform past the end)
#pragma unroll
  for (int q = 0; q < kProdStages - 1; ++q) {
    if (q < nch) prod_issue(sm, c, q * kChunk, q, lane);
    else cp_async_commit();
  }
  for (int ch = 0; ch < nch; ++ch) {
    const int p0 = ch * kChunk, rows = min(kChunk, c.T - p0);
    const int nx = ch + kProdStages - 1;
    if (nx < nch) prod_issue(sm, c, nx * kChunk, nx % kProdStages, lane);
    else cp_async_commit();
    cp_async_wait<kProdStages - 1>();
    __syncwarp();
    float x[32];
    const int rlin = c.fwd ? lane : rows - 1 - lane;   // ascending-frame row of this lane
    const float *r = sm.raw[ch % kProdStages] + max(rlin, 0) * c.N;
    float m = -CUDART_INF_F, mn = CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      x[i] = (i < c.N && lane < rows) ? r[i] : -CUDART_INF_F;
      m = fmaxf(m, x[i]);
      if ((c.tokmask >> i) & 1u) mn = fminf(mn, x[i]);
    }
    // Et = exp(e - m) of a token the recursions use must not flush to zero
    // (the same flush in both directions would pass the consistency guard)
    flush |= lane < rows && mn - m < -Pow2<V>::kFlush;
    // ring slots [p0, p0+rows) previously held p - kRing: every consumer must
    // be past the step that read them (a step j reads index <= j)
    const int need = p0 + rows + 1 - kRing;
    for (int q = 0; q < c.nconsumers; ++q)
      while (ld_relaxed(&sm.cons[q]) < need) __nanosleep(W2L_PROD_SLEEP_NS);
    fence_acq_rel_cta();
    if (lane < rows) {
      V *dd = sm.ering[ring_slot<V>(c.fwd, p0 + lane)];
      double se = 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const V v = i < c.N ? et_of<V>(x[i], m) : (V)0;
        dd[i] = v;
        se += (double)v;
      }
      dd[32] = (V)0;
      // log-probs: the frame's shift is its max; logits (log-softmax fused):
      // max logp = -log sum_i exp(x_i - max x)
      shifts += c.logits ? -log(se) : (double)m;
    }
    __syncwarp();   // raw[ch % kProdStages] is refilled by a later issue
    publish(&sm.prod, p0 + rows, lane);
    if (c.gprog && lane == 0) prod_publish(sm, c, published);
    if (c.gprog && !trig && p0 + rows >= c.trig) {
      pdl_launch_dependents();   // (see lattice_run)
      trig = true;
    }
  }
  if (c.gprog && !trig) pdl_launch_dependents();
  // the recursions trail the producer by up to the ring depth: keep
  // publishing until they are done (T - 1: see prod_publish)
  if (c.gprog && lane == 0) {
    while (published < c.T - 1) {
      __nanosleep(512);
      prod_publish(sm, c, published);
    }
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, flush) && lane == 0) sm.flush = 1;
  if (shift_sum) {
    shifts = warp_sum(shifts);
    if (lane == 0) *shift_sum = shifts;
  }
}

// ------------------------------------------------------------ lattices --
enum { kFac = 0, kCtc = 1 };

struct LatCtx {
  int w, W;          // this lattice warp, lattice warps in the CTA
  int lane, T, N;
  int nstates;       // L (fac) or 2L+1 (CTC)
  int cons_idx;      // counter index of lattice warp 0
  void *rows;        // rows of this utterance: V [W][Tmax][128]
  int *exps;         //                         int [W][Tmax][32]
  int Tmax;
};

template <class V>
struct LatState {
  V v[kSpl];
  V S[kSpl], P[kSpl];       // fac weights (stay, step); CTC: skip flags in P
  int tok[kSpl];            // tokens (E column) of this lane's states
  int nbtok1, nbtok2;       // tokens of the two states after this lane (backward)
  int ex;
  V asc;                    // alignment factor of the neighbour's values
};

// lattice state weights.  fac: tok = y_l, S = M[y_l][y_l], P = M[y_l][y_{l-1}]
// (forward) or M[y_{l+1}][y_l] (backward), M = exp(A - max A).  CTC: tok =
// blank (even s) or y_{s/2}; P = skip flag (forward: edge s-2 -> s; backward:
// edge s+2 -> s).  Padding states read the zero column N.
template <int KIND, bool FWD, class V>
__device__ __forceinline__ void lat_init_weights(LatState<V> &f, int w, int lane, int N, int S,
                                                 const int64_t *y, int L, const float *trans,
                                                 float amax, int blank) {
  auto tok_of = [&](int s) -> int {
    if (s >= S) return N;
    if (KIND == kFac) return (int)y[s];
    return (s & 1) ? (int)y[s >> 1] : blank;
  };
  auto ctc_skip = [&](int s) -> bool {   // edge s-2 -> s exists
    return (s & 1) && s >= 3 && s < S && y[s >> 1] != y[(s >> 1) - 1];
  };
  auto mexp = [&](float a) -> V { return Pow2<V>::ex((V)a - (V)amax); };
  const int base = (w * 32 + lane) * kSpl;
#pragma unroll
  for (int k = 0; k < kSpl; ++k) {
    const int s = base + k;
    f.tok[k] = tok_of(s);
    if (KIND == kFac) {
      if (s < L) {
        const int yl = (int)y[s];
        f.S[k] = mexp(trans[yl * N + yl]);
        if (FWD)
          f.P[k] = s > 0 ? mexp(trans[yl * N + (int)y[s - 1]]) : (V)0;
        else
          f.P[k] = s + 1 < L ? mexp(trans[(int)y[s + 1] * N + yl]) : (V)0;
      } else {
        f.S[k] = (V)0;
        f.P[k] = (V)0;
      }
    } else {
      f.S[k] = (V)1;
      f.P[k] = FWD ? (ctc_skip(s) ? (V)1 : (V)0) : (ctc_skip(s + 2) ? (V)1 : (V)0);
    }
  }
  f.nbtok1 = tok_of(base + kSpl);
  f.nbtok2 = tok_of(base + kSpl + 1);
}

// Inputs of one step, loaded ahead of the recursion (shared-memory loads
// cannot be hoisted by the compiler across the previous steps' stores).
template <class V>
struct StepIn {
  V E[kSpl];     // Et of this lane's states
  V En1, En2;    // Et of the two states after this lane (backward edge lane)
  V b0, b1;      // upstream boundary states after the previous step
  int bex;       // their lane exponent
};

template <int KIND, bool FWD, class V>
__device__ __forceinline__ void load_step_in(StepIn<V> &in, const LatState<V> &f, const V *er,
                                             const BndT<V> *bi, int lane) {
  if (KIND == kCtc) {   // even states are blanks: one shared Et
    const V eblank = er[f.tok[0]];
#pragma unroll
    for (int k = 0; k < kSpl; ++k) in.E[k] = (k & 1) ? er[f.tok[k]] : eblank;
  } else {
#pragma unroll
    for (int k = 0; k < kSpl; ++k) in.E[k] = er[f.tok[k]];
  }
  if (!FWD) {
    in.En1 = er[f.nbtok1];
    in.En2 = KIND == kCtc ? er[f.nbtok2] : (V)0;
  }
  if (bi) {
    const BndT<V> x = *bi;
    in.b0 = x.v0;
    in.b1 = x.v1;
    in.bex = x.ex;
  } else {
    in.b0 = in.b1 = (V)0;
    in.bex = kNegExp;
  }
}

// One recursion step; bo: this warp's boundary slot for this step.
// SLOW: the neighbour's exponent is exchanged every step and dead (all-zero)
// lanes adopt it -- needed while the lattice frontier sweeps the warp.
// FAST (every lane live): lane exponents only move at renormalisations, so
// the neighbour's alignment factor f.asc is recomputed on the step after
// each renormalisation (`check`) and a step is one shuffle plus the
// recursion's arithmetic.
template <int KIND, bool FWD, bool FAST, class V>
__device__ __forceinline__ void lat_step(LatState<V> &f, const StepIn<V> &in, BndT<V> *bo,
                                         int lane, bool renorm, bool check) {
  const bool edge_in = FWD ? lane == 0 : lane == 31;
  if (FWD) {
    V nb = __shfl_up_sync(0xffffffffu, f.v[kSpl - 1], 1);
    if (edge_in) nb = in.b0;
    if (!FAST || check) {
      int nbe = __shfl_up_sync(0xffffffffu, f.ex, 1);
      if (edge_in) nbe = in.bex;
      f.asc = align_factor<kSpl, V>(nbe, f.v, f.ex, check);
    }
    const V n1 = nb * f.asc;
    if (KIND == kFac) {
#pragma unroll
      for (int k = kSpl - 1; k >= 1; --k)
        f.v[k] = in.E[k] * fma(f.S[k], f.v[k], f.P[k] * f.v[k - 1]);
      f.v[0] = in.E[0] * fma(f.S[0], f.v[0], f.P[0] * n1);
    } else {
      // even states are blanks (no skip edge); odd state k skips from k-2,
      // which for k = 1 is the previous lane's last state
#pragma unroll
      for (int k = kSpl - 1; k >= 2; --k)
        f.v[k] = (k & 1) ? in.E[k] * fma(f.P[k], f.v[k - 2], f.v[k] + f.v[k - 1])
                         : in.E[k] * (f.v[k] + f.v[k - 1]);
      const V v1 = in.E[1] * fma(f.P[1], n1, f.v[1] + f.v[0]);
      f.v[0] = in.E[0] * (f.v[0] + n1);
      f.v[1] = v1;
    }
  } else {
    V wv[kSpl];
#pragma unroll
    for (int k = 0; k < kSpl; ++k) wv[k] = in.E[k] * f.v[k];
    V nb1 = __shfl_down_sync(0xffffffffu, wv[0], 1);
    V nb2 = KIND == kCtc ? __shfl_down_sync(0xffffffffu, wv[1], 1) : (V)0;
    if (edge_in) {
      nb1 = in.En1 * in.b0;
      nb2 = in.En2 * in.b1;
    }
    if (!FAST || check) {
      int nbe = __shfl_down_sync(0xffffffffu, f.ex, 1);
      if (edge_in) nbe = in.bex;
      f.asc = align_factor<kSpl, V>(nbe, wv, f.ex, check);
    }
    const V n1 = nb1 * f.asc;
    if (KIND == kFac) {
#pragma unroll
      for (int k = 0; k < kSpl - 1; ++k) f.v[k] = fma(f.S[k], wv[k], f.P[k] * wv[k + 1]);
      f.v[kSpl - 1] = fma(f.S[kSpl - 1], wv[kSpl - 1], f.P[kSpl - 1] * n1);
    } else {
      const V n2 = nb2 * f.asc;
      // P[k] holds the skip flag of the edge k+2 -> k
#pragma unroll
      for (int k = 0; k < kSpl - 2; ++k)
        f.v[k] = (k & 1) ? fma(f.P[k], wv[k + 2], wv[k] + wv[k + 1]) : wv[k] + wv[k + 1];
      f.v[kSpl - 2] = wv[kSpl - 2] + wv[kSpl - 1];
      f.v[kSpl - 1] = fma(f.P[kSpl - 1], n2, wv[kSpl - 1] + n1);
    }
  }
  if (renorm) lane_renorm<kSpl, V>(f.v, f.ex);
  const bool edge = FWD ? lane == 31 : lane == 0;
  if (bo && edge) {
    BndT<V> o;
    o.v0 = FWD ? f.v[kSpl - 1] : f.v[0];
    o.v1 = FWD ? f.v[kSpl - 2] : f.v[1];
    o.ex = f.ex;
    o.pad = 0;
    *bo = o;
  }
}

template <class V>
__device__ __forceinline__ void lat_store_row(const LatState<V> &f, V *row, int *erow, int lane,
                                              bool live) {
#ifdef W2L_NO_ROW_STORES   // timing experiments only: results are wrong
  live = false;
#endif
  if (live) {
    stv(row + lane * kSpl, f.v);
    erow[lane] = f.ex;
  }
}

// Run a lattice warp over the whole utterance; its share of the recursion's
// total goes to sm.fin[w] (log domain) for the CTA epilogue.  Every step's
// lane values and exponents are stored (padding lanes excepted).
template <int KIND, bool FWD, class V, bool STREAM>
__device__ void lattice_run(ChainSm<V> &sm, const LatCtx &c, LatState<V> &f) {
  constexpr int kRing = Ring<V>::n;
  const int T = c.T, lane = c.lane;
  int *mycons = &sm.cons[c.cons_idx + c.w];
  const int up = FWD ? c.w - 1 : c.w + 1, dn = FWD ? c.w + 1 : c.w - 1;
  const bool has_up = up >= 0 && up < c.W, has_dn = dn >= 0 && dn < c.W;
  const int *upcons = &sm.cons[c.cons_idx + (has_up ? up : c.w)];
  const int *dncons = &sm.cons[c.cons_idx + (has_dn ? dn : c.w)];
  const BndT<V> *ubnd = has_up ? sm.bnd[up] : nullptr;
  BndT<V> *mybnd = sm.bnd[c.w];
  V *rows = reinterpret_cast<V *>(c.rows) + (size_t)c.w * c.Tmax * kLatStates;
  int *exps = c.exps + (size_t)c.w * c.Tmax * 32;
  auto row_of = [&](int t) { return rows + (size_t)t * kLatStates; };
  auto exp_of = [&](int t) { return exps + (size_t)t * 32; };

  // ---- step 0: initial values (criterion.py:123-125 / :194, :143-146 / :205-206)
#pragma unroll
  for (int k = 0; k < kSpl; ++k) f.v[k] = (V)0;
  f.ex = 0;
  const int base = (c.w * 32 + lane) * kSpl;
  const bool pad_lane = base >= c.nstates;   // padding states stay 0 (and are not stored)
  if (FWD) {
    wait_ge(&sm.prod, 1);
    const V *er = sm.ering[ring_slot<V>(true, 0)];
    if (base == 0) {
      f.v[0] = er[f.tok[0]];
      if (KIND == kCtc && c.nstates > 1) f.v[1] = er[f.tok[1]];
    }
  } else {
    const int S = c.nstates;
#pragma unroll
    for (int k = 0; k < kSpl; ++k) {
      const int s = base + k;
      f.v[k] = (s == S - 1 || (KIND == kCtc && s == S - 2)) ? (V)1 : (V)0;
    }
  }
  lane_renorm<kSpl, V>(f.v, f.ex);
  f.asc = (V)0;
  {
    const int t = frame_of(FWD, T, 0);
    lat_store_row(f, row_of(t), exp_of(t), lane, !pad_lane);
    if (FWD ? lane == 31 : lane == 0) {
      BndT<V> o;
      o.v0 = FWD ? f.v[kSpl - 1] : f.v[0];
      o.v1 = FWD ? f.v[kSpl - 2] : f.v[1];
      o.ex = f.ex;
      o.pad = 0;
      mybnd[0] = o;
    }
  }
  publish(mycons, 1, lane);

  // generic step (prologue 1..7 and the tail)
  auto generic = [&](int j) {
    wait_ge(&sm.prod, eidx_of(FWD, j) + 1);
    if (has_up) wait_ge(upcons, j);
    if (has_dn) wait_ge(dncons, j + 2 - kBndRing);
    StepIn<V> in;
    load_step_in<KIND, FWD, V>(in, f, sm.ering[j & (kRing - 1)],
                               has_up ? &ubnd[(j - 1) & (kBndRing - 1)] : nullptr, lane);
    lat_step<KIND, FWD, false, V>(f, in, &mybnd[j & (kBndRing - 1)], lane,
                                  (j % kRenormF) == 0 || j == T - 1, true);
    const int t = frame_of(FWD, T, j);
    lat_store_row(f, row_of(t), exp_of(t), lane, !pad_lane);
    publish(mycons, j + 1, lane);
  };
  const int pro_end = min(T, kBlk);
  for (int j = 1; j < pro_end; ++j) generic(j);

  // ---- full blocks of kBlk steps at j0 = 8 m
  const int nfull = T > kBlk ? (T - kBlk) / kBlk : 0;
  // Streamed gradient: the dependent gradient grid launches once every
  // warp of every chain CTA has passed the middle of its utterance, when
  // the first frames have both their rows -- its CTAs then do not hold SMs
  // while there is nothing to do (another criterion's kernels need them).
  const int mtrig = STREAM ? stream_trigger_block<KIND>(T) : -1;
#pragma unroll 1
  for (int m = 1; m <= nfull; ++m) {
    const int j0 = m * kBlk;
    wait3(&sm.prod, eidx_of(FWD, j0 + kBlk - 1) + 1, upcons, has_up ? j0 + kBlk - 1 : 0, dncons,
          has_dn ? j0 + kBlk + 1 - kBndRing : -kDone);
    const V *eb = sm.ering[j0 & (kRing - 1)];
    const BndT<V> *ub0 = has_up ? &ubnd[(j0 - 1) & (kBndRing - 1)] : nullptr;
    const BndT<V> *ub1 = has_up ? &ubnd[j0 & (kBndRing - 1)] : nullptr;   // q >= 1: ub1[q-1]
    BndT<V> *ob = has_dn ? &mybnd[j0 & (kBndRing - 1)] : nullptr;   // no reader: no store
    // rows go straight to global memory (fire-and-forget vector stores)
    const int tb = frame_of(FWD, T, j0);
    V *sv = row_of(tb);
    int *se = exp_of(tb);
    StepIn<V> in[kBlk];
#pragma unroll
    for (int q = 0; q < kBlk; ++q)
      load_step_in<KIND, FWD, V>(in[q], f, eb + q * kStride,
                                 q == 0 ? ub0 : (ub1 ? ub1 + (q - 1) : nullptr), lane);
    // every lane live (and the incoming boundary lane): exponents only move at
    // renormalisations from here on
    const bool fast = __all_sync(0xffffffffu, (f.ex != kNegExp || pad_lane) &&
                                                  (!(FWD ? lane == 0 : lane == 31) || !has_up ||
                                                   in[0].bex != kNegExp));
    auto run_block = [&](auto fast_tag) {
      constexpr bool FAST = decltype(fast_tag)::value;
#pragma unroll
      for (int q = 0; q < kBlk; ++q) {
        lat_step<KIND, FWD, FAST, V>(f, in[q], ob ? ob + q : nullptr, lane, (q % kRenormF) == 0,
                                     (q % kRenormF) == 1);
        const int dq = FWD ? q : -q;
        lat_store_row(f, sv + dq * kLatStates, se + dq * 32, lane, !pad_lane);
      }
    };
    if (fast)
      run_block(std::true_type{});
    else
      run_block(std::false_type{});
    publish(mycons, j0 + kBlk, lane);
    if (STREAM && m == mtrig) pdl_launch_dependents();
  }
  // ---- tail steps
  for (int j = max(pro_end, (nfull + 1) * kBlk); j < T; ++j) generic(j);
  if (STREAM && mtrig > nfull) pdl_launch_dependents();
  publish(mycons, kDone, lane);

  // ---- totals (criterion.py:136-141 CTC, :203 fac forward; backward: the
  // frame-0 emissions times beta'_0)
  const double ln2 = 0.6931471805599453;
  double part = 0.0;
  if (FWD) {
    const int S = c.nstates;
#pragma unroll
    for (int k = 0; k < kSpl; ++k) {
      const int s = base + k;
      if (s == S - 1 || (KIND == kCtc && s == S - 2)) part += (double)f.v[k];
    }
  } else {
    wait_ge(&sm.prod, T);   // frame 0's Et (the last step only waited for T - 1)
    const V *er = sm.ering[ring_slot<V>(false, T - 1)];   // frame 0
    if (base == 0) {
      part = (double)er[f.tok[0]] * (double)f.v[0];
      if (KIND == kCtc && c.nstates > 1) part += (double)er[f.tok[1]] * (double)f.v[1];
    }
  }
  const double lp = part > 0.0 ? log(part) + (double)f.ex * ln2 : -CUDART_INF;
  const double m = warp_max(lp);
  const double sum = warp_sum(lp > -CUDART_INF ? exp(lp - m) : 0.0);
  if (lane == 0) sm.fin[c.w] = isfinite(m) ? m + log(sum) : -CUDART_INF;
}

// combine the per-warp totals (log domain) after a CTA barrier
template <class V>
__device__ __forceinline__ double lattice_total(const ChainSm<V> &sm, int W) {
  double m = -CUDART_INF;
  for (int w = 0; w < W; ++w) m = fmax(m, sm.fin[w]);
  if (!isfinite(m)) return -CUDART_INF;
  double s = 0.0;
  for (int w = 0; w < W; ++w) s += sm.fin[w] > -CUDART_INF ? exp(sm.fin[w] - m) : 0.0;
  return m + log(s);
}

__host__ __device__ inline int lat_warps(int nstates) {
  return nstates <= 0 ? 1 : (nstates + kLatStates - 1) / kLatStates;
}

// 2^x for an integer x, clamped to the type's range (0 below)
template <class V>
__device__ __forceinline__ V pow2_clamped(int x) {
  return Pow2<V>::p2(max(min(x, Pow2<V>::kMaxExp), -Pow2<V>::kMaxExp));
}

}  // namespace w2l
