// Warp-private emission staging and block-floating-point helpers for the
// serial recursions.
//
// A chain warp walks an utterance frame by frame (forward or backward).  Its
// emissions are staged kChunk frames at a time into shared memory with
// cp.async (LDGSTS, one chunk in flight while the previous one is consumed)
// and converted in place to  Et[t][i] = exp(e[t][i] - max_i e[t][i]),
// the per-frame shifted emission probabilities of the scaled linear-domain
// recursions.  Column N of every staged row holds 0 so that padding states
// (token id N) read a zero emission.  Et is bit-identical to the values the
// gradient kernels recompute (same max, same expf).
#pragma once

#include "common.cuh"

namespace w2l {

constexpr int kRenorm = 4;   // frames between lane renormalisations
constexpr int kStride = 33;  // staged row pitch: odd (conflict-free per-lane rows), > 32
constexpr int kUnroll = 8;   // frames per fully unrolled block (immediate smem offsets)

struct ChainCtx {
  const float *trans;
  const float *e;  // &em[b][0][0]
  int N, T, lane;
  float amax;
};

__device__ __forceinline__ void stage_issue(float *dst, const ChainCtx &c, int t0) {
  const int rows = min(kChunk, c.T - t0);
  if (c.lane < c.N)
    for (int r = 0; r < rows; ++r)
      cp_async4(dst + r * kStride + c.lane, c.e + (size_t)(t0 + r) * c.N + c.lane);
  cp_async_commit();
}

// wait for the staged chunk, convert it to Et in place (lane r owns row r)
// and zero columns N..32 (padding states and idle lanes read 0); the row
// maxima are summed into *shift_sum (the CTC loss offset) if given
__device__ __forceinline__ void stage_convert(float *buf, const ChainCtx &c, int rows,
                                              double *shift_sum = nullptr) {
  cp_async_wait<0>();
  __syncwarp();
  if (c.lane < rows) {
    float *r = buf + c.lane * kStride;
    float m = -CUDART_INF_F;
    for (int i = 0; i < c.N; ++i) m = fmaxf(m, r[i]);
    for (int i = 0; i < c.N; ++i) r[i] = expf(r[i] - m);
    for (int i = c.N; i < kStride; ++i) r[i] = 0.f;
    if (shift_sum) *shift_sum += (double)m;
  }
  __syncwarp();
}

// The same per-frame shift and conversion, computed by a whole warp for one
// frame (lane i < N holds token i): used by the gradient kernels.
__device__ __forceinline__ float shifted_prob(const float *erow, int N, int lane, float *shift) {
  const float v = lane < N ? erow[lane] : -CUDART_INF_F;
  float m = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (shift) *shift = m;
  return lane < N ? expf(v - m) : 0.f;
}

// Block floating point for a lane's SPL consecutive chain states: scale them
// so the largest lies in [1, 2) and fold the power of two into the lane
// exponent (an all-zero lane is marked dead with kNegExp).
// max over a register array as a balanced tree (depth log2 SPL, not SPL)
template <int SPL>
__device__ __forceinline__ float tree_max(const float (&v)[SPL]) {
  float m[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) m[k] = v[k];
#pragma unroll
  for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < SPL; k += 2 * w) m[k] = fmaxf(m[k], m[k + w]);
  return fmaxf(m[0], 0.f);
}

template <int SPL>
__device__ __forceinline__ void lane_renorm(float (&v)[SPL], int &ex) {
  const float mx = tree_max<SPL>(v);
  // branch-free: an all-zero block keeps zeros and is marked dead
  const int kx = exponent_of(mx);           // -127 for mx == 0
  const float sc = pow2f_fast(-kx);
#pragma unroll
  for (int k = 0; k < SPL; ++k) v[k] *= sc;
  ex = mx > 0.f ? ex + kx : kNegExp;
}

// one frame's chain row, lane-major ([lane][k]): SPL is even, so a lane's
// states go out as SPL/2 8-byte stores
template <int SPL>
__device__ __forceinline__ void lane_store(const float (&v)[SPL], int ex, float *out, int *oute,
                                           int lane, int t) {
  static_assert(SPL % 2 == 0, "SPL must be even");
  constexpr int lp = SPL * 32;
  float2 *o = reinterpret_cast<float2 *>(out + t * lp + lane * SPL);
#pragma unroll
  for (int k = 0; k < SPL / 2; ++k) o[k] = make_float2(v[2 * k], v[2 * k + 1]);
  oute[t * 32 + lane] = ex;
}

template <int SPL>
__device__ __forceinline__ void lane_load(float (&v)[SPL], const float *row, int lane) {
  const float2 *o = reinterpret_cast<const float2 *>(row + lane * SPL);
#pragma unroll
  for (int k = 0; k < SPL / 2; ++k) {
    const float2 x = o[k];
    v[2 * k] = x.x;
    v[2 * k + 1] = x.y;
  }
}

// align the neighbour lane's value to this lane's exponent.  kCheck: the
// full version -- if the neighbour dominates by more than 2^64, rebase this
// lane onto it first (a branch).  Lane exponents only move at
// renormalisation steps, so the unrolled blocks run the full version on the
// step after each renormalisation and the branch-free one elsewhere (a dead
// lane adopts the neighbour's exponent; the shift is clamped to 2^126).
template <int SPL>
__device__ __forceinline__ float align_neighbour(float nb, int nbe, float (&v)[SPL], int &ex,
                                                 bool check) {
  if (check) {
    int dd = nbe - ex;
    if (dd > 64) {
      const float sc = pow2f(-dd);
#pragma unroll
      for (int k = 0; k < SPL; ++k) v[k] *= sc;
      ex = nbe;
      dd = 0;
    }
    return nb * pow2f_fast(dd);
  }
  ex = ex == kNegExp ? nbe : ex;
  return nb * pow2f_fast(min(nbe - ex, 126));
}

// The same alignment, returning the power-of-two factor for the neighbour's
// values (it stays valid until the next renormalisation or adoption).
template <int SPL>
__device__ __forceinline__ float align_factor(int nbe, float (&v)[SPL], int &ex, bool check) {
  if (check) {
    int dd = nbe - ex;
    if (dd > 64) {
      const float sc = pow2f_fast(max(-dd, -127));
#pragma unroll
      for (int k = 0; k < SPL; ++k) v[k] *= sc;
      ex = nbe;
      dd = 0;
    }
    return pow2f_fast(dd);
  }
  ex = ex == kNegExp ? nbe : ex;
  return pow2f_fast(min(nbe - ex, 126));
}

// floor(log2(max_k a[k] b[k])) + ea + eb, a bound on this lane's largest
// alpha*beta product (kNegExp if either side is dead or all-zero)
template <int SPL>
__device__ __forceinline__ int lane_pair_exponent(const float (&a)[SPL], const float (&b)[SPL],
                                                  int ea, int eb) {
  float p[SPL];
#pragma unroll
  for (int k = 0; k < SPL; ++k) p[k] = a[k] * b[k];
  const float m = tree_max<SPL>(p);
  if (!(m > 0.f) || ea <= kNegExp / 2 || eb <= kNegExp / 2) return kNegExp;
  return ea + eb + exponent_of(m);
}

// ---- TMA bulk stores of staged chain rows (smem -> global, async proxy).
// Chain warps write each block of kUnroll frame rows into a shared-memory
// staging slot and one lane hands the contiguous block to the bulk-copy
// engine, so the serial recursion never waits on the LSU store path.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_fence() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// double-buffered staging for kUnroll rows of kRowFloats values + kRowInts ints
template <int kRowFloats, int kRowInts>
struct RowStage {
  float v[2][kUnroll * kRowFloats];
  int e[2][kUnroll * kRowInts];
};

// before writing slot (gi & 1): its previous bulk copy must have read it
__device__ __forceinline__ void stage_acquire(int gi, int lane) {
  if (gi >= 2 && lane == 0) bulk_wait_read1();
  __syncwarp();
}

// hand the finished slot to the bulk engine
template <int kRowFloats, int kRowInts>
__device__ __forceinline__ void stage_release(RowStage<kRowFloats, kRowInts> &st, int slot,
                                              float *gv, int *ge, int lane) {
  static_assert((kUnroll * kRowInts * sizeof(int)) % 16 == 0, "bulk copies move 16B multiples");
  bulk_fence();
  __syncwarp();
  if (lane == 0) {
    bulk_store(gv, st.v[slot], kUnroll * kRowFloats * sizeof(float));
    bulk_store(ge, st.e[slot], kUnroll * kRowInts * sizeof(int));
    bulk_commit();
  }
}

__device__ __forceinline__ void stage_drain(int lane) {
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// ---- mbarrier / named-barrier primitives (producer -> consumer rings)
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void named_barrier(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
// make completed bulk (async-proxy) global writes visible to generic loads
__device__ __forceinline__ void bulk_publish() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  __threadfence_block();
}

}  // namespace w2l
