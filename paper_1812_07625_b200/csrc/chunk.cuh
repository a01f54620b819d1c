// Warp-private emission staging for the serial recursions.
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

struct EmissionPipe {
  float *buf;        // [2][kChunk][stride] shared memory
  const float *e;    // &em[b][0][0]
  int T, N, stride, lane;
  bool fwd;
  int cur;           // chunk resident in buf[cur & 1], -1 before the first
  double shift_sum;  // sum of this lane's row maxima (CTC loss offset)

  __device__ void init(float *smem, const float *e_, int T_, int N_, bool fwd_) {
    buf = smem;
    e = e_;
    T = T_;
    N = N_;
    stride = em_stride(N_);
    lane = threadIdx.x & 31;
    fwd = fwd_;
    cur = -1;
    shift_sum = 0.0;
    issue(fwd ? 0 : (T - 1) / kChunk);
  }

  __device__ void issue(int c) {
    const int t0 = c * kChunk;
    const int rows = min(kChunk, T - t0);
    float *dst = buf + (c & 1) * kChunk * stride;
    if (lane < N)
      for (int r = 0; r < rows; ++r)
        cp_async4(dst + r * stride + lane, e + (size_t)(t0 + r) * N + lane);
    cp_async_commit();
  }

  // make chunk c (the next one in walk order) resident and converted
  __device__ void advance(int c) {
    cp_async_wait<0>();
    __syncwarp();
    const int t0 = c * kChunk;
    const int rows = min(kChunk, T - t0);
    float *rb = buf + (c & 1) * kChunk * stride;
    if (lane < rows) {
      float *r = rb + lane * stride;
      float m = -CUDART_INF_F;
      for (int i = 0; i < N; ++i) m = fmaxf(m, r[i]);
      for (int i = 0; i < N; ++i) r[i] = expf(r[i] - m);
      r[N] = 0.f;
      shift_sum += (double)m;
    }
    __syncwarp();
    const int nxt = fwd ? c + 1 : c - 1;
    if (nxt >= 0 && nxt * kChunk < T) issue(nxt);
    cur = c;
  }

  // shared-memory row of Et for frame t (frames must be requested in walk order)
  __device__ __forceinline__ const float *row(int t) {
    const int c = t / kChunk;
    if (c != cur) advance(c);
    return buf + (c & 1) * kChunk * stride + (t - c * kChunk) * stride;
  }
};

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
template <int SPL>
__device__ __forceinline__ void lane_renorm(float (&v)[SPL], int &ex) {
  float mx = 0.f;
#pragma unroll
  for (int k = 0; k < SPL; ++k) mx = fmaxf(mx, v[k]);
  if (mx > 0.f) {
    const int kx = exponent_of(mx);
    const float sc = pow2f(-kx);
#pragma unroll
    for (int k = 0; k < SPL; ++k) v[k] *= sc;
    ex += kx;
  } else {
    ex = kNegExp;
  }
}

// one frame's chain row, slot-major ([k][lane]) so every store is coalesced
template <int SPL>
__device__ __forceinline__ void lane_store(const float (&v)[SPL], int ex, float *out, int *oute,
                                           int lp, int lane, int t) {
  float *o = out + t * lp + lane;
#pragma unroll
  for (int k = 0; k < SPL; ++k) o[k * 32] = v[k];
  oute[t * 32 + lane] = ex;
}

}  // namespace w2l
