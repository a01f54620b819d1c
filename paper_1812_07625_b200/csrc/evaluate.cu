// Batched greedy evaluation: the reference's evaluate loop
// (trainer.py:465-514) per utterance on the device -- collapse the Viterbi
// path (criterion.py:287-310), then the token edit distance to the target
// and the word edit distance over silence-delimited token groups
// (lexicon.py:182-195).
//
// One CTA per utterance.  The collapse is a stream compaction (keep a frame
// when it starts a run and, for CTC, is not the blank; ASG expands the
// repetition token into its predecessor).  Each Levenshtein distance is
// computed row by row: with prev the previous row,
//   tmp[j] = min(prev[j] + 1, prev[j-1] + (r_i != h_j)),
//   cur[j] = min_{k <= j} (tmp[k] + (j - k))      (the insertions)
// so a row is one parallel step plus a block prefix-min of tmp[k] - k.
// Words are compared by content (length and tokens), not by hash.

#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kEvThreads = 256;
constexpr int kEvWarps = kEvThreads / 32;

// exclusive block sum of v; returns the total (sbuf: kEvWarps + 1 ints)
__device__ __forceinline__ int block_excl_sum(int v, int &excl, int *sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sbuf[warp] = x;
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < kEvWarps; ++w) {
    if (w < warp) base += sbuf[w];
    tot += sbuf[w];
  }
  excl = base + x - v;
  __syncthreads();
  return tot;
}

// inclusive block prefix-min of v (in thread order); *last = the block min
__device__ __forceinline__ int block_incl_min(int v, int *sbuf, int &last) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = min(x, y);
  }
  if (lane == 31) sbuf[warp] = x;
  __syncthreads();
  int pre = INT_MAX, all = INT_MAX;
  for (int w = 0; w < kEvWarps; ++w) {
    if (w < warp) pre = min(pre, sbuf[w]);
    all = min(all, sbuf[w]);
  }
  last = all;
  __syncthreads();
  return min(pre, x);
}

// Levenshtein distance between sequences of n_r and n_h items; eq(i, j)
// tells whether ref item i equals hyp item j.  prev / cur: n_h + 1 ints each.
template <class Eq>
__device__ int block_edit_distance(int n_r, int n_h, Eq eq, int *prev, int *cur, int *sbuf) {
  if (n_r == 0) return n_h;
  for (int j = threadIdx.x; j <= n_h; j += kEvThreads) prev[j] = j;
  __syncthreads();
  for (int i = 1; i <= n_r; ++i) {
    int carry = INT_MAX;   // prefix min of the chunks before
    for (int j0 = 0; j0 <= n_h; j0 += kEvThreads) {
      const int j = j0 + threadIdx.x;
      int v = INT_MAX;
      if (j <= n_h) {
        const int tmp = j == 0 ? i : min(prev[j] + 1, prev[j - 1] + (eq(i - 1, j - 1) ? 0 : 1));
        v = tmp - j;
      }
      int last;
      const int pm = min(block_incl_min(v, sbuf, last), carry);
      if (j <= n_h) cur[j] = j + pm;
      carry = min(carry, last);
    }
    __syncthreads();
    int *t = prev;
    prev = cur;
    cur = t;
  }
  return prev[n_h];
}

// starts and lengths of the silence-free groups of seq[0 .. n) (empty groups
// dropped); silence < 0: the whole sequence is one group, even when empty
__device__ int block_groups(const int *seq, int n, int silence, int *gstart, int *glen,
                            int *sbuf) {
  if (silence < 0) {
    if (threadIdx.x == 0) {
      gstart[0] = 0;
      glen[0] = n;
    }
    __syncthreads();
    return 1;
  }
  int ng = 0;
  for (int k0 = 0; k0 < n; k0 += kEvThreads) {
    const int k = k0 + threadIdx.x;
    const bool start = k < n && seq[k] != silence && (k == 0 || seq[k - 1] == silence);
    int excl;
    const int tot = block_excl_sum(start ? 1 : 0, excl, sbuf);
    if (start) {
      int e = k;
      while (e + 1 < n && seq[e + 1] != silence) ++e;
      gstart[ng + excl] = k;
      glen[ng + excl] = e - k + 1;
    }
    ng += tot;
  }
  __syncthreads();
  return ng;
}

__global__ void __launch_bounds__(kEvThreads)
    greedy_eval_kernel(const int64_t *__restrict__ path, const int32_t *__restrict__ path_len,
                       int B, int Tmax, int kind, int special, const int64_t *__restrict__ ref,
                       const int32_t *__restrict__ ref_len, int Lmax, int silence,
                       int64_t *__restrict__ hyp, int32_t *__restrict__ hyp_len,
                       int32_t *__restrict__ tok_dist, int32_t *__restrict__ word_dist,
                       int32_t *__restrict__ ref_words, int32_t *__restrict__ status) {
  extern __shared__ int esm[];
  __shared__ int sbuf[kEvWarps + 1];
  __shared__ int s_bad;
  const int b = blockIdx.x;
  // shared layout: htok[Tmax] rtok[Lmax] prev[Tmax+2] cur[Tmax+2]
  //                hgs[Tmax] hgl[Tmax] rgs[Lmax] rgl[Lmax]
  int *htok = esm, *rtok = htok + Tmax, *prev = rtok + Lmax, *cur = prev + Tmax + 2;
  int *hgs = cur + Tmax + 2, *hgl = hgs + Tmax, *rgs = hgl + Tmax, *rgl = rgs + Lmax;
  const int T = path_len[b], L = ref_len[b];
  if (threadIdx.x == 0) s_bad = (T < 0 || T > Tmax || L < 0 || L > Lmax) ? 1 : 0;
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) {
      status[b] = W2L_ERR_CONTRACT;
      hyp_len[b] = tok_dist[b] = word_dist[b] = ref_words[b] = 0;
    }
    return;
  }
  const int64_t *p = path + (size_t)b * Tmax;
  // ---- collapse (criterion.py:287-310)
  int H = 0;
  for (int t0 = 0; t0 < T; t0 += kEvThreads) {
    const int t = t0 + threadIdx.x;
    const int pt = t < T ? (int)p[t] : -1;
    const int pp = (t > 0 && t < T) ? (int)p[t - 1] : -1;
    bool keep = t < T && (t == 0 || pt != pp);
    int tok = pt;
    if (kind == 1) {                       // CTC: the blank leaves
      keep = keep && pt != special;
    } else if (special >= 0 && pt == special && keep) {   // ASG: the repetition token
      if (t == 0) atomicOr(&s_bad, 1);     // "repetition token with no preceding token"
      tok = pp;                            // = its predecessor in the deduplicated path
    }
    int excl;
    const int tot = block_excl_sum(keep ? 1 : 0, excl, sbuf);
    if (keep) {
      htok[H + excl] = tok;
      hyp[(size_t)b * Tmax + H + excl] = tok;
    }
    H += tot;
  }
  for (int k = H + threadIdx.x; k < Tmax; k += kEvThreads) hyp[(size_t)b * Tmax + k] = -1;
  for (int l = threadIdx.x; l < L; l += kEvThreads) rtok[l] = (int)ref[(size_t)b * Lmax + l];
  __syncthreads();
  // ---- token edit distance (trainer.py:465-476, 503-504)
  const int td = block_edit_distance(
      L, H, [&](int i, int j) { return rtok[i] == htok[j]; }, prev, cur, sbuf);
  // ---- word edit distance over silence-delimited groups (trainer.py:505-510)
  const int nr = block_groups(rtok, L, silence, rgs, rgl, sbuf);
  const int nh = block_groups(htok, H, silence, hgs, hgl, sbuf);
  auto word_eq = [&](int i, int j) {
    if (rgl[i] != hgl[j]) return false;
    for (int k = 0; k < rgl[i]; ++k)
      if (rtok[rgs[i] + k] != htok[hgs[j] + k]) return false;
    return true;
  };
  const int wd = block_edit_distance(nr, nh, word_eq, prev, cur, sbuf);
  if (threadIdx.x == 0) {
    hyp_len[b] = H;
    tok_dist[b] = td;
    word_dist[b] = wd;
    ref_words[b] = nr;
    status[b] = s_bad ? W2L_ERR_CONTRACT : W2L_OK;
  }
}

}  // namespace

size_t greedy_eval_smem_bytes(int Tmax, int Lmax) {
  return sizeof(int) * ((size_t)Tmax * 5 + 4 + (size_t)Lmax * 3);
}

cudaError_t launch_greedy_eval(const int64_t *path, const int32_t *path_len, int B, int Tmax,
                               int kind, int special, const int64_t *ref, const int32_t *ref_len,
                               int Lmax, int silence, int64_t *hyp, int32_t *hyp_len,
                               int32_t *tok_dist, int32_t *word_dist, int32_t *ref_words,
                               int32_t *status, cudaStream_t s) {
  const size_t smem = greedy_eval_smem_bytes(Tmax, Lmax);
  cudaError_t err = cudaFuncSetAttribute(greedy_eval_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  greedy_eval_kernel<<<B, kEvThreads, smem, s>>>(path, path_len, B, Tmax, kind, special, ref,
                                                 ref_len, Lmax, silence, hyp, hyp_len, tok_dist,
                                                 word_dist, ref_words, status);
  return cudaGetLastError();
}

}  // namespace w2l
