// Microbenchmark of the fcc recursion step (asg_fast.cu fcc_alpha_step) in one
// warp: v' = e (.) (M v), the vector exchanged between steps through shared
// memory (variant 0, the kernel's), 64-bit loads (1), shuffles (2), or not
// exchanged at all (3: the FMA-chain latency alone).  Prints cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fcc_probe tools/fcc_probe.cu
#include <cstdio>

template <int V>
__global__ void fcc_probe(float *out, long long *cyc, int steps) {
  __shared__ __align__(16) float vec[2][32];
  const int lane = threadIdx.x;
  float m[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // V 6: m rotated by float4 blocks, V 7: rotated by elements
    const int jj = V == 6 ? (4 * (((j >> 2) + lane) & 7) + (j & 3)) : (V == 7 ? ((j + lane) & 31) : j);
    m[j] = 0.03f * ((lane * 7 + jj * 3) % 11);
  }
  float v = 1.f;
  vec[0][lane] = v;
  __syncwarp();
  const long long t0 = clock64();
  for (int t = 1; t < steps; ++t) {
    const int par = t & 1;
    float acc[8];
    if (V == 0 || V == 4) {
      const float4 *pv = reinterpret_cast<const float4 *>(vec[par ^ 1]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x = pv[q];
        acc[q] = m[4 * q] * x.x;
        acc[q] = fmaf(m[4 * q + 1], x.y, acc[q]);
        acc[q] = fmaf(m[4 * q + 2], x.z, acc[q]);
        acc[q] = fmaf(m[4 * q + 3], x.w, acc[q]);
      }
    } else if (V == 1) {
      const float2 *pv = reinterpret_cast<const float2 *>(vec[par ^ 1]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 x = pv[2 * q], y = pv[2 * q + 1];
        acc[q] = m[4 * q] * x.x;
        acc[q] = fmaf(m[4 * q + 1], x.y, acc[q]);
        acc[q] = fmaf(m[4 * q + 2], y.x, acc[q]);
        acc[q] = fmaf(m[4 * q + 3], y.y, acc[q]);
      }
    } else if (V == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q] = m[4 * q] * __shfl_sync(0xffffffffu, v, 4 * q);
        acc[q] = fmaf(m[4 * q + 1], __shfl_sync(0xffffffffu, v, 4 * q + 1), acc[q]);
        acc[q] = fmaf(m[4 * q + 2], __shfl_sync(0xffffffffu, v, 4 * q + 2), acc[q]);
        acc[q] = fmaf(m[4 * q + 3], __shfl_sync(0xffffffffu, v, 4 * q + 3), acc[q]);
      }
    } else if (V == 6) {
      const float4 *pv = reinterpret_cast<const float4 *>(vec[par ^ 1]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x = pv[(q + lane) & 7];
        acc[q] = m[4 * q] * x.x;
        acc[q] = fmaf(m[4 * q + 1], x.y, acc[q]);
        acc[q] = fmaf(m[4 * q + 2], x.z, acc[q]);
        acc[q] = fmaf(m[4 * q + 3], x.w, acc[q]);
      }
    } else if (V == 7) {
      const float *pv = vec[par ^ 1];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q] = m[4 * q] * pv[(4 * q + lane) & 31];
        acc[q] = fmaf(m[4 * q + 1], pv[(4 * q + 1 + lane) & 31], acc[q]);
        acc[q] = fmaf(m[4 * q + 2], pv[(4 * q + 2 + lane) & 31], acc[q]);
        acc[q] = fmaf(m[4 * q + 3], pv[(4 * q + 3 + lane) & 31], acc[q]);
      }
    } else if (V == 5) {
      const float x = vec[par ^ 1][lane];   // own slot only: bare store->load round trip
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q] = m[4 * q] * x;
        acc[q] = fmaf(m[4 * q + 1], x, acc[q]);
        acc[q] = fmaf(m[4 * q + 2], x, acc[q]);
        acc[q] = fmaf(m[4 * q + 3], x, acc[q]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q] = m[4 * q] * v;
        acc[q] = fmaf(m[4 * q + 1], v, acc[q]);
        acc[q] = fmaf(m[4 * q + 2], v, acc[q]);
        acc[q] = fmaf(m[4 * q + 3], v, acc[q]);
      }
    }
    const float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    v = s * 0.5f;
    if (V <= 1 || V >= 5) {
      vec[par][lane] = v;
      __syncwarp();
    } else if (V == 4) {
      vec[par][lane] = v;   // no __syncwarp (converged warp, in-order shared memory)
    }
  }
  const long long t1 = clock64();
  out[lane] = v;
  if (lane == 0) *cyc = t1 - t0;
}

// two warps: warp w sums columns [16w, 16w+16) of row `lane`; partial sums
// cross through shared memory behind a 64-thread named barrier; each warp
// keeps its own copy of the new vector (no second barrier)
__global__ void fcc_probe2(float *out, long long *cyc, int steps) {
  __shared__ __align__(16) float vbuf[2][32];     // per-warp copy of v
  __shared__ float part[2][2][32];                // [parity][warp][row]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float m[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) m[j] = 0.03f * ((lane * 7 + (16 * w + j) * 3) % 11);
  float v = 1.f;
  vbuf[w][lane] = v;
  __syncwarp();
  const long long t0 = clock64();
  for (int t = 1; t < steps; ++t) {
    const float4 *pv = reinterpret_cast<const float4 *>(vbuf[w]) + 4 * w;
    float acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 x = pv[q];
      acc[q] = m[4 * q] * x.x;
      acc[q] = fmaf(m[4 * q + 1], x.y, acc[q]);
      acc[q] = fmaf(m[4 * q + 2], x.z, acc[q]);
      acc[q] = fmaf(m[4 * q + 3], x.w, acc[q]);
    }
    const float sw = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    part[t & 1][w][lane] = sw;
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const float so = part[t & 1][w ^ 1][lane];
    v = (w == 0 ? sw + so : so + sw) * 0.5f;       // same order in both warps
    vbuf[w][lane] = v;
    __syncwarp();
  }
  const long long t1 = clock64();
  if (w == 0) out[lane] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float *out;
  long long *cyc, h;
  cudaMalloc(&out, 32 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  const int steps = 1600;
  const char *names[] = {"smem LDS.128 broadcast (kernel)", "smem LDS.64", "shuffles",
                         "no exchange (FMA chain only)", "LDS.128 broadcast, no syncwarp",
                         "own slot STS->LDS round trip", "rotated LDS.128 (conflict-free)",
                         "rotated LDS.32 x32"};
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 8; ++v) {
      if (v == 0) fcc_probe<0><<<1, 32>>>(out, cyc, steps);
      if (v == 1) fcc_probe<1><<<1, 32>>>(out, cyc, steps);
      if (v == 2) fcc_probe<2><<<1, 32>>>(out, cyc, steps);
      if (v == 3) fcc_probe<3><<<1, 32>>>(out, cyc, steps);
      if (v == 4) fcc_probe<4><<<1, 32>>>(out, cyc, steps);
      if (v == 5) fcc_probe<5><<<1, 32>>>(out, cyc, steps);
      if (v == 6) fcc_probe<6><<<1, 32>>>(out, cyc, steps);
      if (v == 7) fcc_probe<7><<<1, 32>>>(out, cyc, steps);
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep) printf("%-34s %6.1f cycles/step\n", names[v], (double)h / (steps - 1));
    }
  for (int rep = 0; rep < 2; ++rep) {
    fcc_probe2<<<1, 64>>>(out, cyc, steps);
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    if (rep) printf("%-34s %6.1f cycles/step\n", "two warps, named barrier", (double)h / (steps - 1));
  }
  return 0;
}
