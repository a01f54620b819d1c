// Microbenchmark of the fac lattice step (lattice.cuh lat_step, forward,
// 4 states per lane) in one warp: v[k] = E[k] (S v[k] + P v[k-1]), state 0
// taking the previous lane's last state through a shuffle (variant 0), or
// through shared memory (1), or not at all (2: the lane-local chain alone).
// Prints cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_step_probe tools/lat_step_probe.cu
#include <cstdio>

template <int V>
__global__ void lat_probe(float *out, long long *cyc, int steps) {
  __shared__ float xch[2][32];
  const int lane = threadIdx.x;
  float v[4] = {1.f, 0.5f, 0.25f, 0.125f};
  const float S = 0.6f, P = 0.3f;
  float E[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) E[k] = 0.9f + 0.01f * ((lane + k) % 7);
  const long long t0 = clock64();
  for (int t = 1; t < steps; ++t) {
    float nb;
    if (V == 0) {
      nb = __shfl_up_sync(0xffffffffu, v[3], 1);
    } else if (V == 1) {
      xch[t & 1][lane] = v[3];
      __syncwarp();
      nb = xch[t & 1][(lane + 31) & 31];
    } else {
      nb = v[3];
    }
    if (lane == 0) nb = 0.f;
#pragma unroll
    for (int k = 3; k >= 1; --k) v[k] = E[k] * fmaf(S, v[k], P * v[k - 1]);
    v[0] = E[0] * fmaf(S, v[0], P * nb);
    if ((t & 3) == 0) {   // renormalise every 4 steps (power of two from the max)
      const float mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
      const int e = ((__float_as_int(mx) >> 23) & 0xff) - 127;
      const float sc = __int_as_float((127 - e) << 23);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] *= sc;
    }
  }
  const long long t1 = clock64();
  out[lane] = v[0] + v[1] + v[2] + v[3];
  if (lane == 0) *cyc = t1 - t0;
}

int main() {
  float *out;
  long long *cyc, h;
  cudaMalloc(&out, 32 * sizeof(float));
  cudaMalloc(&cyc, sizeof(long long));
  const int steps = 1600;
  const char *names[] = {"neighbour via shuffle (kernel)", "neighbour via shared memory",
                         "no neighbour (lane-local chain)"};
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 3; ++v) {
      if (v == 0) lat_probe<0><<<1, 32>>>(out, cyc, steps);
      if (v == 1) lat_probe<1><<<1, 32>>>(out, cyc, steps);
      if (v == 2) lat_probe<2><<<1, 32>>>(out, cyc, steps);
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep) printf("%-34s %6.1f cycles/step\n", names[v], (double)h / (steps - 1));
    }
  return 0;
}
