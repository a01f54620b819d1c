// Dependent-chain latency microbenchmarks (one warp): cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *outd, float *outf, long long *cyc, int n) {
  double d = threadIdx.x * 1e-3 + 1.0, e = 1.0000001;
  float f = threadIdx.x * 1e-3f + 1.f;
  int iv = threadIdx.x;
  __shared__ float sm[1024];
  sm[threadIdx.x] = (float)threadIdx.x;
  __syncwarp();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = fma(d, e, 1e-9); d = fma(d, e, 1e-9); d = fma(d, e, 1e-9); d = fma(d, e, 1e-9); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4 * n);
  // DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = d + e; d = d + e; d = d + e; d = d + e; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / (4 * n);
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = d * e; d = d * e; d = d * e; d = d * e; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / (4 * n);
  // FFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) { f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / (4 * n);
  // SHFL float
  t0 = clock64();
  for (int i = 0; i < n; ++i) { f = __shfl_up_sync(~0u, f, 1); f = __shfl_up_sync(~0u, f, 1); f = __shfl_up_sync(~0u, f, 1); f = __shfl_up_sync(~0u, f, 1); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / (4 * n);
  // SHFL double
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / (4 * n);
  // LDS dependent
  t0 = clock64();
  for (int i = 0; i < n; ++i) { iv = (int)sm[iv & 1023]; iv = (int)sm[iv & 1023]; iv = (int)sm[iv & 1023]; iv = (int)sm[iv & 1023]; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / (4 * n);
  // double -> float conversion chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { f = (float)((double)f * e); f = (float)((double)f * e); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / (2 * n);
  // FFMA2 packed
  float2 p = make_float2(f, f + 1.f);
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&p) : "l"(0x3f8000003f800000ull), "l"(0x3f8000003f800000ull));
    asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*(unsigned long long*)&p) : "l"(0x3f8000003f800000ull), "l"(0x3f8000003f800000ull));
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) / (2 * n);
  // DFMA throughput: 8 independent chains, one warp
  double a0=d,a1=d+1,a2=d+2,a3=d+3,a4=d+4,a5=d+5,a6=d+6,a7=d+7;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a0=fma(a0,e,1e-9);a1=fma(a1,e,1e-9);a2=fma(a2,e,1e-9);a3=fma(a3,e,1e-9);a4=fma(a4,e,1e-9);a5=fma(a5,e,1e-9);a6=fma(a6,e,1e-9);a7=fma(a7,e,1e-9); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[9] = (t1 - t0) * 100 / (8 * n);
  d += a0+a1+a2+a3+a4+a5+a6+a7;
  outd[threadIdx.x] = d + iv;
  outf[threadIdx.x] = f + p.x + p.y;
}
int main() {
  double *od; float *of; long long *c;
  cudaMalloc(&od, 256); cudaMalloc(&of, 128); cudaMallocManaged(&c, 16 * 8);
  k<<<1, 32>>>(od, of, c, 1000);
  k<<<1, 32>>>(od, of, c, 1000);
  cudaDeviceSynchronize();
  const char *names[] = {"DFMA", "DADD", "DMUL", "FFMA", "SHFL32", "SHFL64", "LDS", "F2F d->f (+DMUL)", "FFMA2", "DFMA issue x100"};
  for (int i = 0; i < 10; ++i) printf("%-18s %lld cyc\n", names[i], c[i]);
  return 0;
}
