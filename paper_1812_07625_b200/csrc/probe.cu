// Microbenchmarks for the roofline denominators that MEASURED_PEAKS.json
// does not carry: MUFU ex2 throughput (the SFU bound the SURVEY uses for the
// log-semiring work), FP64 add throughput (Viterbi) and FP32 FMA throughput
// (the scaled linear-domain recursions).  Each kernel runs independent
// dependency chains so the pipe, not latency, is the limit.
#include "common.cuh"
#include "kernels.h"

namespace w2l {
namespace {

constexpr int kIters = 2048;
constexpr int kChains = 8;

__global__ void mufu_probe(float *sink, float seed) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed * (threadIdx.x + c) * 1e-6f - 1.f;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) sink[0] = s;
}

__global__ void dadd_probe(double *sink, double seed) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed + threadIdx.x + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[c]) : "d"(seed));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) sink[0] = s;
}

__global__ void ffma_probe(float *sink, float seed) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed + threadIdx.x + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x[c]) : "f"(seed));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) sink[0] = s;
}

template <class F>
double time_ops(F launch, double ops) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ops * 5 / (ms * 1e-3);
}

}  // namespace

int probe_peaks(double *mufu, double *dadd, double *ffma) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return W2L_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void *sink = nullptr;
  if (cudaMalloc(&sink, 64) != cudaSuccess) return W2L_ERR_CUDA;
  const int blocks = sms * 8, threads = 256;
  const double n = (double)blocks * threads * kIters * kChains;
  if (mufu) *mufu = time_ops([&] { mufu_probe<<<blocks, threads>>>((float *)sink, 0.5f); }, n);
  if (dadd) *dadd = time_ops([&] { dadd_probe<<<blocks, threads>>>((double *)sink, 1e-9); }, n);
  if (ffma) *ffma = time_ops([&] { ffma_probe<<<blocks, threads>>>((float *)sink, 0.999f); }, n);
  const cudaError_t err = cudaDeviceSynchronize();
  cudaFree(sink);
  return err == cudaSuccess ? W2L_OK : W2L_ERR_CUDA;
}

}  // namespace w2l
