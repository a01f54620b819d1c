// Probe: a conditional graph node (IF) whose condition a gate kernel sets,
// vs the same kernels launched eagerly.  Body kernels early-exit on a flag.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cond_probe tools/cond_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void gate(const int *status, int n, cudaGraphConditionalHandle h) {
  int any = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) any |= status[i] != 0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) cudaGraphSetConditional(h, any ? 1u : 0u);
}
__global__ void body(const int *status, int *out) {
  extern __shared__ int sm[];
  if (status[blockIdx.x % 64] == 0) return;
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
}
__global__ void spin(long long ns) {
  long long t0 = clock64();
  while (clock64() - t0 < ns) {}
}
int main() {
  int *status, *out;
  cudaMalloc(&status, 64 * 4);
  cudaMalloc(&out, 4096 * 4);
  cudaMemset(status, 0, 64 * 4);
  cudaStream_t s, cap;
  cudaStreamCreate(&s);
  cudaStreamCreate(&cap);
  cudaFuncSetAttribute(body, cudaFuncAttributeMaxDynamicSharedMemorySize, 90 * 1024);
  // graph: gate -> IF { body(128 CTAs), body(1664 CTAs), body(64 CTAs) } (body by capture)
  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
    printf("handle create failed\n");
    return 1;
  }
  cudaGraphNode_t ng;
  cudaKernelNodeParams kp = {};
  int n = 64;
  void *gargs[] = {&status, &n, &h};
  kp.func = (void *)gate;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(256);
  kp.kernelParams = gargs;
  cudaError_t e = cudaGraphAddKernelNode(&ng, g, nullptr, 0, &kp);
  printf("add gate: %s\n", cudaGetErrorString(e));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t nc;
  e = cudaGraphAddNode(&nc, g, &ng, 1, &cp);
  printf("add cond: %s\n", cudaGetErrorString(e));
  cudaGraph_t bg = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(cap, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("begin capture: %s\n", cudaGetErrorString(e));
  body<<<128, 256, 90 * 1024, cap>>>(status, out);
  body<<<1664, 256, 90 * 1024, cap>>>(status, out);
  body<<<64, 512, 16 * 1024, cap>>>(status, out);
  cudaGraph_t tmp;
  e = cudaStreamEndCapture(cap, &tmp);
  printf("end capture: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex;
  e = cudaGraphInstantiate(&ex, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    if (mode == 2) cudaMemset(status, 1, 64 * 4);   // body does work
    float best = 1e9;
    for (int it = 0; it < 20; ++it) {
      spin<<<1, 1, 0, s>>>(200000);
      cudaEventRecord(a, s);
      if (mode % 2 == 0) {
        body<<<128, 256, 90 * 1024, s>>>(status, out);
        body<<<1664, 256, 90 * 1024, s>>>(status, out);
        body<<<64, 512, 16 * 1024, s>>>(status, out);
      } else {
        cudaGraphLaunch(ex, s);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%s status=%d: %.2f us\n", mode % 2 ? "graph" : "eager", mode >= 2, best * 1e3);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
