// FP64 issue-rate probe for the DMMA-vs-FMA decision (north star: "FP64
// tensor-core DMMA for the D contractions only if ncu shows it beats the FMA
// path").  Measures, on one B200, the sustained FP64 rate of
//   (a) DFMA chains (the FMA path's instruction), and
//   (b) mma.sync.aligned.m8n8k4 f64 (DMMA; 256 FMAs per warp instruction),
// with enough independent accumulators per warp to cover latency, over a
// grid of 148 x 8 warps.  Build:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/dmma_probe.cu -o tools/_dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[CH][2];
#pragma unroll
  for (int q = 0; q < CH; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < CH; ++q) dmma(c[q][0], c[q][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[CH];
#pragma unroll
  for (int q = 0; q < CH; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < CH; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < CH; ++q) s += c[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
float run(K kern, double* out, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters / 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    const int threads = 32 * warps;
    {
      float ms = run(k_dfma<8>, out, sms, threads, iters);
      double flops = 2.0 * sms * threads * 8.0 * iters;
      printf("DFMA  warps/SM=%2d chains=8 : %.3f ms  %.2f TFLOP/s\n", warps, ms,
             flops / ms / 1e9);
    }
    {
      float ms = run(k_dmma<4>, out, sms, threads, iters);
      double flops = 2.0 * sms * warps * 256.0 * 4 * iters;
      printf("DMMA  warps/SM=%2d chains=4 : %.3f ms  %.2f TFLOP/s\n", warps, ms,
             flops / ms / 1e9);
    }
    {
      float ms = run(k_dmma<8>, out, sms, threads, iters);
      double flops = 2.0 * sms * warps * 256.0 * 8 * iters;
      printf("DMMA  warps/SM=%2d chains=8 : %.3f ms  %.2f TFLOP/s\n", warps, ms,
             flops / ms / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
