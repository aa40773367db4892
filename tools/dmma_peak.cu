// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput probe vs the DFMA probe.
// Decides whether the banded-LU trailing update should use DMMA (BASELINE.json:
// "tensor cores only if a dense sub-block ... is shown to gain from FP64 DMMA").
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters, double a, double b) {
  double c[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) c[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[2 * k], c[2 * k + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += c[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dmma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double flops = 2.0 * 256 * 8 * (double)iters * warps;
  printf("{\"dmma_fp64_tflops\": %.3f, \"best_ms\": %.4f, \"err\": \"%s\"}\n", flops / (best * 1e-3) / 1e12,
         best, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
