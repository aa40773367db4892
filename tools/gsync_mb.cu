// Grid-wide all-reduce latency (one 512-thread block per SM, warp 0 does the
// exchange): arrival counter(s) + partial loads.  Modes: K split counters
// (block b arrives on counter b % K, lane k < K polls counter k).  The block
// count is varied to see how the latency scales with participants.
#include <cstdio>
template <int K>
__global__ void __launch_bounds__(512, 1) kern(int rounds, double* part, unsigned long long* bar, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nb = gridDim.x;
  if (wid != 0) return;
  double v = blockIdx.x;
  unsigned long long target = 0;
  for (int r = 1; r <= rounds; ++r) {
    if (lane == 0) {
      part[(r & 1) * nb + blockIdx.x] = v;
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(bar + 32 * (blockIdx.x % K)) : "memory");
    }
    if (lane < K) {
      const unsigned long long tgt = (unsigned long long)r * ((nb - lane + K - 1) / K);
      unsigned long long c;
      do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(bar + 32 * lane) : "memory"); } while (c < tgt);
    }
    __syncwarp();
    double s = 0;
    for (int k = 0; k < 5; ++k) { int b = lane + 32 * k; if (b < nb) s += __ldcg(part + (r & 1) * nb + b); }
    v = s;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    v *= 1e-3;
  }
  if (v == 1234.5) out[0] = v;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out; unsigned long long* bar;
  cudaMalloc(&part, 4096 * 8); cudaMalloc(&bar, 32 * 32 * 8); cudaMalloc(&out, 8);
  int rounds = 20000;
  void* fns[4] = {(void*)kern<1>, (void*)kern<4>, (void*)kern<8>, (void*)kern<16>};
  int ks[4] = {1, 4, 8, 16};
  int nbs[3] = {sms, sms / 2, sms / 4};
  for (int m = 0; m < 4; ++m)
    for (int q = 0; q < 3; ++q) {
      cudaMemset(bar, 0, 32 * 32 * 8);
      void* args[] = {&rounds, &part, &bar, &out};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(fns[m], nbs[q], 512, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("K=%2d counters, %3d blocks: %.3f us per round (%s)\n", ks[m], nbs[q], ms * 1e3 / rounds, cudaGetErrorString(e));
    }
  return 0;
}
