// HBM read-bandwidth probe: (a) grid-stride LDG.128 sum, (b) TMA bulk-copy ring
// into shared memory (4 x 24 KB stages per CTA, 2 CTAs per SM) - the access
// pattern of the JVP solve without its arithmetic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ldg(const double2* __restrict__ x, long long n2, double* out) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(x + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGES>
__global__ void k_bulk(const double* __restrict__ x, long long per_cta, int chunk, double* out,
                       int pf = 0, int delay = 0) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  const double* src = x + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int t) {
    const int st = t % STAGES;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[st])), "r"(chunk * 8));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + st * chunk)), "l"(src + (long long)t * chunk), "r"(chunk * 8), "r"(su32(&bars[st])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int t = 0; t < STAGES && t < nch; ++t) issue(t);
    for (int t = STAGES; t < STAGES + pf && t < nch; ++t)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (long long)t * chunk), "r"(chunk * 8) : "memory");
  }
  double s = 0.0;
  for (int t = 0; t < nch; ++t) {
    const int st = t % STAGES;
    const uint32_t ph = (t / STAGES) & 1;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(su32(&bars[st])), "r"(ph) : "memory");
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) s += sm[st * chunk + i];
    if (delay) { const long long t0 = clock64(); while (clock64() - t0 < delay) {} }
    __syncthreads();
    if (threadIdx.x == 0 && t + STAGES < nch) {
      issue(t + STAGES);
      if (pf && t + STAGES + pf < nch)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (long long)(t + STAGES + pf) * chunk), "r"(chunk * 8) : "memory");
    }
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  const long long n = 4LL << 27;   // 4 GiB of doubles / 8 = 512 Mi doubles -> 4 GB
  double *x, *out;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_ldg<<<sms * 8, 256>>>((const double2*)x, n / 2, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg.128 grid-stride: %.1f GB/s\n", n * 8 / ms / 1e6);
  }
  const int chunk = 2880;   // 23 KB (the JVP stage)
  const int grid = 256;     // one CTA per subdomain, 2 per SM
  const long long per = (n / 2 / grid) / chunk * chunk;   // 8 MB per CTA
  const int smem = 4 * chunk * 8;
  cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int delay : {0, 1000, 2000, 4000}) {
    for (int pf : {0, 2, 4, 8, 16}) {
      cudaEventRecord(a);
      k_bulk<4><<<grid, 256, smem>>>(x, per, chunk, out, pf, delay);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("256 CTAs, ring 4 x 23 KB, consumer delay %4d cyc/stage, L2 prefetch %2d stages ahead: %.1f GB/s\n",
             delay, pf, grid * per * 8 / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
