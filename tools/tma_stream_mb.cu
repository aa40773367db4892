// HBM -> shared-memory streaming rate of one CTA per SM with TMA bulk copies,
// as the MGS kernel stages basis vectors: each "pass" every CTA pulls its
// 113 KB slice of one 16.7 MB vector; NBUF buffers of 226 KB / NBUF, i.e.
// NBUF copies in flight of a pass's worth split in NBUF/2 chunks.
#include "../paper_2411_00546_b200/csrc/ocp_tma.cuh"
#include <cstdio>
using namespace ocp;
template <int NBUF>
__global__ void __launch_bounds__(512, 1) kern(const double* Q, long long n, int passes, long long per, double* out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[NBUF];
  const long long b0 = blockIdx.x * per;
  const int chunk = (int)(per / (NBUF / 2)) & ~1;   // doubles per copy (2 copies of the pass... NBUF/2 per pass)
  if (threadIdx.x == 0) { for (int i = 0; i < NBUF; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int per_pass = NBUF / 2;   // copies per pass
  const long long total = (long long)passes * per_pass;
  auto issue = [&](long long t) {
    const int b = (int)(t % NBUF);
    const int v = (int)((t / per_pass) % 64);
    const int c = (int)(t % per_pass);
    mbar_expect_tx(&bars[b], chunk * 8u);
    bulk_g2s(sm + (long long)b * chunk, Q + (long long)v * n + b0 + (long long)c * chunk, chunk * 8u, &bars[b]);
  };
  if (threadIdx.x == 0) for (long long t = 0; t < NBUF && t < total; ++t) issue(t);
  double acc = 0;
  for (long long t = 0; t < total; ++t) {
    const int b = (int)(t % NBUF);
    mbar_wait(&bars[b], (uint32_t)((t / NBUF) & 1));
    for (int e = threadIdx.x; e < chunk; e += 512) acc += sm[(long long)b * chunk + e];
    __syncthreads();
    if (threadIdx.x == 0 && t + NBUF < total) issue(t + NBUF);
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long n = 2093058; double *Q, *out;
  cudaMalloc(&Q, 64 * n * 8); cudaMemset(Q, 0, 64 * n * 8); cudaMalloc(&out, 8);
  long long per = (n + sms - 1) / sms; per += per & 1;
  int passes = 2000;
  void* fns[4] = {(void*)kern<2>, (void*)kern<4>, (void*)kern<8>, (void*)kern<16>};
  int nb[4] = {2, 4, 8, 16};
  for (int m = 0; m < 4; ++m) {
    int smem = (int)(2 * per * 8 + 64);
    cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void* args[] = {&Q, &n, &passes, &per, &out};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernel(fns[m], sms, 512, args, smem, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("NBUF %2d (%d copies/pass of %lld KB): %.3f us per pass, %.0f GB/s (%s)\n", nb[m], nb[m] / 2, per * 8 / (nb[m] / 2) / 1024, ms * 1e3 / passes,
           (double)passes * n * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
  }
  return 0;
}
