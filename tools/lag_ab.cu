// Time k_arnoldi_lag<28> on config-4-sized vectors, J Arnoldi steps on a
// random basis; prints us per MGS pass and a checksum of the Hessenberg
// columns (compile with different -DOCP_LAG_* flags for an A/B).
#include "../paper_2411_00546_b200/csrc/ocp_krylov.cu"
#include <cstdio>
#include <vector>
#include <curand_kernel.h>
__global__ void fill(double* x, long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    curandStatePhilox4_32_10_t s; curand_init(seed, i, 0, &s); x[i] = curand_normal_double(&s) * 1e-3;
  }
}
int main(int argc, char** argv) {
  const long long n = 2093058; const int J = argc > 1 ? atoi(argv[1]) : 145;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *Q, *W, *part, *h; unsigned long long* bar;
  cudaMalloc(&Q, (size_t)(J + 2) * n * 8); cudaMalloc(&W, (size_t)J * n * 8); cudaMalloc(&part, 2 * 2048 * 8);
  cudaMalloc(&h, (size_t)(J + 2) * J * 8); cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  fill<<<1024, 256>>>(Q, (J + 2) * n, 1); fill<<<1024, 256>>>(W, J * n, 2); cudaDeviceSynchronize();
  unsigned long long epoch = 0; long long per = (n + sms - 1) / sms; per += per & 1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    for (int j = 0; j < J; ++j)
      if (ocp::launch_lag<28>(0, sms, (int)per, n, Q, n, j, W + (long long)j * n, part, h + (long long)j * (J + 2), bar, &epoch) != cudaSuccess) { printf("launch failed\n"); return 1; }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("k_arnoldi_lag<28>: %.3f us per pass\n", ms * 1e3 / ((double)J * (J + 1) / 2 + J));
  }
  std::vector<double> hv((size_t)(J + 2) * J); cudaMemcpy(hv.data(), h, hv.size() * 8, cudaMemcpyDeviceToHost);
  double cs = 0; for (int j = 0; j < J; ++j) for (int i = 0; i <= j + 1; ++i) cs += hv[(size_t)j * (J + 2) + i] * (1 + 1e-3 * i);
  printf("checksum %.17g (%s)\n", cs, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
