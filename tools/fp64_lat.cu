// Dependent-chain latency probe: cycles per dependent DFMA / DADD / DMUL / MUFU
// rcp and per shared-memory load, one warp alone on the GPU.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 1e-3;
  __syncthreads();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = y + b;
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = z * b;
  long long t3 = clock64();
  int idx = threadIdx.x & 31;
  double s = 0.0;
  for (int i = 0; i < n; ++i) { s += sm[idx]; idx = ((int)(s * 1e-9) + idx + 1) & 31; }
  long long t4 = clock64();
  double r = a;
  for (int i = 0; i < n; ++i) { double q; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(r)); r = q + 1.0; }
  long long t5 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) w = __shfl_xor_sync(0xffffffffu, w, 1) + 1.0;
  long long t6 = clock64();
  out[threadIdx.x] = x + y + z + s + r + w;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
  }
  printf("cycles per dependent op: DFMA %.1f  DADD %.1f  DMUL %.1f  LDS+DADD %.1f  MUFU.RCP64+DADD %.1f  SHFL+DADD %.1f\n",
         (double)cyc[0] / n, (double)cyc[1] / n, (double)cyc[2] / n, (double)cyc[3] / n, (double)cyc[4] / n, (double)cyc[5] / n);
  return 0;
}
