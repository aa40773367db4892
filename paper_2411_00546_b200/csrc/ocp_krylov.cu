// One Arnoldi step of the reference's MGS-GMRES in a single cooperative kernel.
//
// krylov.py:110-122 for iteration j:
//     w = A q_j  (already computed, read-only input)
//     for i in 0..j:  h_i = q_i . w ;  w -= h_i q_i        (modified Gram-Schmidt)
//     h_{j+1} = ||w|| ;  q_{j+1} = w / h_{j+1}
//
// The MGS dependency chain (each h_i needs the w updated by h_{i-1}) is kept
// exactly.  The grid is co-resident (cooperative launch); every thread owns a
// fixed strided set of CH elements of w and keeps them in registers across
// all j+1 passes, so each pass streams only q_i from HBM once: q_i is staged
// in shared memory (CH x 512 doubles per block), the dot is reduced (block tree, then a grid barrier, then
// every block sums the per-block partials in the same fixed order - a
// deterministic result identical in all blocks), and the axpy reuses the
// registers.  q_{j+1} is written unconditionally; the host ignores it on a
// happy breakdown (krylov.py:120-122).
#include <cooperative_groups.h>

#include "ocp_kernels.cuh"
#include "ocp_tma.cuh"

namespace cg = cooperative_groups;

namespace ocp {

template <int THREADS>
__device__ __forceinline__ double block_sum_all(double v, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = lane < THREADS / 32 ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;  // valid in every thread
}

constexpr int ARN_THREADS = 512;

// optional per-phase cycle counters of block 0 (build with -DOCP_PHASE_TIMING; tools/aphase_dbg.py)
#ifdef OCP_PHASE_TIMING
__device__ unsigned long long g_aphase[8];
void read_aphase(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_aphase, 8 * sizeof(unsigned long long));
}
#define APH_START() long long t_last = clock64()
#define APH(k)                                                                          \
  do {                                                                                  \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                          \
      const long long now = clock64();                                                  \
      atomicAdd(&g_aphase[k], (unsigned long long)(now - t_last));                      \
      t_last = now;                                                                     \
    }                                                                                   \
  } while (0)
#else
#define APH_START() (void)0
#define APH(k) (void)0
#endif

template <int CH>
__global__ void __launch_bounds__(ARN_THREADS, 1)
k_arnoldi(long long n, const double* __restrict__ Q, long long ldq, int j,
          const double* __restrict__ w_in, double* partials, double* h_out) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double qs[];  // [CH][ARN_THREADS]
  __shared__ double red[32];
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double w[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const long long e = e0 + k * stride;
    w[k] = e < n ? w_in[e] : 0.0;
  }
  const int nb = gridDim.x;
  for (int i = 0; i <= j + 1; ++i) {
    const bool norm_pass = (i == j + 1);
    const double* q = Q + (long long)i * ldq;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const long long e = e0 + k * stride;
      const double qv = (!norm_pass && e < n) ? q[e] : 0.0;
      qs[k * ARN_THREADS + threadIdx.x] = qv;
      acc = norm_pass ? fma(w[k], w[k], acc) : fma(qv, w[k], acc);
    }
    const double bsum = block_sum_all<ARN_THREADS>(acc, red);
    double* part = partials + (i & 1) * nb;
    if (threadIdx.x == 0) part[blockIdx.x] = bsum;
    grid.sync();
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) v += __ldcg(part + b);
    const double h = block_sum_all<ARN_THREADS>(v, red);
    if (norm_pass) {
      const double hn = sqrt(h);
      if (blockIdx.x == 0 && threadIdx.x == 0) h_out[i] = hn;
      double* qn = const_cast<double*>(Q) + (long long)(j + 1) * ldq;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const long long e = e0 + k * stride;
        if (e < n) qn[e] = __ddiv_rn(w[k], hn);
      }
    } else {
      if (blockIdx.x == 0 && threadIdx.x == 0) h_out[i] = h;
#pragma unroll
      for (int k = 0; k < CH; ++k)
        w[k] = __dsub_rn(w[k], __dmul_rn(h, qs[k * ARN_THREADS + threadIdx.x]));
    }
  }
}

// Double-buffered variant for vectors whose per-SM share fits twice in shared
// memory (config 4: 2 x 110 KB): block b owns the contiguous range
// [b*per, b*per + per) and thread t its elements t + 512 k.  q_{i+1} streams
// into the idle buffer by one TMA bulk copy issued at the start of pass i, so
// the HBM transfer of the next basis vector runs under this pass's barrier and
// reductions instead of after them (measured: a pass that loads q after the
// grid barrier costs ~3x the bare HBM stream time).
template <int CH>
__global__ void __launch_bounds__(ARN_THREADS, 1)
k_arnoldi_db(long long n, const double* __restrict__ Q, long long ldq, int j,
             const double* __restrict__ w_in, double* partials, double* h_out, int per) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double qb[];  // [2][per]
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t bars[2];
  const int tid = threadIdx.x;
  const long long b0 = (long long)blockIdx.x * per;
  const int cnt = (int)(n - b0 < per ? (n - b0 > 0 ? n - b0 : 0) : per);
  const uint32_t bytes = (uint32_t)cnt * 8u;
  double w[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int e = tid + k * ARN_THREADS;
    w[k] = e < cnt ? w_in[b0 + e] : 0.0;
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && cnt > 0) {
    mbar_expect_tx(&bars[0], bytes);
    bulk_g2s(qb, Q + b0, bytes, &bars[0]);
  }
  const int nb = gridDim.x;
  APH_START();
  for (int i = 0; i <= j + 1; ++i) {
    const bool norm_pass = (i == j + 1);
    const double* cur = qb + (i & 1) * per;
    double acc = 0.0;
    // q_{i+1} goes into the buffer of q_{i-1} as soon as every thread is done
    // with pass i-1's axpy: the HBM stream then runs under this whole pass
    __syncthreads();
    if (tid == 0 && i + 1 <= j && cnt > 0) {
      uint64_t* bar = &bars[(i + 1) & 1];
      mbar_expect_tx(bar, bytes);
      bulk_g2s(qb + ((i + 1) & 1) * per, Q + (long long)(i + 1) * ldq + b0, bytes, bar);
    }
    double qv[CH];   // q_i stays in registers for the axpy (one shared-memory read)
    if (!norm_pass) {
      if (cnt > 0) mbar_wait(&bars[i & 1], (i >> 1) & 1);
      APH(0);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int e = tid + k * ARN_THREADS;
        qv[k] = e < cnt ? cur[e] : 0.0;
        acc = fma(qv[k], w[k], acc);
      }
    } else {
#pragma unroll
      for (int k = 0; k < CH; ++k) acc = fma(w[k], w[k], acc);
    }
    const double bsum = block_sum_all<ARN_THREADS>(acc, red);
    double* part = partials + (i & 1) * nb;
    if (tid == 0) part[blockIdx.x] = bsum;
    APH(1);
    grid.sync();
    APH(2);
    double v = 0.0;
    for (int b = tid; b < nb; b += blockDim.x) v += __ldcg(part + b);
    const double h = block_sum_all<ARN_THREADS>(v, red);
    APH(3);
    if (norm_pass) {
      const double hn = sqrt(h);
      if (blockIdx.x == 0 && tid == 0) h_out[i] = hn;
      double* qn = const_cast<double*>(Q) + (long long)(j + 1) * ldq + b0;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int e = tid + k * ARN_THREADS;
        if (e < cnt) qn[e] = __ddiv_rn(w[k], hn);
      }
    } else {
      if (blockIdx.x == 0 && tid == 0) h_out[i] = h;
#pragma unroll
      for (int k = 0; k < CH; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, qv[k]));
    }
    APH(4);
  }
}

template <int CH>
static cudaError_t launch_db(cudaStream_t st, int grid, int per, long long n, const double* Q,
                             long long ldq, int j, const double* w_in, double* partials,
                             double* h_out) {
  void* fn = (void*)k_arnoldi_db<CH>;
  const int smem = 2 * per * (int)sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ARN_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  void* args[] = {(void*)&n, (void*)&Q, (void*)&ldq, (void*)&j, (void*)&w_in, (void*)&partials,
                  (void*)&h_out, (void*)&per};
  return cudaLaunchCooperativeKernel(fn, grid, ARN_THREADS, args, smem, st);
}

// grid of co-resident blocks; returns cudaErrorNotSupported when n does not
// fit the register-resident variant (caller falls back to per-pass kernels)
cudaError_t launch_arnoldi(cudaStream_t st, int num_sms, long long n, const double* Q,
                           long long ldq, int j, const double* w_in, double* partials,
                           double* h_out) {
  // double-buffered variant when the aligned per-SM share fits twice in shared memory
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    long long per = (n + num_sms - 1) / num_sms;
    per += per & 1;
    const bool aligned = (n % 2 == 0) && (ldq % 2 == 0) &&
                         ((reinterpret_cast<uintptr_t>(Q) & 15) == 0);
    if (aligned && n > 0 && num_sms <= 256 && 16 * per + 512 <= optin && per <= 32 * ARN_THREADS) {
      const int p = (int)per;
      cudaError_t e;
      if (per <= 8 * ARN_THREADS) e = launch_db<8>(st, num_sms, p, n, Q, ldq, j, w_in, partials, h_out);
      else if (per <= 16 * ARN_THREADS) e = launch_db<16>(st, num_sms, p, n, Q, ldq, j, w_in, partials, h_out);
      else if (per <= 24 * ARN_THREADS) e = launch_db<24>(st, num_sms, p, n, Q, ldq, j, w_in, partials, h_out);
      else if (per <= 28 * ARN_THREADS) e = launch_db<28>(st, num_sms, p, n, Q, ldq, j, w_in, partials, h_out);
      else e = launch_db<32>(st, num_sms, p, n, Q, ldq, j, w_in, partials, h_out);
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
    }
  }
  const long long threads = (long long)num_sms * ARN_THREADS;
  const long long ch = (n + threads - 1) / threads;
  void* fn = nullptr;
  int c = 0;
  if (ch <= 8) { fn = (void*)k_arnoldi<8>; c = 8; }
  else if (ch <= 16) { fn = (void*)k_arnoldi<16>; c = 16; }
  else if (ch <= 24) { fn = (void*)k_arnoldi<24>; c = 24; }
  else if (ch <= 32) { fn = (void*)k_arnoldi<32>; c = 32; }
  else return cudaErrorNotSupported;
  const int smem = c * ARN_THREADS * (int)sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ARN_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  int grid = num_sms;
  void* args[] = {(void*)&n, (void*)&Q, (void*)&ldq, (void*)&j, (void*)&w_in, (void*)&partials,
                  (void*)&h_out};
  return cudaLaunchCooperativeKernel(fn, grid, ARN_THREADS, args, smem, st);
}

}  // namespace ocp
