// One Arnoldi step of the reference's MGS-GMRES in a single cooperative kernel.
//
// krylov.py:110-122 for iteration j:
//     w = A q_j  (already computed, read-only input)
//     for i in 0..j:  h_i = q_i . w ;  w -= h_i q_i        (modified Gram-Schmidt)
//     h_{j+1} = ||w|| ;  q_{j+1} = w / h_{j+1}
//
// The MGS update order is kept: w is updated element by element with each
// h_i in turn.  The grid is co-resident (cooperative launch); every thread
// owns a fixed set of CH elements of w and keeps them in registers across all
// j+1 passes, so each pass streams only q_i from HBM once.  Dots are reduced
// block tree first, then every block sums the per-block partials in the same
// fixed order (a deterministic value, identical in all blocks).  k_arnoldi_lag
// (the config-4 path) computes the local partials of pass i+1 while the grid
// reduction of pass i is in flight; k_arnoldi is the strided fallback for
// vectors whose per-SM share does not fit shared memory twice.  q_{j+1} is
// written unconditionally; the host ignores it on a happy breakdown
// (krylov.py:120-122).
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
#ifndef OCP_LAG_THREADS
#define OCP_LAG_THREADS 512
#endif
constexpr int LAG_THREADS = OCP_LAG_THREADS;          // lagged kernel: threads per block (256 x 2 per SM measured 2 % slower)
constexpr int LAG_BPSM = 512 / LAG_THREADS;           // and blocks per SM
#ifndef OCP_ARN_SLEEP
#define OCP_ARN_SLEEP 50   // ns between barrier polls (measured ~2 % faster than spinning)
#endif
#ifndef OCP_ARN_PF
#define OCP_ARN_PF 1
#endif
constexpr int ARN_PF = OCP_ARN_PF;   // basis vectors prefetched into L2 ahead of the staged one

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

// Split grid barrier on a monotonically increasing 64-bit arrival counter
// (target = epoch + arrivals so far; the host advances epoch by every
// launch's arrivals; blocks are co-resident by the cooperative launch).
// arrive releases the block's partial, wait acquires all of them.
// (one red.release instead of __threadfence + atomicAdd: the release orders
// the partial's store without a full SC fence; 1.3 % per pass, tools/gsync_mb.cu)
__device__ __forceinline__ void gbar_arrive(unsigned long long* bar) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void gbar_wait(const unsigned long long* bar, unsigned long long target) {
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    if (v >= target) break;
#if OCP_ARN_SLEEP > 0
    __nanosleep(OCP_ARN_SLEEP);
#endif
  }
}

// two values summed over the block (fixed order), valid in every thread
template <int THREADS>
__device__ __forceinline__ double2 block_sum2(double a, double b, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if (lane == 0) {
    red[wid] = a;
    red[16 + wid] = b;
  }
  __syncthreads();
  double ra = lane < THREADS / 32 ? red[lane] : 0.0;
  double rb = lane < THREADS / 32 ? red[16 + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ra += __shfl_xor_sync(0xffffffffu, ra, o);
    rb += __shfl_xor_sync(0xffffffffu, rb, o);
  }
  return make_double2(ra, rb);
}

// MGS with the dot of pass i+1 computed while the grid reduction of pass i is
// in flight.  With w' = w - h_i q_i (the MGS update, applied per element
// exactly as before),
//     q_{i+1} . w' = q_{i+1} . w - h_i (q_{i+1} . q_i),
// so a block forms its partials A = q_{i+1} . w and B = q_{i+1} . q_i before
// h_i is known and publishes A - h_i B the moment h_i arrives: the only
// work left on the per-pass critical path is one FMA, the barrier and the
// fixed-order sum of the block partials (identical in every block).  Block b
// owns [b*per, b*per + per); q_{i+1} is staged in shared memory by one TMA
// bulk copy issued two passes ahead and read directly from there, q_i stays in
// registers for the axpy, and basis vectors further ahead stream into L2.
template <int CH>
__global__ void __launch_bounds__(LAG_THREADS, LAG_BPSM)
k_arnoldi_lag(long long n, const double* __restrict__ Q, long long ldq, int j,
              const double* __restrict__ w_in, double* partials, double* h_out, int per,
              unsigned long long* bar, unsigned long long epoch) {
  extern __shared__ __align__(16) double qb[];  // [2][per]
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t bars[2];
  const int tid = threadIdx.x, nb = gridDim.x;
  const long long b0 = (long long)blockIdx.x * per;
  const int cnt = (int)(n - b0 < per ? (n - b0 > 0 ? n - b0 : 0) : per);
  const uint32_t bytes = (uint32_t)cnt * 8u;
  auto load = [&](int v, int buf) {   // q_v -> shared buffer buf (thread 0)
    if (cnt > 0) {
      mbar_expect_tx(&bars[buf], bytes);
      bulk_g2s(qb + buf * per, Q + (long long)v * ldq + b0, bytes, &bars[buf]);
    }
  };
  double w[CH], qv[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int e = tid + k * LAG_THREADS;
    w[k] = e < cnt ? w_in[b0 + e] : 0.0;
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    load(0, 0);
    if (j >= 1) load(1, 1);
    for (int v = 2; v <= 1 + ARN_PF && v <= j; ++v)
      if (cnt > 0) bulk_prefetch_l2(Q + (long long)v * ldq + b0, bytes);
  }
  // pass 0 head: A = q_0 . w
  if (cnt > 0) mbar_wait(&bars[0], 0);
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int e = tid + k * LAG_THREADS;
    qv[k] = e < cnt ? qb[e] : 0.0;
    a = fma(qv[k], w[k], a);
  }
  {
    const double2 r = block_sum2<LAG_THREADS>(a, 0.0, red);
    if (tid == 0) {
      partials[blockIdx.x] = r.x;
      gbar_arrive(bar);
    }
  }
  unsigned long long target = epoch;
  APH_START();
  for (int i = 0; i <= j; ++i) {
    target += nb;
    const bool more = i + 1 <= j;
    // (1) buffer i&1 is free (q_i is in registers): stage q_{i+2}
    __syncthreads();
    if (tid == 0 && i + 2 <= j) {
      load(i + 2, i & 1);
      if (ARN_PF > 0 && i + 2 + ARN_PF <= j && cnt > 0)
        bulk_prefetch_l2(Q + (long long)(i + 2 + ARN_PF) * ldq + b0, bytes);
    }
    // (2) partials of pass i+1 while barrier i is in flight
    double2 AB = make_double2(0.0, 0.0);
    const double* q1 = qb + ((i + 1) & 1) * per;
    if (more) {
      if (cnt > 0) mbar_wait(&bars[(i + 1) & 1], ((i + 1) >> 1) & 1);
      APH(0);
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int e = tid + k * LAG_THREADS;
        const double x = e < cnt ? q1[e] : 0.0;
        sa = fma(x, w[k], sa);
        sb = fma(x, qv[k], sb);
      }
      AB = block_sum2<LAG_THREADS>(sa, sb, red);
    }
    APH(1);
    // (3) h_i: fixed-order sum of the block partials of pass i
    if (tid == 0) gbar_wait(bar, target);
    __syncthreads();
    APH(2);
    const double* part = partials + (i & 1) * nb;
    double v = 0.0;
    for (int b = tid; b < nb; b += blockDim.x) v += __ldcg(part + b);
    const double h = block_sum_all<LAG_THREADS>(v, red);
    APH(3);
    // (4) publish pass i+1 (critical path: one FMA)
    if (more && tid == 0) {
      partials[((i + 1) & 1) * nb + blockIdx.x] = fma(-h, AB.y, AB.x);
      gbar_arrive(bar);
    }
    // (5) the MGS update with h_i, then q_{i+1} into registers
    if (blockIdx.x == 0 && tid == 0) h_out[i] = h;
#pragma unroll
    for (int k = 0; k < CH; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, qv[k]));
    if (more) {
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int e = tid + k * LAG_THREADS;
        qv[k] = e < cnt ? q1[e] : 0.0;
      }
    }
    APH(4);
  }
  // norm pass: h_{j+1} = ||w||, q_{j+1} = w / h_{j+1}
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) acc = fma(w[k], w[k], acc);
  const double bsum = block_sum_all<LAG_THREADS>(acc, red);
  if (tid == 0) {
    partials[((j + 1) & 1) * nb + blockIdx.x] = bsum;
    gbar_arrive(bar);
    gbar_wait(bar, target + nb);
  }
  __syncthreads();
  const double* part = partials + ((j + 1) & 1) * nb;
  double v = 0.0;
  for (int b = tid; b < nb; b += blockDim.x) v += __ldcg(part + b);
  const double hn = sqrt(block_sum_all<LAG_THREADS>(v, red));
  if (blockIdx.x == 0 && tid == 0) h_out[j + 1] = hn;
  double* qn = const_cast<double*>(Q) + (long long)(j + 1) * ldq + b0;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int e = tid + k * LAG_THREADS;
    if (e < cnt) qn[e] = __ddiv_rn(w[k], hn);
  }
}

template <int CH>
static cudaError_t launch_lag(cudaStream_t st, int grid, int per, long long n, const double* Q,
                              long long ldq, int j, const double* w_in, double* partials,
                              double* h_out, unsigned long long* bar, unsigned long long* epoch) {
  void* fn = (void*)k_arnoldi_lag<CH>;
  const int smem = 2 * per * (int)sizeof(double);
  cudaError_t e = raise_smem_limit((const void*)fn, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LAG_THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  unsigned long long ep = *epoch;
  void* args[] = {(void*)&n, (void*)&Q, (void*)&ldq, (void*)&j, (void*)&w_in, (void*)&partials,
                  (void*)&h_out, (void*)&per, (void*)&bar, (void*)&ep};
  e = cudaLaunchCooperativeKernel(fn, grid, LAG_THREADS, args, smem, st);
  if (e == cudaSuccess) *epoch += (unsigned long long)grid * (j + 2);
  return e;
}

// grid of co-resident blocks; returns cudaErrorNotSupported when n does not
// fit the register-resident variant (caller falls back to per-pass kernels)
cudaError_t launch_arnoldi(cudaStream_t st, int num_sms, long long n, const double* Q,
                           long long ldq, int j, const double* w_in, double* partials,
                           double* h_out, unsigned long long* bar, unsigned long long* epoch) {
  // lagged-dot variant when the aligned per-SM share fits twice in shared memory
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int lgrid = num_sms * LAG_BPSM;
    long long per = (n + lgrid - 1) / lgrid;
    per += per & 1;
    const bool aligned = (n % 2 == 0) && (ldq % 2 == 0) &&
                         ((reinterpret_cast<uintptr_t>(Q) & 15) == 0);
    if (aligned && n > 0 && lgrid <= 1024 && LAG_BPSM * (16 * per + 1024) <= optin && per <= 28 * LAG_THREADS) {
      const int p = (int)per;
      cudaError_t e;
      if (per <= 8 * LAG_THREADS) e = launch_lag<8>(st, lgrid, p, n, Q, ldq, j, w_in, partials, h_out, bar, epoch);
      else if (per <= 16 * LAG_THREADS) e = launch_lag<16>(st, lgrid, p, n, Q, ldq, j, w_in, partials, h_out, bar, epoch);
      else if (per <= 24 * LAG_THREADS) e = launch_lag<24>(st, lgrid, p, n, Q, ldq, j, w_in, partials, h_out, bar, epoch);
      else e = launch_lag<28>(st, lgrid, p, n, Q, ldq, j, w_in, partials, h_out, bar, epoch);
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
  cudaError_t e = raise_smem_limit((const void*)fn, smem);
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
