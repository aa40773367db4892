// Banded forward/backward solve with the stored local factors (sm_100a, FP64).
//
// Replaces SuperLU.solve (newton.py:127 for the inner Newton direction,
// schwarz.py:343 inside raspen_jacobian_apply).  One CTA per subdomain:
//
//   * the factor blocks ([L | U] per panel of NB unknowns, ocp_band.cu) stream
//     from HBM through a STAGES-deep ring of shared-memory buffers filled by
//     TMA bulk copies (cp.async.bulk + mbarrier complete_tx), issued STAGES
//     blocks ahead of use;
//   * the active part of the vector (W + 2 NB entries) lives in a circular
//     shared buffer; finished forward values go to the output vector and
//     come back for the backward sweep;
//   * blocks of 32 unknowns; the 32x32 diagonal triangles were inverted at
//     factorisation time, so each block costs two barrier-separated phases of
//     independent FMAs:
//       forward  y_K = L11^{-1} b_K ;  b_{K+1..} -= L21 y_K
//       backward x_K = U11^{-1} (z_K - U12 x_{K+1..})
//
// rhs = scale * in_pool, solution -> out_pool (band order; in place allowed).
// Every global access on the per-block critical path is prefetched one
// block ahead (entering rhs rows, z of the next backward block).
// MODE 1 (JVP): only the ownership block of the solution is consumed
// (schwarz.py:344), so the backward sweep stops above the first owned row.
#include <cstdint>

#include "ocp_kernels.cuh"
#include "ocp_tma.cuh"

namespace ocp {

// circular vector window: >= W + 2 NBF entries, power of two (index by mask)
__host__ __device__ __forceinline__ int ring_size(int w) {
  int r = 64;
  while (r < w + 2 * NBF) r <<= 1;
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2)
k_band_solve(const SubInfo* subs, const int* list, const double* fac_pool, const double* in_pool,
             double scale, double* out_pool, int max_w) {
  extern __shared__ __align__(16) double smem[];
  constexpr int B = NBF;                            // 32 unknowns per factor block
  const int SB = B * (max_w + 1);                   // doubles per stage
  const int RMAX = ring_size(max_w);
  double* stage = smem;                             // SOLVE_STAGES x SB
  double* ring = smem + SOLVE_STAGES * SB;          // RMAX (power of two)
  double* ys = ring + RMAX;                         // B
  uint64_t* bars = reinterpret_cast<uint64_t*>(ys + B);  // 2 x SOLVE_STAGES

  const SubInfo s = subs[list[blockIdx.x]];
  const int tid = threadIdx.x;
  const int W = s.W, LD = W + 1, NP = s.NP, nblk = NP / B;
  const int RM = ring_size(W) - 1;                  // ring index mask
  const long long bstride = 2LL * B * LD;
  const double* fac = fac_pool + s.fac;
  double* zx = out_pool + s.loc;                    // z after the forward sweep, x after the backward
  const double* in = in_pool + s.loc;
  const int gi = tid >> 3, gj = tid & 7;            // 32 x 8 thread grid for the block mat-vecs

  if (tid == 0) {
    for (int st = 0; st < 2 * SOLVE_STAGES; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k <= RM; k += blockDim.x) ring[k] = 0.0;
  __syncthreads();
  // ---------------- forward: L y = b ----------------
  const uint32_t lbytes = (uint32_t)(B * LD * sizeof(double));
  if (tid == 0) {
    for (int st = 0; st < SOLVE_STAGES && st < nblk; ++st) {
      mbar_expect_tx(&bars[st], lbytes);
      bulk_g2s(stage + st * SB, fac + st * bstride, lbytes, &bars[st]);
    }
  }
  for (int k = tid; k < W + B && k < NP; k += blockDim.x) ring[k & RM] = scale * in[k];
  // rows entering the window at step K are [k0+B+W, k0+2B+W): prefetched one step ahead
  double rreg = 0.0;
  if (tid < B && B + W + tid < NP) rreg = in[B + W + tid];
  __syncthreads();
  for (int K = 0; K < nblk; ++K) {
    const int k0 = K * B, st = K % SOLVE_STAGES;
    const double* Lb = stage + st * SB;
    mbar_wait(&bars[st], (K / SOLVE_STAGES) & 1);
    {  // y_K = L11^{-1} b_K   (row gi, 8 lanes reduce over j = gj + 8m)
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int j = gj + 8 * m;
        const double bj = ring[(k0 + j) & RM];
        const double l = Lb[j * LD + ((gi - j - 1) & 31)];
        v += j < gi ? l * bj : (j == gi ? bj : 0.0);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (gj == 0) ys[gi] = v;
    }
    __syncthreads();
    if (tid < B) {
      const double y = ys[tid];
      ring[(k0 + tid) & RM] = y;
      zx[k0 + tid] = y;
      const int r = k0 + B + W + tid;                // entering row (slot of k0 - B + tid)
      if (r < NP) ring[r & RM] = scale * rreg;
      const int rn = r + B;
      rreg = rn < NP ? in[rn] : 0.0;
    }
    {  // b_r -= L21 y_K, r = k0 + B + t
      const int t = tid;
      const int r = k0 + B + t;
      if (t < W && r < NP) {
        const double* lp = Lb + (B - 1) + t;         // column c entry at lp + c * (LD - 1)
        double acc[4] = {ring[r & RM], 0.0, 0.0, 0.0};
        if (t + B <= W) {
#pragma unroll
          for (int c = 0; c < B; ++c) acc[c & 3] = fma(-lp[c * (LD - 1)], ys[c], acc[c & 3]);
        } else {
#pragma unroll
          for (int c = 0; c < B; ++c)
            if (B - 1 + t - c < W) acc[c & 3] = fma(-lp[c * (LD - 1)], ys[c], acc[c & 3]);
        }
        ring[r & RM] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
    }
    __syncthreads();
    if (tid == 0 && K + SOLVE_STAGES < nblk) {
      mbar_expect_tx(&bars[st], lbytes);
      bulk_g2s(stage + st * SB, fac + (K + SOLVE_STAGES) * bstride, lbytes, &bars[st]);
    }
  }
  // ---------------- backward: U x = z ----------------
  int kstop = 0;  // first row whose solution is needed
  if (MODE == 1) {
    const int a_own = s.orient == 0 ? s.or0 - s.r0 : s.oc0 - s.c0;
    kstop = 2 * s.nc * a_own;
  }
  const uint32_t ubytes = (uint32_t)(B * LD * sizeof(double));
  uint64_t* ubars = bars + SOLVE_STAGES;
  if (tid == 0) {
    for (int st = 0; st < SOLVE_STAGES && st < nblk; ++st) {
      const int K = nblk - 1 - st;
      mbar_expect_tx(&ubars[st], ubytes);
      bulk_g2s(stage + st * SB, fac + K * bstride + B * LD, ubytes, &ubars[st]);
    }
  }
  // ring slots of indices >= NP must read as 0 (their U entries are 0 too)
  for (int k = NP + tid; k < NP + W + B; k += blockDim.x) ring[k & RM] = 0.0;
  __syncthreads();
  // z of block K is in the ring when step K starts; z of K-1 is held in a
  // register one step ahead
  if (tid < B) ring[(NP - B + tid) & RM] = zx[NP - B + tid];
  double zreg = (tid < B && nblk >= 2) ? zx[NP - 2 * B + tid] : 0.0;
  const int MW = (W + 7) / 8 + 1;  // band columns per lane (stride 8)
  __syncthreads();
  int step = 0;
  for (; step < nblk; ++step) {
    const int K = nblk - 1 - step, k0 = K * B, st = step % SOLVE_STAGES;
    if (k0 + B <= kstop) break;
    const double* Ub = stage + st * SB;
    mbar_wait(&ubars[st], (step / SOLVE_STAGES) & 1);
    {  // r_c = z_c - U12 x   (row gi, lanes gj stride 8 over the band)
      double acc0 = 0.0, acc1 = 0.0;
      const double* up = Ub + gi * LD;
      const int base = k0 + gi;
#pragma unroll 4
      for (int m = 0; m < MW; m += 2) {
        const int sidx = B - gi + gj + 8 * m;
        if (sidx <= W) acc0 = fma(up[sidx], ring[(base + sidx) & RM], acc0);
        if (sidx + 8 <= W) acc1 = fma(up[sidx + 8], ring[(base + sidx + 8) & RM], acc1);
      }
      double acc = acc0 + acc1;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (gj == 0) ys[gi] = ring[(k0 + gi) & RM] - acc;
    }
    __syncthreads();
    {  // x_K = U11^{-1} r
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int j = gj + 8 * m;
        const double u = Ub[gi * LD + ((j - gi) & 31)];
        v += j >= gi ? u * ys[j] : 0.0;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (gj == 0) {
        ring[(k0 + gi) & RM] = v;
        zx[k0 + gi] = v;
      }
    }
    if (tid < B && k0 >= B) {
      ring[(k0 - B + tid) & RM] = zreg;
      zreg = k0 >= 2 * B ? zx[k0 - 2 * B + tid] : 0.0;
    }
    __syncthreads();
    if (tid == 0 && step + SOLVE_STAGES < nblk) {
      const int Kn = nblk - 1 - (step + SOLVE_STAGES);
      mbar_expect_tx(&ubars[st], ubytes);
      bulk_g2s(stage + st * SB, fac + Kn * bstride + B * LD, ubytes, &ubars[st]);
    }
  }
  // an early stop leaves up to SOLVE_STAGES bulk copies in flight: wait for
  // them before the CTA (and its shared memory) retires
  for (int s2 = step; s2 < nblk && s2 < step + SOLVE_STAGES; ++s2)
    mbar_wait(&ubars[s2 % SOLVE_STAGES], (s2 / SOLVE_STAGES) & 1);
}

size_t solve_smem_bytes(int max_w) {
  return sizeof(double) * ((size_t)SOLVE_STAGES * NBF * (max_w + 1) + ring_size(max_w) + NBF) +
         sizeof(uint64_t) * 2 * SOLVE_STAGES;
}

cudaError_t launch_band_solve(int mode, int grid, cudaStream_t st, const SubInfo* subs,
                              const int* list, const double* fac, const double* in, double scale,
                              double* out_pool, int max_w) {
  const size_t smem = solve_smem_bytes(max_w);
  if (mode == 0)
    k_band_solve<0><<<grid, 256, smem, st>>>(subs, list, fac, in, scale, out_pool, max_w);
  else
    k_band_solve<1><<<grid, 256, smem, st>>>(subs, list, fac, in, scale, out_pool, max_w);
  return cudaGetLastError();
}

cudaError_t set_band_solve_smem(int bytes) {
  cudaError_t e = raise_smem_limit((const void*)k_band_solve<0>, bytes);
  if (e != cudaSuccess) return e;
  return raise_smem_limit((const void*)k_band_solve<1>, bytes);
}

}  // namespace ocp
