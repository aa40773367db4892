// Kernel declarations shared by the translation units.
#pragma once
#include "ocp_common.cuh"

// local residual: RQ flat local points per CTA of RES_THREADS threads, min
// resident CTAs per SM (measured on config 4 / 5: 128 x 4 x 8 fastest)
#ifndef OCP_RES_THREADS
#define OCP_RES_THREADS 128
#endif
#ifndef OCP_RES_PPT
#define OCP_RES_PPT 4
#endif
constexpr int RES_THREADS = OCP_RES_THREADS;
constexpr int RQ = OCP_RES_THREADS * OCP_RES_PPT;
#ifndef OCP_RES_MINB
#define OCP_RES_MINB 8
#endif

namespace ocp {

__global__ void k_gather(const SubInfo* subs, const int* list, Phys P, const double* x, double* pool);
size_t residual_smem_bytes(int max_nc);
template <bool DIRECT>
__global__ void k_residual(const SubInfo* subs, const int* list, Phys P, const double* x,
                           const double* Vpool, const double* Dpool, const double* alpha,
                           const double* f, const double* yd, double eps, double* Rpool,
                           double* partials, double* JDpool, unsigned long long* badparts);
__global__ void k_jacdiag(const SubInfo* subs, const int* list, Phys P, const double* Vpool,
                          double eps, double* JDpool, long long* bad);
__global__ void k_update(const SubInfo* subs, const int* list, double* Vpool, const double* Dpool,
                         const double* alpha);
__global__ void k_scatter_fval(const SubInfo* subs, Phys P, const double* Vpool, const double* x,
                               double* fval);
__global__ void k_ref_to_band(const SubInfo* subs, const double* ref, double* pool);
__global__ void k_band_to_ref(const SubInfo* subs, const double* pool, double* ref);
__global__ void k_dot(long long n, const double* x, const double* y, double* partials,
                      unsigned int* counter, double* result, int take_sqrt);
__global__ void k_mgs_pass(long long n, double* w, const double* q_prev, const double* h_prev,
                           const double* q_i, double* partials, unsigned int* counter,
                           double* h_out);
__global__ void k_add_scaled(long long n, const double* x, double alpha, const double* d, double* out);
__global__ void k_scale(long long n, double a, const double* x, double* out);
__global__ void k_div(long long n, const double* x, double s, double* out);
__global__ void k_flags(long long n, const double* x, const double* y, int* flag);
__global__ void k_gemv_add(long long n, const double* Q, long long ldq, int k, const double* y,
                           const double* x, double* out);
__global__ void k_recover_control(long long n, Phys P, const double* p, double eps, double* u);

// whole-grid operators of newton-ras-eps (ocp_global.cu)
__global__ void k_global_residual(Phys P, const double* x, const double* f, const double* yd,
                                  double eps, double* r);
__global__ void k_global_jacdiag(Phys P, const double* x, double eps, double4* JD,
                                 unsigned long long* bad);
__global__ void k_global_jvp(Phys P, const double4* JD, const double* d, double* out);
__global__ void k_state_residual(Phys P, const double* y, const double* rhs, double* out);
__global__ void k_state_diag(Phys P, const double* y, double* dg, unsigned long long* bad);
__global__ void k_cg_ap(Phys P, const double* dg, const double* p, double* Ap, double* partials,
                        unsigned int* counter, double* sc);
__global__ void k_cg_xr(long long N, const double* p, const double* Ap, double* x, double* r,
                        double* partials, unsigned int* counter, double* sc, double* hist, int it);
__global__ void k_cg_p(long long N, const double* r, double* p, const double* sc);
__global__ void k_manufacture_yd(Phys P, const double* ybar, const double* pbar, double* yd);

// block-tridiagonal format (ocp_block.cu)
// Per line the store keeps the upper triangle of 16x16 tiles of
// W_a = S_a^{-1} P (P swaps the y / p unknowns of every point; W_a is
// symmetric because P J is), by tile columns: tile column c holds columns
// 16c .. 16c+15, rows 0 .. 16c+15, column-major with stride 16c+18 (two pad
// doubles per column keep the transposed reads of the solve free of
// shared-memory bank conflicts and every column 16-byte aligned).  The tile
// columns are laid out in the order 0, cpb-1, 1, cpb-2, ...: the pair
// (k, cpb-1-k) is one contiguous range of 256 cpb + 320 doubles, the unit
// the solve streams.
__host__ __device__ constexpr long long block_col_doubles(int c) { return 16LL * (16 * c + 18); }
__host__ __device__ constexpr long long block_col_off(int c, int cpb) {
  return (c < cpb - 1 - c ? c : cpb - 1 - c) * (256LL * cpb + 320) +
         (c > cpb - 1 - c ? block_col_doubles(cpb - 1 - c) : 0LL);
}
__host__ __device__ constexpr long long block_line_doubles(int nps) {
  return 128LL * (nps / 16) * (nps / 16) + 160LL * (nps / 16);
}
__global__ void k_block_factor(const SubInfo* subs, const int* list, int cnt, Phys P,
                               const double* JDpool, double* fac_pool, double* gscratch,
                               long long gs_stride, int* status);
int block_factor_smem_bytes(int max_npb);
int block_factor_threads();
// few wide subdomains: K CTAs per subdomain (cooperative), Schur blocks in mscratch
cudaError_t launch_block_factor_mc(int cnt, int K, cudaStream_t st, const SubInfo* subs,
                                   const int* list, const Phys* P, const double* JDpool,
                                   double* fac_pool, double* mscratch, long long ms_stride,
                                   int* status, unsigned long long* bars);
size_t block_solve_smem_bytes(int max_npb);
int block_solve_max_nps();
// few wide subdomains: K CTAs per subdomain (cooperative), one barrier per line
cudaError_t launch_block_solve_mc(int mode, int cnt, int K, cudaStream_t st, const SubInfo* subs,
                                  const int* list, const double* fac, const double* in,
                                  double scale, double* out_pool, double off, int max_nps,
                                  const double* dglob, double* oglob, int gn, double* partials,
                                  unsigned long long* bars);
cudaError_t launch_block_solve(int mode, int grid, cudaStream_t st, const SubInfo* subs,
                               const int* list, const double* fac, const double* in, double scale,
                               double* out_pool, double off, int max_npb,
                               const double* dglob = nullptr, double* oglob = nullptr, int gn = 0);
cudaError_t set_block_kernel_smem(int factor_bytes, int solve_bytes);
// narrow-line instance of the block factor (ocp_block_narrow.cu)
int narrow_factor_max_npb();
int narrow_factor_ctas_per_sm();
cudaError_t narrow_set_factor_smem();
cudaError_t launch_narrow_factor(int grid, cudaStream_t st, const SubInfo* subs, const int* list,
                                 int cnt, const Phys* P, const double* JDpool, double* fac_pool,
                                 double* scratch, long long ws_stride, int* status);
// one full MGS Arnoldi step (ocp_krylov.cu); cudaErrorNotSupported if n too large
cudaError_t launch_arnoldi(cudaStream_t st, int num_sms, long long n, const double* Q,
                           long long ldq, int j, const double* w_in, double* partials,
                           double* h_out, unsigned long long* bar, unsigned long long* epoch);

}  // namespace ocp
