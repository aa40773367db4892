// Whole-grid operators of the linear-RAS Newton-Krylov method (newton-ras-eps)
// and the RAS preconditioner's scatter (sm_100a, FP64).
//
//   k_global_residual  F_eps(x) on all n^2 points          system.py:147-152
//   k_global_jacdiag   Jacobian diagonals + finite checks  system.py:135-144,155-160
//   k_global_jvp       J(x) d, the CSR row sums of bmat    system.py:155-160
//   k_state_*          the semilinear state equation A y + phi(y) = f + u of
//                      the manufactured problems (system.py:181-197, 257-265):
//                      residual, diagonal of A + diag(phi'(y)), matrix-free CG
//                      steps with device-side scalars, and y_d of _manufacture
//
// Every row sum follows the reference's CSR entry order (columns ascending,
// scipy csr_matvec: sum starts at 0.0, one rounded product and one rounded
// add per stored entry), so results are bitwise those of the reference for
// finite inputs.  Threads run along the global column index: all loads are
// coalesced, the +-1 / +-n neighbours hit L1/L2.
#include "ocp_kernels.cuh"
#include "ocp_reduce.cuh"

namespace ocp {

__global__ void __launch_bounds__(256) k_global_residual(Phys P, const double* __restrict__ x,
                                                         const double* __restrict__ f,
                                                         const double* __restrict__ yd, double eps,
                                                         double* __restrict__ r) {
  const int n = P.n;
  const long long N = (long long)n * n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (long long)i * n);
    const double* y = x;
    const double* p = x + N;
    // A y and A p: kron Laplacian row, columns (i-1,j) (i,j-1) (i,j) (i,j+1) (i+1,j)
    double ay = 0.0, ap = 0.0;
    if (i > 0) { ay = add(ay, mul(P.off, y[k - n])); ap = add(ap, mul(P.off, p[k - n])); }
    if (j > 0) { ay = add(ay, mul(P.off, y[k - 1])); ap = add(ap, mul(P.off, p[k - 1])); }
    const double yk = y[k], pk = p[k];
    ay = add(ay, mul(P.diag, yk));
    ap = add(ap, mul(P.diag, pk));
    if (j < n - 1) { ay = add(ay, mul(P.off, y[k + 1])); ap = add(ap, mul(P.off, p[k + 1])); }
    if (i < n - 1) { ay = add(ay, mul(P.off, y[k + n])); ap = add(ap, mul(P.off, p[k + n])); }
    double r1, r2;
    residual_rows(P, ay, ap, yk, pk, f[k], yd[k], eps, r1, r2);
    r[k] = r1;
    r[N + k] = r2;
  }
}

// JD[k] = (4/h^2 + phi'(y), (1 - P'_eps(-p/mu))/nu, phi''(y) p - 1, 0); the
// reference evaluates phi.derivative / second_derivative with check=True, so
// the first nonfinite entry (phi' before phi'', lowest index) is recorded in
// *bad as (which << 32 | index); *bad must hold ~0 on entry.
__global__ void __launch_bounds__(256) k_global_jacdiag(Phys P, const double* __restrict__ x,
                                                        double eps, double4* __restrict__ JD,
                                                        unsigned long long* bad) {
  const long long N = (long long)P.n * P.n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const double y = x[k], p = x[N + k];
    const double d1 = phi_d1(P, y);
    const double d2 = phi_d2(P, y);
    bool bad1 = !isfinite(d1), bad2 = !isfinite(d2);
    if (P.phi_kind == 0 && P.kappa != 0.0 && mul(P.kappa, y) > 700.0) bad1 = bad2 = true;
    if (P.phi_kind == 2 && y > 700.0) bad1 = bad2 = true;
    if (bad1 || bad2)
      atomicMin(bad, ((bad1 ? 0ull : 1ull) << 32) | (unsigned long long)k);
    const double b12 = dvd(sub(1.0, dp_eps(dvd(-p, P.mu), eps)), P.nu);
    const double b21 = sub(mul(d2, p), 1.0);
    JD[k] = make_double4(add(P.diag, d1), b12, b21, 0.0);
  }
}

// out = J d with J = [[A + diag(phi'), diag(b12)], [diag(b21), A + diag(phi')]]
// (bmat -> CSR, columns ascending: the y row ends with b12 at N+k, the p row
// starts with b21 at k)
__global__ void __launch_bounds__(256) k_global_jvp(Phys P, const double4* __restrict__ JD,
                                                    const double* __restrict__ d,
                                                    double* __restrict__ out) {
  const int n = P.n;
  const long long N = (long long)n * n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (long long)i * n);
    const double* dy = d;
    const double* dp = d + N;
    const double4 jd = JD[k];
    const double dyk = dy[k], dpk = dp[k];
    double sy = 0.0, sp = add(0.0, mul(jd.z, dyk));
    if (i > 0) { sy = add(sy, mul(P.off, dy[k - n])); sp = add(sp, mul(P.off, dp[k - n])); }
    if (j > 0) { sy = add(sy, mul(P.off, dy[k - 1])); sp = add(sp, mul(P.off, dp[k - 1])); }
    sy = add(sy, mul(jd.x, dyk));
    sp = add(sp, mul(jd.x, dpk));
    if (j < n - 1) { sy = add(sy, mul(P.off, dy[k + 1])); sp = add(sp, mul(P.off, dp[k + 1])); }
    if (i < n - 1) { sy = add(sy, mul(P.off, dy[k + n])); sp = add(sp, mul(P.off, dp[k + n])); }
    sy = add(sy, mul(jd.y, dpk));
    out[k] = sy;
    out[N + k] = sp;
  }
}


// ---------------------------------------------------------------------------
// state equation (solve_state, system.py:181-197)
// ---------------------------------------------------------------------------
// (A v)[k] in the kron Laplacian's CSR order with diagonal entry dk
__device__ __forceinline__ double stencil_row(const Phys& P, const double* v, long long k, int i, int j,
                                              double dk) {
  const int n = P.n;
  double s = 0.0;
  if (i > 0) s = add(s, mul(P.off, v[k - n]));
  if (j > 0) s = add(s, mul(P.off, v[k - 1]));
  s = add(s, mul(dk, v[k]));
  if (j < n - 1) s = add(s, mul(P.off, v[k + 1]));
  if (i < n - 1) s = add(s, mul(P.off, v[k + n]));
  return s;
}

// out = A y + phi(y) - rhs   (state_residual, check=False, system.py:188-189)
__global__ void __launch_bounds__(256) k_state_residual(Phys P, const double* __restrict__ y,
                                                        const double* __restrict__ rhs,
                                                        double* __restrict__ out) {
  const int n = P.n;
  const long long N = (long long)n * n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (long long)i * n);
    out[k] = sub(add(stencil_row(P, y, k, i, j, P.diag), phi_value(P, y[k])), rhs[k]);
  }
}

// dg[k] = 4/h^2 + phi'(y_k): the diagonal of (A + diags(phi'(y))).tocsr()
// (state_jacobian, system.py:191-192; phi.derivative checks => *bad)
__global__ void __launch_bounds__(256) k_state_diag(Phys P, const double* __restrict__ y,
                                                    double* __restrict__ dg,
                                                    unsigned long long* bad) {
  const long long N = (long long)P.n * P.n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const double d1 = phi_d1(P, y[k]);
    bool b = !isfinite(d1);
    if (P.phi_kind == 0 && P.kappa != 0.0 && mul(P.kappa, y[k]) > 700.0) b = true;
    if (P.phi_kind == 2 && y[k] > 700.0) b = true;
    if (b) atomicMin(bad, (unsigned long long)k);
    dg[k] = add(P.diag, d1);
  }
}

// CG scalars on the device: sc[0] = r.r, sc[1] = p.Ap, sc[2] = alpha,
// sc[3] = beta; hist[it] = r.r after iteration it
__global__ void __launch_bounds__(RED_THREADS) k_cg_ap(Phys P, const double* __restrict__ dg,
                                                       const double* __restrict__ p,
                                                       double* __restrict__ Ap, double* partials,
                                                       unsigned int* counter, double* sc) {
  __shared__ double red[32];
  // converged (r.r <= thr2 in sc[4]): the host polls every CG_POLL iterations,
  // so later iterations of the batch leave x, r, p and the scalars untouched
  if (sc[0] <= sc[4]) return;
  const int n = P.n;
  const long long N = (long long)n * n;
  double acc = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (long long)i * n);
    const double v = stencil_row(P, p, k, i, j, dg[k]);
    Ap[k] = v;
    acc = fma(p[k], v, acc);
  }
  const double tot = block_sum<RED_THREADS>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
  if (!last_block_done(counter)) return;
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += partials[b];
  const double pap = block_sum<RED_THREADS>(v, red);
  if (threadIdx.x == 0) {
    sc[1] = pap;
    sc[2] = sc[0] / pap;
    *counter = 0u;
  }
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_xr(long long N, const double* __restrict__ p,
                                                       const double* __restrict__ Ap,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* partials, unsigned int* counter,
                                                       double* sc, double* hist, int it) {
  __shared__ double red[32];
  if (sc[0] <= sc[4]) return;   // converged in an earlier iteration of the batch
  const double alpha = sc[2];
  double acc = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    x[k] = fma(alpha, p[k], x[k]);
    const double rk = fma(-alpha, Ap[k], r[k]);
    r[k] = rk;
    acc = fma(rk, rk, acc);
  }
  const double tot = block_sum<RED_THREADS>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
  if (!last_block_done(counter)) return;
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += partials[b];
  const double rr = block_sum<RED_THREADS>(v, red);
  if (threadIdx.x == 0) {
    sc[3] = rr / sc[0];
    sc[0] = rr;
    hist[it] = rr;
    *counter = 0u;
  }
}

__global__ void k_cg_p(long long N, const double* __restrict__ r, double* __restrict__ p,
                       const double* sc) {
  if (sc[0] <= sc[4]) return;   // converged: p is not needed again
  const double beta = sc[3];
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x)
    p[k] = fma(beta, p[k], r[k]);
}

// y_d = y_bar - A p_bar - phi'(y_bar) p_bar   (_manufacture, system.py:263)
__global__ void __launch_bounds__(256) k_manufacture_yd(Phys P, const double* __restrict__ ybar,
                                                        const double* __restrict__ pbar,
                                                        double* __restrict__ yd) {
  const int n = P.n;
  const long long N = (long long)n * n;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N;
       k += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(k / n), j = (int)(k - (long long)i * n);
    yd[k] = sub(sub(ybar[k], stencil_row(P, pbar, k, i, j, P.diag)), mul(phi_d1(P, ybar[k]), pbar[k]));
  }
}

}  // namespace ocp
