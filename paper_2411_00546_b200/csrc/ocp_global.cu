// Whole-grid operators of the linear-RAS Newton-Krylov method (newton-ras-eps)
// and the RAS preconditioner's scatter (sm_100a, FP64).
//
//   k_global_residual  F_eps(x) on all n^2 points          system.py:147-152
//   k_global_jacdiag   Jacobian diagonals + finite checks  system.py:135-144,155-160
//   k_global_jvp       J(x) d, the CSR row sums of bmat    system.py:155-160
//   k_ras_out          out[own_i] = z_i[own_in_local]       schwarz.py:234-239
//
// Every row sum follows the reference's CSR entry order (columns ascending,
// scipy csr_matvec: sum starts at 0.0, one rounded product and one rounded
// add per stored entry), so results are bitwise those of the reference for
// finite inputs.  Threads run along the global column index: all loads are
// coalesced, the +-1 / +-n neighbours hit L1/L2.
#include "ocp_kernels.cuh"

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

// restricted prolongation of the local solutions: out[own_i] = z_i (band order)
__global__ void k_ras_out(const SubInfo* subs, Phys P, const double* Zpool, double* out) {
  const SubInfo s = subs[blockIdx.x];
  const double2* Z = reinterpret_cast<const double2*>(Zpool + s.loc);
  const long long Ntot = (long long)P.n * P.n;
  const int oc = s.oc1 - s.oc0, cnt = (s.or1 - s.or0) * oc;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < cnt; e += gridDim.y * blockDim.x) {
    const int i = s.or0 + e / oc, j = s.oc0 + e % oc;
    const long long g = (long long)i * P.n + j;
    const double2 z = Z[global_to_q(s, i, j)];
    out[g] = z.x;
    out[Ntot + g] = z.y;
  }
}

}  // namespace ocp
