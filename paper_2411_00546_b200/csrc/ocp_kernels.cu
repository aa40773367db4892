// Pointwise / stencil / scatter kernels of the RASPEN hot path (sm_100a).
//
// Every value that feeds a Newton decision is computed with explicit
// round-to-nearest operations in the reference's evaluation order
// (system.py:118-144, schwarz.py:174-186, scipy CSR row order), so the local
// residuals match the CPU oracle bitwise for the polynomial phi's.
#include "ocp_kernels.cuh"
#include "ocp_reduce.cuh"

namespace ocp {

// ---------------------------------------------------------------------------
// deterministic block reduction (fixed tree, fixed blockDim)
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// local value of the (optionally line-searched) iterate: v + alpha*d
// (newton.py:106: x + alpha * d, product rounded first)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 lval(const double2* V, const double2* D, double alpha, int q) {
  double2 v = V[q];
  if (D) {
    const double2 d = D[q];
    v.x = add(v.x, mul(alpha, d.x));
    v.y = add(v.y, mul(alpha, d.y));
  }
  return v;
}

// 5-point stencil action on one local point with the exterior ring frozen at
// the global iterate: (a_loc @ v)_q + (a_ext @ x)_q for both fields, each sum
// in ascending global column order starting from 0.0 (csr_matvec), the two
// parts added last (schwarz.py:183).
__device__ __forceinline__ void stencil_point(const SubInfo& s, const Phys& P, const double2* V,
                                              const double2* D, double alpha, const double* x,
                                              long long Ntot, int i, int j, double& ay, double& ap) {
  const int n = P.n;
  double sly = 0.0, slp = 0.0, sey = 0.0, sep = 0.0;
  const int di[5] = {-1, 0, 0, 0, 1};
  const int dj[5] = {0, -1, 0, 1, 0};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int ii = i + di[t], jj = j + dj[t];
    if (ii < 0 || ii >= n || jj < 0 || jj >= n) continue;
    const double coef = (t == 2) ? P.diag : P.off;
    if (in_rect(s, ii, jj)) {
      const double2 v = lval(V, D, alpha, global_to_q(s, ii, jj));
      sly = add(sly, mul(coef, v.x));
      slp = add(slp, mul(coef, v.y));
    } else {
      const long long g = (long long)ii * n + jj;
      sey = add(sey, mul(coef, x[g]));
      sep = add(sep, mul(coef, x[Ntot + g]));
    }
  }
  ay = add(sly, sey);
  ap = add(slp, sep);
}

// ---------------------------------------------------------------------------
// gather v0 = x[pair_idx] into band order (schwarz.py:196)
// ---------------------------------------------------------------------------
__global__ void k_gather(const SubInfo* subs, const int* list, Phys P, const double* x,
                         double* pool) {
  const SubInfo s = subs[list[blockIdx.x]];
  double2* V = reinterpret_cast<double2*>(pool + s.loc);
  const long long Ntot = (long long)P.n * P.n;
  const int npts = s.NP / 2, real = s.nr * s.nc;
  for (int q = threadIdx.x; q < npts; q += blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (q < real) {
      int i, j;
      local_to_global(s, q / s.nc, q % s.nc, i, j);
      const long long g = (long long)i * P.n + j;
      v = make_double2(x[g], x[Ntot + g]);
    }
    V[q] = v;
  }
}

// ---------------------------------------------------------------------------
// local residual (+ squared norm) of the listed subdomains at V + alpha_i D
// _local_problem.local_residual (schwarz.py:181-186); R may be null (trial)
// ---------------------------------------------------------------------------
// A CTA owns RQ consecutive local points q of one subdomain (flat band order
// q = a * nc + b), RQ / RES_THREADS per thread in a ROLLED loop: one compact
// code path for both orientations (the orientation only picks the offsets of
// the four neighbours, taken in ascending global column order) - the
// round-1 kernel unrolled the points and instantiated both orientations,
// 10 k instructions, and lost 12 % of its issue slots to instruction fetch.
//  * D == null (the first residual, the residual of an accepted step): the
//    stencil reads V through L1 - no staging, no barrier; the loads of a
//    point issue right where they are used.
//  * D != null (line-search trial): v + alpha d (newton.py:106: product
//    rounded first) of q in [base - nc, base + RQ + nc) - the CTA's points
//    plus one local row of halo either side - is staged in shared memory
//    once (contiguous, coalesced loads) and the stencil reads that.
// f / y_d are read at the point's global index (coalesced for orient 0,
// per-lane strided rows for orient 1); the residual is stored at q
// (coalesced).  An absent stencil entry is fed as 0.0 instead of branching
// (off * 0.0 = -0.0 and s + -0.0 == s bitwise), so the sums keep the
// reference's CSR order and rounding.  The divisions and square roots of the
// pointwise part are the branch-free div_fast / sqrt_fast / dvd_const_fast
// (ocp_common.cuh; bitwise the IEEE intrinsics on their range); a point with
// an operand outside the range is recomputed with the intrinsics.
// With JD != null the Jacobian diagonals of the same values and eps are
// produced as well - what k_jacdiag would compute next - sharing x = -p/mu,
// the two square roots of P_eps and phi'(y); badkey receives the thread's
// first nonfinite phi'/phi'' (k_jacdiag's packed key).  Every value is
// bitwise k_jacdiag's.
template <bool STAGED>
__device__ __forceinline__ double residual_points(const SubInfo& s, const Phys& P,
                                                  const double* __restrict__ x,
                                                  const double2* __restrict__ V,
                                                  const double* __restrict__ f,
                                                  const double* __restrict__ yd, double eps,
                                                  double2* __restrict__ R, int base,
                                                  double2* __restrict__ JD,
                                                  unsigned long long& badkey,
                                                  const double2* __restrict__ D, double al,
                                                  double2* tv) {
  constexpr int PPT = RQ / RES_THREADS;
  const int nr = s.nr, nc = s.nc, n = P.n, real = nr * nc;
  const long long Ntot = (long long)n * n;
  const float inv_nc = 1.0f / (float)nc;
  const int lo = base - nc;
  if (STAGED) {
    const int cnt = RQ + 2 * nc;
    for (int e = threadIdx.x; e < cnt; e += RES_THREADS) {
      const int q = lo + e;
      double2 v = make_double2(0.0, 0.0);
      if (q >= 0 && q < real) {
        v = V[q];
        const double2 d = D[q];
        v.x = add(v.x, mul(al, d.x));
        v.y = add(v.y, mul(al, d.y));
      }
      tv[e] = v;
    }
    __syncthreads();
  }
  const bool tr = s.orient != 0;
  // neighbour offsets in ascending global column order (csr_matvec):
  // (i-1,j), (i,j-1), (i,j+1), (i+1,j)
  const int o0 = tr ? -1 : -nc, o1 = tr ? -nc : -1, o2 = tr ? nc : 1, o3 = tr ? 1 : nc;
  double acc = 0.0;
#ifndef OCP_RES_UNROLL
#define OCP_RES_UNROLL 1
#endif
  constexpr int UNR = OCP_RES_UNROLL;   // rolled: measured fastest (instruction footprint)
#pragma unroll UNR
  for (int u = 0; u < PPT; ++u) {
    const int q = base + threadIdx.x + RES_THREADS * u;
    if (q >= real) break;
    // q / nc by a float reciprocal (off by at most one for q < 2^24) + fix-up
    int a = __float2int_rz(__int2float_rn(q) * inv_nc), b = q - a * nc;
    if (b < 0) { --a; b += nc; }
    else if (b >= nc) { ++a; b -= nc; }
    const int i = s.r0 + (tr ? b : a), j = s.c0 + (tr ? a : b);
    const long long g0 = (long long)i * n + j;
    const double fv = f[g0], ydv = yd[g0];
    const double2* c = STAGED ? tv + (q - lo) : V + q;
    const double2 cv = c[0];
    const bool fu = a > 0, fd = a < nr - 1, fl = b > 0, fr = b < nc - 1;
    const bool in0 = tr ? fl : fu, in1 = tr ? fu : fl, in2 = tr ? fd : fr, in3 = tr ? fr : fd;
    const double2 zz = make_double2(0.0, 0.0);
    // (an absent neighbour may lie outside the subdomain's vector: not loaded)
    const double2 n0 = in0 ? c[o0] : zz, n1 = in1 ? c[o1] : zz, n2 = in2 ? c[o2] : zz, n3 = in3 ? c[o3] : zz;
    // local part, exterior part from the frozen global iterate; off * 0.0 =
    // -0.0 and s + -0.0 == s bitwise for every s, so an absent entry
    // contributes exactly nothing
    double sly = 0.0, slp = 0.0;
    sly = add(sly, mul(P.off, n0.x)); slp = add(slp, mul(P.off, n0.y));
    sly = add(sly, mul(P.off, n1.x)); slp = add(slp, mul(P.off, n1.y));
    sly = add(sly, mul(P.diag, cv.x)); slp = add(slp, mul(P.diag, cv.y));
    sly = add(sly, mul(P.off, n2.x)); slp = add(slp, mul(P.off, n2.y));
    sly = add(sly, mul(P.off, n3.x)); slp = add(slp, mul(P.off, n3.y));
    double sey = 0.0, sep = 0.0;
    if (!(in0 && in1 && in2 && in3)) {
      const bool in[4] = {in0, in1, in2, in3};
      const int di[4] = {-1, 0, 0, 1};
      const int dj[4] = {0, -1, 1, 0};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int ii = i + di[t], jj = j + dj[t];
        if (in[t] || ii < 0 || ii >= n || jj < 0 || jj >= n) continue;
        const long long g = (long long)ii * n + jj;
        sey = add(sey, mul(P.off, x[g]));
        sep = add(sep, mul(P.off, x[Ntot + g]));
      }
    }
    const double ay = add(sly, sey), ap = add(slp, sep);
    const double y = cv.x, p = cv.y;
    // residual_rows (system.py:118-132) with the smoothed projection's parts kept
    bool slow = false;
    double xm = dvd_const_fast(-p, P.mu, P.rmu, slow), a1 = add(xm, 1.0), b1 = sub(xm, 1.0);
    double sa = sqrt_fast(add(mul(a1, a1), eps), slow), sb = sqrt_fast(add(mul(b1, b1), eps), slow);
    const double d1 = phi_d1(P, y);
    double ctrl = dvd_const_fast(add(p, mul(P.mu, mul(0.5, sub(sa, sb)))), P.nu, P.rnu, slow);
    double b12 = 0.0;
    if (JD) b12 = dvd_const_fast(sub(1.0, mul(0.5, sub(div_fast(a1, sa, slow), div_fast(b1, sb, slow)))), P.nu, P.rnu, slow);
    if (slow) {
      xm = dvd_const(-p, P.mu, P.rmu), a1 = add(xm, 1.0), b1 = sub(xm, 1.0);
      sa = __dsqrt_rn(add(mul(a1, a1), eps)), sb = __dsqrt_rn(add(mul(b1, b1), eps));
      ctrl = dvd_const(add(p, mul(P.mu, mul(0.5, sub(sa, sb)))), P.nu, P.rnu);
      if (JD) b12 = dvd_const(sub(1.0, mul(0.5, sub(dvd(a1, sa), dvd(b1, sb)))), P.nu, P.rnu);
    }
    const double r1 = add(sub(add(ay, phi_value(P, y)), fv), ctrl);
    const double r2 = add(sub(add(ap, mul(d1, p)), y), ydv);
    acc = fma(r1, r1, acc);
    acc = fma(r2, r2, acc);
    if (R) R[q] = make_double2(r1, r2);
    if (JD) {   // jacobian_diagonals (system.py:135-144), k_jacdiag's operation order
      const double d2 = phi_d2(P, y);
      bool bad1 = !isfinite(d1), bad2 = !isfinite(d2);
      if (P.phi_kind == 0 && P.kappa != 0.0 && mul(P.kappa, y) > 700.0) bad1 = bad2 = true;
      if (P.phi_kind == 2 && y > 700.0) bad1 = bad2 = true;
      if (bad1 || bad2) {
        const unsigned long long ref = (unsigned long long)((i - s.r0) * (s.c1 - s.c0) + (j - s.c0));
        const unsigned long long key = ((bad1 ? 0ull : 1ull) << 32) | ref;
        badkey = key < badkey ? key : badkey;
      }
      const double b21 = sub(mul(d2, p), 1.0);
      JD[2 * q] = make_double2(add(P.diag, d1), b12);
      JD[2 * q + 1] = make_double2(b21, 0.0);
    }
  }
  return acc;
}

size_t residual_smem_bytes(int max_nc) { return (size_t)(RQ + 2 * max_nc) * sizeof(double2); }

template <bool DIRECT>
__global__ void __launch_bounds__(RES_THREADS, OCP_RES_MINB) k_residual(const SubInfo* subs, const int* list, Phys P,
                                                      const double* x, const double* Vpool,
                                                      const double* Dpool, const double* alpha,
                                                      const double* f, const double* yd, double eps,
                                                      double* Rpool, double* partials,
                                                      double* JDpool, unsigned long long* badparts) {
  extern __shared__ double2 tv[];
  __shared__ double red[32];
  __shared__ unsigned long long bmin;
  const int sid = list ? list[blockIdx.x] : blockIdx.x;   // null list: all subdomains
  const SubInfo s = subs[sid];
  const double2* V = reinterpret_cast<const double2*>(Vpool + s.loc);
  const double2* D = Dpool ? reinterpret_cast<const double2*>(Dpool + s.loc) : nullptr;
  double2* R = Rpool ? reinterpret_cast<double2*>(Rpool + s.loc) : nullptr;
  const double al = alpha ? alpha[sid] : 0.0;
  const int base = blockIdx.y * RQ;
  double2* JD = JDpool ? reinterpret_cast<double2*>(JDpool + 2 * s.loc) : nullptr;
  if (JD && threadIdx.x == 0) bmin = ~0ull;
  double acc = 0.0;
  unsigned long long key = ~0ull;
  if (base < s.nr * s.nc) {
    acc = residual_points<!DIRECT>(s, P, x, V, f, yd, eps, R, base, JD, key, D, al, tv);
  }
  if (JD && key != ~0ull) atomicMin(&bmin, key);   // (bmin set before the staging barrier)
  const double tot = block_sum<RES_THREADS>(acc, red);
  // one squared-norm partial (and first-bad key) per CTA; the host adds a
  // subdomain's partials in CTA order after the copy it makes anyway, so a
  // CTA ends without a fence / ticket round trip holding its SM slot
  if (threadIdx.x == 0) {
    partials[(long long)sid * gridDim.y + blockIdx.y] = tot;
    if (JD) badparts[(long long)sid * gridDim.y + blockIdx.y] = bmin;
  }
}

template __global__ void k_residual<false>(const SubInfo*, const int*, Phys, const double*, const double*,
                                           const double*, const double*, const double*, const double*,
                                           double, double*, double*, double*, unsigned long long*);
template __global__ void k_residual<true>(const SubInfo*, const int*, Phys, const double*, const double*,
                                          const double*, const double*, const double*, const double*,
                                          double, double*, double*, double*, unsigned long long*);

// ---------------------------------------------------------------------------
// Jacobian diagonals per point (system.py:135-144) + the reference's finite
// checks of phi'(y) and phi''(y) (system.py:56-74, check=True)
// JD: 4 doubles per point: (4/h^2 + phi'(y), b12, b21, 0)
// bad: per subdomain packed (which << 32 | first reference index), or -1
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_jacdiag(const SubInfo* subs, const int* list, Phys P,
                                                 const double* Vpool, double eps, double* JDpool,
                                                 long long* bad) {
  const int sid = list[blockIdx.x];
  const SubInfo s = subs[sid];
  const double2* V = reinterpret_cast<const double2*>(Vpool + s.loc);
  double* JD = JDpool + 2 * s.loc;
  const int real = s.nr * s.nc;
  __shared__ unsigned long long first;
  if (threadIdx.x == 0) first = ~0ull;
  __syncthreads();
  for (int q = threadIdx.x; q < real; q += blockDim.x) {
    const double2 v = V[q];
    const double y = v.x, p = v.y;
    const double d1 = phi_d1(P, y);
    const double d2 = phi_d2(P, y);
    bool bad1 = !isfinite(d1), bad2 = !isfinite(d2);
    if (P.phi_kind == 0 && P.kappa != 0.0 && mul(P.kappa, y) > 700.0) bad1 = bad2 = true;
    if (P.phi_kind == 2 && y > 700.0) bad1 = bad2 = true;
    if (bad1 || bad2) {
      // reference index: row-major position in the rectangle
      int i, j;
      local_to_global(s, q / s.nc, q % s.nc, i, j);
      const unsigned long long ref = (unsigned long long)((i - s.r0) * (s.c1 - s.c0) + (j - s.c0));
      const unsigned long long key = ((bad1 ? 0ull : 1ull) << 32) | ref;
      atomicMin(&first, key);
    }
    const double b12 = dvd(sub(1.0, dp_eps(dvd(-p, P.mu), eps)), P.nu);
    const double b21 = sub(mul(d2, p), 1.0);
    reinterpret_cast<double2*>(JD)[2 * q] = make_double2(add(P.diag, d1), b12);
    reinterpret_cast<double2*>(JD)[2 * q + 1] = make_double2(b21, 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) bad[sid] = first == ~0ull ? -1ll : (long long)first;
}

// ---------------------------------------------------------------------------
// v += alpha_i d (newton.py:169) for the listed subdomains
// ---------------------------------------------------------------------------
__global__ void k_update(const SubInfo* subs, const int* list, double* Vpool, const double* Dpool,
                         const double* alpha) {
  const int sid = list[blockIdx.x];
  const SubInfo s = subs[sid];
  double2* V = reinterpret_cast<double2*>(Vpool + s.loc);
  const double2* D = reinterpret_cast<const double2*>(Dpool + s.loc);
  const double a = alpha[sid];
  const int real = s.nr * s.nc;
  for (int q = threadIdx.x; q < real; q += blockDim.x) {
    double2 v = V[q];
    const double2 d = D[q];
    v.x = add(v.x, mul(a, d.x));
    v.y = add(v.y, mul(a, d.y));
    V[q] = v;
  }
}

// ---------------------------------------------------------------------------
// restricted prolongation: fval[own] = values[own_in_local] - x[own]
// (_scatter_own + "- x", schwarz.py:247-250,317); grid (I, chunks)
// ---------------------------------------------------------------------------
__global__ void k_scatter_fval(const SubInfo* subs, Phys P, const double* Vpool, const double* x,
                               double* fval) {
  const SubInfo s = subs[blockIdx.x];
  const double2* V = reinterpret_cast<const double2*>(Vpool + s.loc);
  const long long Ntot = (long long)P.n * P.n;
  const int oc = s.oc1 - s.oc0, cnt = (s.or1 - s.or0) * oc;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < cnt; e += gridDim.y * blockDim.x) {
    const int i = s.or0 + e / oc, j = s.oc0 + e % oc;
    const long long g = (long long)i * P.n + j;
    const double2 v = V[global_to_q(s, i, j)];
    fval[g] = sub(v.x, x[g]);
    fval[Ntot + g] = sub(v.y, x[Ntot + g]);
  }
}



// ---------------------------------------------------------------------------
// layout conversion between the reference local layout ([y_loc; p_loc],
// rectangle row-major) and band order
// ---------------------------------------------------------------------------
__global__ void k_ref_to_band(const SubInfo* subs, const double* ref, double* pool) {
  const SubInfo s = subs[blockIdx.x];
  const int C = s.c1 - s.c0, size = (s.r1 - s.r0) * C;
  const double* src = ref + s.ref;
  double2* V = reinterpret_cast<double2*>(pool + s.loc);
  const int npts = s.NP / 2;
  for (int q = threadIdx.x; q < npts; q += blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (q < size) {
      int i, j;
      local_to_global(s, q / s.nc, q % s.nc, i, j);
      const int rr = (i - s.r0) * C + (j - s.c0);
      v = make_double2(src[rr], src[size + rr]);
    }
    V[q] = v;
  }
}

__global__ void k_band_to_ref(const SubInfo* subs, const double* pool, double* ref) {
  const SubInfo s = subs[blockIdx.x];
  const int C = s.c1 - s.c0, size = (s.r1 - s.r0) * C;
  double* dst = ref + s.ref;
  const double2* V = reinterpret_cast<const double2*>(pool + s.loc);
  for (int rr = threadIdx.x; rr < size; rr += blockDim.x) {
    const int i = s.r0 + rr / C, j = s.c0 + rr % C;
    const double2 v = V[global_to_q(s, i, j)];
    dst[rr] = v.x;
    dst[size + rr] = v.y;
  }
}

// ---------------------------------------------------------------------------
// vector kernels for GMRES (krylov.py), grid-stride, deterministic
// "last block reduces" pattern: partials in fixed slots, the last block to
// finish sums them in a fixed tree.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void finish_reduction(double* partials, unsigned int* counter,
                                                 double* result, bool take_sqrt, double* red) {
  if (!last_block_done(counter)) return;
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += partials[b];
  const double tot = block_sum<RED_THREADS>(v, red);
  if (threadIdx.x == 0) {
    *result = take_sqrt ? sqrt(tot) : tot;
    *counter = 0u;
  }
}

__global__ void __launch_bounds__(RED_THREADS) k_dot(long long n, const double* x, const double* y,
                                                     double* partials, unsigned int* counter,
                                                     double* result, int take_sqrt) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    acc = fma(x[e], y[e], acc);
  const double tot = block_sum<RED_THREADS>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
  finish_reduction(partials, counter, result, take_sqrt != 0, red);
}

// MGS pass i (krylov.py:113-116): w -= h_prev * q_prev (if has_prev), then
// partial q_i . w (or ||w||^2 when q_i is null) -> h_out
__global__ void __launch_bounds__(RED_THREADS) k_mgs_pass(long long n, double* w, const double* q_prev,
                                                          const double* h_prev, const double* q_i,
                                                          double* partials, unsigned int* counter,
                                                          double* h_out) {
  __shared__ double red[32];
  const double hp = q_prev ? *h_prev : 0.0;
  double acc = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    double we = w[e];
    if (q_prev) {
      we = sub(we, mul(hp, q_prev[e]));
      w[e] = we;
    }
    acc = q_i ? fma(q_i[e], we, acc) : fma(we, we, acc);
  }
  const double tot = block_sum<RED_THREADS>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
  finish_reduction(partials, counter, h_out, q_i == nullptr, red);
}

__global__ void k_add_scaled(long long n, const double* x, double alpha, const double* d, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = add(x[e], mul(alpha, d[e]));
}

__global__ void k_scale(long long n, double a, const double* x, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = mul(a, x[e]);
}

__global__ void k_div(long long n, const double* x, double s, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = dvd(x[e], s);
}

__global__ void k_flags(long long n, const double* x, const double* y, int* flag) {
  // flag[0] cleared if x != y (bitwise, numpy.array_equal on floats: NaN != NaN);
  // flag[1] cleared if x has a nonfinite entry
  bool neq = false, nonfin = false;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const double a = x[e];
    if (y && !(a == y[e])) neq = true;
    if (!isfinite(a)) nonfin = true;
  }
  if (__syncthreads_or(neq) && threadIdx.x == 0) flag[0] = 0;
  if (__syncthreads_or(nonfin) && threadIdx.x == 0) flag[1] = 0;
}

// out = x + Q[:, :k] y, sum over columns in index order (krylov.py:151)
__global__ void k_gemv_add(long long n, const double* Q, long long ldq, int k, const double* y,
                           const double* x, double* out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < k; ++c) acc = fma(Q[c * ldq + e], y[c], acc);
    out[e] = add(x[e], acc);
  }
}

__global__ void k_recover_control(long long n, Phys P, const double* p, double eps, double* u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const double pe = p[e];
    const double proj = eps == 0.0 ? fmin(fmax(dvd(-pe, P.mu), -1.0), 1.0)
                                   : p_eps(dvd(-pe, P.mu), eps);
    u[e] = dvd(-add(pe, mul(P.mu, proj)), P.nu);
  }
}

}  // namespace ocp
