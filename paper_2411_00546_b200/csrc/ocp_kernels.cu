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
// Shared-memory halo tiles: a CTA owns a 32x32 tile of the oriented local
// grid.  The (v + alpha d) tile plus its 1-point halo is staged in shared
// memory with loads coalesced in local (band) order; the points are then
// evaluated with threads running fast along the GLOBAL column index, so the
// f / y_d / exterior-ring reads are coalesced for both orientations; the
// residual tile goes back through shared memory to be stored in local order.
constexpr int RT = 32;   // tile edge (oriented points)

__global__ void __launch_bounds__(256, 4) k_residual(const SubInfo* subs, const int* list, Phys P,
                                                  const double* x, const double* Vpool,
                                                  const double* Dpool, const double* alpha,
                                                  const double* f, const double* yd, double eps,
                                                  double* Rpool, double* norm2, double* partials,
                                                  unsigned int* counters) {
  __shared__ double2 tv[(RT + 2) * (RT + 2)];   // halo tile of v + alpha d, [a+1][b+1];
                                                // reused for the residual tile [a][b] (+1 pad)
  double2* tr = tv;
  __shared__ double red[32];
  __shared__ bool is_last;
  const int sid = list[blockIdx.x];
  const SubInfo s = subs[sid];
  const double2* V = reinterpret_cast<const double2*>(Vpool + s.loc);
  const double2* D = Dpool ? reinterpret_cast<const double2*>(Dpool + s.loc) : nullptr;
  double2* R = Rpool ? reinterpret_cast<double2*>(Rpool + s.loc) : nullptr;
  const double al = alpha ? alpha[sid] : 0.0;
  const long long Ntot = (long long)P.n * P.n;
  const int tb_n = (s.nc + RT - 1) / RT;
  const int tile = blockIdx.y;
  const int a0 = (tile / tb_n) * RT, b0 = (tile % tb_n) * RT;
  double acc = 0.0;
  if (a0 < s.nr) {
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;
    const int n = P.n;
    // 0. issue this thread's f / y_d loads first (independent of the tile)
    double fv[RT / 8], ydv[RT / 8];
#pragma unroll
    for (int u = 0; u < RT / 8; ++u) {
      const int k = row + 8 * u;
      const int ta = s.orient == 0 ? k : lane, tbb = s.orient == 0 ? lane : k;
      const int la = a0 + ta, lb = b0 + tbb;
      fv[u] = ydv[u] = 0.0;
      if (la < s.nr && lb < s.nc) {
        int i, j;
        local_to_global(s, la, lb, i, j);
        const long long g = (long long)i * n + j;
        fv[u] = f[g];
        ydv[u] = yd[g];
      }
    }
    // 1. stage the halo tile (local order, coalesced along b); all loads of
    //    this thread are issued before the first use (latency overlap)
    {
      constexpr int HALO = (RT + 2) * (RT + 2);
      constexpr int PER = (HALO + 255) / 256;
      double2 hv[PER], hd[PER];
      unsigned inmask = 0u;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = threadIdx.x + 256 * u;
        const int ta = e / (RT + 2), tbb = e - ta * (RT + 2);
        const int la = a0 + ta - 1, lb = b0 + tbb - 1;
        const bool in = e < HALO && la >= 0 && la < s.nr && lb >= 0 && lb < s.nc;
        inmask |= in ? (1u << u) : 0u;
        hv[u] = in ? V[la * s.nc + lb] : make_double2(0.0, 0.0);
        hd[u] = (in && D) ? D[la * s.nc + lb] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int e = threadIdx.x + 256 * u;
        if (e < HALO) {
          double2 v = hv[u];
          if (D && (inmask >> u & 1u)) {
            v.x = add(v.x, mul(al, hd[u].x));
            v.y = add(v.y, mul(al, hd[u].y));
          }
          tv[e] = v;
        }
      }
    }
    __syncthreads();
    // 2. evaluate, threads fast along the global column
    double2 res[RT / 8];
#pragma unroll
    for (int u = 0; u < RT / 8; ++u) {
      res[u] = make_double2(0.0, 0.0);
      const int k = row + 8 * u;
      // orient 0: global column = b -> (a, b) = (k, lane); orient 1: column = a -> (lane, k)
      const int ta = s.orient == 0 ? k : lane, tbb = s.orient == 0 ? lane : k;
      const int la = a0 + ta, lb = b0 + tbb;
      if (la >= s.nr || lb >= s.nc) continue;
      int i, j;
      local_to_global(s, la, lb, i, j);
      // neighbours in ascending global column order (csr_matvec), local part
      // from the tile, exterior part from the frozen global iterate
      double sly = 0.0, slp = 0.0, sey = 0.0, sep = 0.0;
      const double2* c = tv + (ta + 1) * (RT + 2) + tbb + 1;
      if (la > 0 && la < s.nr - 1 && lb > 0 && lb < s.nc - 1) {
        // interior of the rectangle: all five entries are local; tile
        // offsets of (i-1,j), (i,j-1), (i,j+1), (i+1,j) for this orientation
        const int o1 = s.orient == 0 ? -(RT + 2) : -1;
        const int o2 = s.orient == 0 ? -1 : -(RT + 2);
        const double2 v1 = c[o1], v2 = c[o2], v3 = c[0], v4 = c[-o2], v5 = c[-o1];
        sly = add(0.0, mul(P.off, v1.x));   // csr_matvec starts its sum at 0.0
        slp = add(0.0, mul(P.off, v1.y));
        sly = add(sly, mul(P.off, v2.x));
        slp = add(slp, mul(P.off, v2.y));
        sly = add(sly, mul(P.diag, v3.x));
        slp = add(slp, mul(P.diag, v3.y));
        sly = add(sly, mul(P.off, v4.x));
        slp = add(slp, mul(P.off, v4.y));
        sly = add(sly, mul(P.off, v5.x));
        slp = add(slp, mul(P.off, v5.y));
        sly = add(sly, 0.0);   // the empty exterior part (csr sum of no terms is 0.0)
        slp = add(slp, 0.0);
      } else {
        const int di[5] = {-1, 0, 0, 0, 1};
        const int dj[5] = {0, -1, 0, 1, 0};
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int ii = i + di[t], jj = j + dj[t];
          if (ii < 0 || ii >= n || jj < 0 || jj >= n) continue;
          const double coef = (t == 2) ? P.diag : P.off;
          if (in_rect(s, ii, jj)) {
            // oriented offsets of the neighbour inside the tile (+1 halo)
            const int na = s.orient == 0 ? ii - s.r0 : jj - s.c0;
            const int nbb = s.orient == 0 ? jj - s.c0 : ii - s.r0;
            const double2 v = tv[(na - a0 + 1) * (RT + 2) + (nbb - b0 + 1)];
            sly = add(sly, mul(coef, v.x));
            slp = add(slp, mul(coef, v.y));
          } else {
            const long long g = (long long)ii * n + jj;
            sey = add(sey, mul(coef, x[g]));
            sep = add(sep, mul(coef, x[Ntot + g]));
          }
        }
      }
      const double ay = add(sly, sey), ap = add(slp, sep);
      const double2 v = c[0];
      double r1, r2;
      residual_rows(P, ay, ap, v.x, v.y, fv[u], ydv[u], eps, r1, r2);
      res[u] = make_double2(r1, r2);
      acc = fma(r1, r1, acc);
      acc = fma(r2, r2, acc);
    }
    // 3. residual tile back in local order (through the staging tile)
    if (R) {
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RT / 8; ++u) {
        const int k = row + 8 * u;
        const int ta = s.orient == 0 ? k : lane, tbb = s.orient == 0 ? lane : k;
        tr[ta * (RT + 1) + tbb] = res[u];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < RT * RT; e += blockDim.x) {
        const int ta = e / RT, tbb = e - ta * RT;
        const int la = a0 + ta, lb = b0 + tbb;
        if (la < s.nr && lb < s.nc) R[la * s.nc + lb] = tr[ta * (RT + 1) + tbb];
      }
    }
  }
  const double tot = block_sum<256>(acc, red);
  if (threadIdx.x == 0) {
    partials[(long long)sid * gridDim.y + blockIdx.y] = tot;
    __threadfence();
    const unsigned int ticket = atomicAdd(&counters[sid], 1u);
    is_last = (ticket == gridDim.y - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double v = 0.0;
    for (int y = 0; y < (int)gridDim.y; ++y) v += partials[(long long)sid * gridDim.y + y];
    norm2[sid] = v;
    counters[sid] = 0u;
  }
}

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
// JVP right-hand side e = [a_ext @ dy; a_ext @ dp] in band order
// (schwarz.py:341-342); zero away from the ring
// ---------------------------------------------------------------------------
__global__ void k_jvp_rhs(const SubInfo* subs, Phys P, const double* d, double* Bpool) {
  const SubInfo s = subs[blockIdx.x];
  double2* B = reinterpret_cast<double2*>(Bpool + s.loc);
  const long long Ntot = (long long)P.n * P.n;
  const int n = P.n, npts = s.NP / 2, real = s.nr * s.nc;
  for (int q = blockIdx.y * blockDim.x + threadIdx.x; q < npts; q += gridDim.y * blockDim.x) {
    double ey = 0.0, ep = 0.0;
    if (q < real) {
      int i, j;
      local_to_global(s, q / s.nc, q % s.nc, i, j);
      const int di[4] = {-1, 0, 0, 1};
      const int dj[4] = {0, -1, 1, 0};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int ii = i + di[t], jj = j + dj[t];
        if (ii < 0 || ii >= n || jj < 0 || jj >= n || in_rect(s, ii, jj)) continue;
        const long long g = (long long)ii * n + jj;
        ey = add(ey, mul(P.off, d[g]));
        ep = add(ep, mul(P.off, d[Ntot + g]));
      }
    }
    B[q] = make_double2(ey, ep);
  }
}

// out[own] = -(d_loc + J^{-1} e)[own]   (schwarz.py:343-344)
__global__ void k_jvp_out(const SubInfo* subs, Phys P, const double* d, const double* Zpool,
                          double* out) {
  const SubInfo s = subs[blockIdx.x];
  const double2* Z = reinterpret_cast<const double2*>(Zpool + s.loc);
  const long long Ntot = (long long)P.n * P.n;
  const int oc = s.oc1 - s.oc0, cnt = (s.or1 - s.or0) * oc;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < cnt; e += gridDim.y * blockDim.x) {
    const int i = s.or0 + e / oc, j = s.oc0 + e % oc;
    const long long g = (long long)i * P.n + j;
    const double2 z = Z[global_to_q(s, i, j)];
    out[g] = -add(d[g], z.x);
    out[Ntot + g] = -add(d[Ntot + g], z.y);
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
