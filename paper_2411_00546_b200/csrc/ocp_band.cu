// Batched banded LU factorisation of the local 2-field Jacobians (sm_100a, FP64).
//
// Replaces SuperLU gstrf on the local systems (newton.py:127,
// schwarz.py:305-315).  Each subdomain matrix is generated in-kernel from the
// per-point Jacobian diagonals (no CSR assembly, schwarz.py:166-171): in band
// order (unknown k = 2q + f along the short rectangle side) the 2-field
// Jacobian is banded with half-bandwidth w = 2*nc, and the local systems are
// diagonally dominant (growth factor 1.000), so the
// factorisation runs without pivoting; a zero / nonfinite pivot is reported
// as a singular local Jacobian.
//
// Right-looking blocked LU, panels of NBF = 32 columns, one CTA per
// subdomain (persistent over the work list, 2 CTAs per SM).  Per panel:
//   1. panel (W+32 rows x 32) and U row block (32 x W) -> shared memory;
//   2. the 32x32 diagonal block in two 16x16 levels: a single warp factors a
//      16x16 block in registers (shuffles, no block barrier) and replaces it
//      by its packed triangular inverses; everything else is products with
//      those inverses, all threads in parallel:
//        LU(A_aa);  U_ab = La^-1 A_ab, L_ba = A_ba Ua^-1, X_a = A21_a Ua^-1,
//        Y_a = La^-1 A12_a;  S = A_bb - L_ba U_ab, LU(S)  (warp 0) while the
//        other warps form A21_b - X_a U_ab and A12_b - L_ba Y_a;  then
//        X_b = (.) Uc^-1, Y_b = Lc^-1 (.)       (L21 = [X_a X_b], U12 = [Y_a; Y_b]);
//   3. rank-32 trailing update of the W x W window on the FP64 tensor cores
//      (DMMA m8n8k4, 16x16 warp tiles; measured 37.1 TFLOP/s vs 34.2 for
//      DFMA on this B200, tools/dmma_peak.cu); the window is a circular
//      (W+32)^2 buffer in a per-CTA global scratch that stays L2-resident
//      (0.5 B of L2 traffic per FMA), plus the streaming of the two finished
//      16-blocks to the factor store and the matrix entries entering the window.
//
// Factor store, per 16-block K (the unit the solve kernel streams):
//   [L: 16 x (W+1)  L[k0+c+1+s][k0+c], s < W][U: 16 x (W+1)  U[k0+c][k0+c+s]]
// with the in-block triangles replaced by their inverses: L entries with
// c+1+s < 16 hold (L11^{-1})[c+1+s][c], U entries with c+s < 16 hold
// (U11^{-1})[c][c+s].
#include "ocp_kernels.cuh"

namespace ocp {

constexpr int LDP = NBF + 4; // panel row stride, = 4 (mod 16): conflict-free DMMA A fragments

// original Jacobian entry (i, j) of the padded band-ordered local system
struct RowInfo {
  int i, q, f, b;            // unknown, point, field, position in the grid row
  double dg, cpl;            // diagonal and y<->p coupling of this row
  bool real, padded;
};

__device__ __forceinline__ RowInfo row_info(const SubInfo& s, const double* JD, int i) {
  RowInfo r;
  r.i = i;
  r.real = i < s.N;
  r.padded = i < s.NP;
  r.q = i >> 1;
  r.f = i & 1;
  r.b = r.real ? r.q % s.nc : 0;
  r.dg = r.real ? JD[4 * r.q] : 1.0;
  r.cpl = r.real ? JD[4 * r.q + 1 + r.f] : 0.0;  // b12 on the y row, b21 on the p row
  return r;
}

__device__ __forceinline__ double entry(const SubInfo& s, const RowInfo& r, int j, double off) {
  if (!r.padded || j >= s.NP) return 0.0;
  if (!r.real || j >= s.N) return j == r.i ? 1.0 : 0.0;
  const int d = j - r.i;
  if (d == 0) return r.dg;
  if (d == (r.f == 0 ? 1 : -1)) return r.cpl;
  if (d == 2 * s.nc || d == -2 * s.nc) return off;
  if (d == 2 && r.b != s.nc - 1) return off;
  if (d == -2 && r.b != 0) return off;
  return 0.0;
}


__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One warp: factor the 16x16 block at P[(o+i)*LDP + o+j] (no pivoting) and
// replace it by its packed inverses: strict lower part = (L^-1) (unit
// diagonal implied), upper part incl. diagonal = U^-1.
__device__ __forceinline__ void warp_lu16_inverse(double* P, int o, int lane, int* bad) {
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = P[(o + r) * LDP + o + j];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double piv = __shfl_sync(0xffffffffu, a[c], c);
    if (lane == 0 && !(piv != 0.0 && isfinite(piv))) *bad = 1;
    const double l = a[c] / piv;
#pragma unroll
    for (int j = c + 1; j < 16; ++j) {
      const double pj = __shfl_sync(0xffffffffu, a[j], c);
      if (r > c) a[j] = fma(-l, pj, a[j]);
    }
    if (r > c) a[c] = l;
  }
  if (lane < 16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) P[(o + r) * LDP + o + j] = a[j];
  }
  __syncwarp();
  // column j of L^-1 (lanes 0..15) or of U^-1 (lanes 16..31)
  const int j = lane & 15;
  double x[16];
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double acc = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fma(-P[(o + i) * LDP + o + k], x[k], acc);
      x[i] = i >= j ? acc : 0.0;
    }
  } else {
#pragma unroll
    for (int i = 15; i >= 0; --i) {
      double acc = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = i + 1; k < 16; ++k) acc = fma(-P[(o + i) * LDP + o + k], x[k], acc);
      x[i] = i <= j ? acc / P[(o + i) * LDP + o + i] : 0.0;
    }
  }
  __syncwarp();
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i > j) P[(o + i) * LDP + o + j] = x[i];
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i <= j) P[(o + i) * LDP + o + j] = x[i];
  }
}

// row task: out[0..16) = a[0..16) U^-1, U^-1 packed in the upper part of P block (o, o)
__device__ __forceinline__ void row_times_uinv(double* row, const double* P, int o) {
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = row[k];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k <= c; ++k) acc = fma(a[k], P[(o + k) * LDP + o + c], acc);
    row[c] = acc;
  }
}

// column task: out[t*ld] = (L^-1 a)[t], L^-1 packed in the strict lower part of P block (o, o)
__device__ __forceinline__ void linv_times_col(double* col, int ld, const double* P, int o) {
  double a[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) a[t] = col[t * ld];
#pragma unroll
  for (int t = 15; t >= 0; --t) {
    double acc = a[t];
#pragma unroll
    for (int k = 0; k < t; ++k) acc = fma(P[(o + t) * LDP + o + k], a[k], acc);
    col[t * ld] = acc;
  }
}

__global__ void __launch_bounds__(LU_THREADS, 2)
k_band_factor(const SubInfo* subs, const int* list, int cnt, Phys P_, const double* JDpool,
              double* fac_pool, double* scratch, long long ws_stride, int* status) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* win = scratch + (long long)blockIdx.x * ws_stride;
  for (int li = blockIdx.x; li < cnt; li += gridDim.x) {
    const int sid = list[li];
    const SubInfo s = subs[sid];
    const int W = s.W, WS = W + NBF, NP = s.NP, LD = W + 1, LDU = W + 4;
    const double off = P_.off;
    const double* JD = JDpool + 2 * s.loc;
    double* fac = fac_pool + s.fac;
    double* P = sm;                          // P[r*LDP + c]: panel row k0+r, column k0+c
    double* U = P + (W + NBF) * LDP;         // U[t*LDU + c]: U12 row k0+t, column k0+32+c
    if (tid == 0) bad = 0;
    // initial window [0, WS)^2
    for (int i = warp; i < WS; i += LU_THREADS / 32) {
      const RowInfo r = row_info(s, JD, i);
      for (int j = lane; j < WS; j += 32) win[(long long)i * WS + j] = entry(s, r, j, off);
    }
    __syncthreads();
    const int nblk = NP / NBF;
    int ks = 0;  // k0 mod WS
    for (int K = 0; K < nblk; ++K) {
      const int k0 = K * NBF;
      // ---- 1. panel + U row block -> shared (warp per row, lanes along columns)
      {
        int pcol = ks + lane; pcol -= pcol >= WS ? WS : 0;
        for (int r = warp; r < W + NBF; r += 2 * (LU_THREADS / 32)) {
          int pr0 = ks + r; pr0 -= pr0 >= WS ? WS : 0; pr0 -= pr0 >= WS ? WS : 0;
          const int r1 = r + LU_THREADS / 32;
          int pr1 = ks + r1; pr1 -= pr1 >= WS ? WS : 0; pr1 -= pr1 >= WS ? WS : 0;
          const double v0 = win[(long long)pr0 * WS + pcol];
          const double v1 = r1 < W + NBF ? win[(long long)pr1 * WS + pcol] : 0.0;
          P[r * LDP + lane] = v0;
          if (r1 < W + NBF) P[r1 * LDP + lane] = v1;
        }
        for (int t = warp; t < NBF; t += LU_THREADS / 32) {
          int pr = ks + t; pr -= pr >= WS ? WS : 0;
          const double* src = win + (long long)pr * WS;
          double v[8];
          int nv = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = lane + 32 * q;
            if (c < W) {
              int pc = ks + NBF + c; pc -= pc >= WS ? WS : 0; pc -= pc >= WS ? WS : 0;
              v[q] = src[pc];
              nv = q + 1;
            }
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < nv) U[t * LDU + lane + 32 * q] = v[q];
        }
      }
      __syncthreads();
      // ---- 2a. LU(A_aa) and its inverses (warp 0)
      if (warp == 0) warp_lu16_inverse(P, 0, lane, &bad);
      __syncthreads();
      // ---- 2b. rows 16..W+31, cols 0..15: times Ua^-1  (L_ba and X_a)
      //          cols: P[0..16)[16..32) and U[0..16)[*]: La^-1 times  (U_ab and Y_a)
      for (int task = tid; task < 2 * (W + 16); task += LU_THREADS) {
        if (task < W + 16) row_times_uinv(P + (16 + task) * LDP, P, 0);
        else {
          const int c = task - (W + 16);
          if (c < 16) linv_times_col(P + 16 + c, LDP, P, 0);
          else linv_times_col(U + (c - 16), LDU, P, 0);
        }
      }
      __syncthreads();
      // ---- 2c. warp 0: S = A_bb - L_ba U_ab, LU(S) + inverses;
      //          warps 1..7: A21_b -= X_a U_ab (rows 32..), A12_b -= L_ba Y_a
      if (warp == 0) {
        if (lane < 16) {
          double* row = P + (16 + lane) * LDP + 16;
          double a[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) a[j] = row[j];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const double lk = P[(16 + lane) * LDP + k];
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = fma(-lk, P[k * LDP + 16 + j], a[j]);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) row[j] = a[j];
        }
        __syncwarp();
        warp_lu16_inverse(P, 16, lane, &bad);
      } else {
        for (int task = tid - 32; task < 2 * W; task += LU_THREADS - 32) {
          if (task < W) {  // row 32+task: cols 16..31 -= X_a[row] U_ab
            double* row = P + (NBF + task) * LDP;
            double a[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = row[16 + j];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const double xk = row[k];
#pragma unroll
              for (int j = 0; j < 16; ++j) a[j] = fma(-xk, P[k * LDP + 16 + j], a[j]);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) row[16 + j] = a[j];
          } else {         // column c of U rows 16..31 -= L_ba Y_a[:, c]
            const int c = task - W;
            double y[16], a[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) { y[k] = U[k * LDU + c]; a[k] = U[(16 + k) * LDU + c]; }
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              double acc = a[t];
#pragma unroll
              for (int k = 0; k < 16; ++k) acc = fma(-P[(16 + t) * LDP + k], y[k], acc);
              U[(16 + t) * LDU + c] = acc;
            }
          }
        }
      }
      __syncthreads();
      // ---- 2d. X_b = (.) Uc^-1 (rows 32..), Y_b = Lc^-1 (.) (U rows 16..31)
      for (int task = tid; task < 2 * W; task += LU_THREADS) {
        if (task < W) row_times_uinv(P + (NBF + task) * LDP + 16, P, 16);
        else linv_times_col(U + 16 * LDU + (task - W), LDU, P, 16);
      }
      __syncthreads();
      // ---- 3a. rank-32 trailing update on [k0+32, k0+32+W)^2 with DMMA
      {
        const int TW = W >> 4, g = lane >> 2, t4 = lane & 3;
        for (int wt = warp; wt < TW * TW; wt += LU_THREADS / 32) {
          const int tr = wt / TW, tc = wt - tr * TW;
          const int R0 = 16 * tr, C0 = 16 * tc;
          double c[2][2][2];
          long long addr[2][2];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            int pr = ks + NBF + R0 + 8 * mi + g; pr -= pr >= WS ? WS : 0; pr -= pr >= WS ? WS : 0;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              int pc = ks + NBF + C0 + 8 * ni + 2 * t4; pc -= pc >= WS ? WS : 0; pc -= pc >= WS ? WS : 0;
              addr[mi][ni] = (long long)pr * WS + pc;
              const double2 v = *reinterpret_cast<const double2*>(win + addr[mi][ni]);
              c[mi][ni][0] = v.x;
              c[mi][ni][1] = v.y;
            }
          }
          const double* ap = P + (NBF + R0 + g) * LDP + t4;
          const double* bp = U + t4 * LDU + C0 + g;
#pragma unroll
          for (int kk = 0; kk < NBF; kk += 4) {
            const double a0 = -ap[kk], a1 = -ap[8 * LDP + kk];
            const double b0 = bp[kk * LDU], b1 = bp[kk * LDU + 8];
            dmma_884(c[0][0][0], c[0][0][1], a0, b0);
            dmma_884(c[0][1][0], c[0][1][1], a0, b1);
            dmma_884(c[1][0][0], c[1][0][1], a1, b0);
            dmma_884(c[1][1][0], c[1][1][1], a1, b1);
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
              *reinterpret_cast<double2*>(win + addr[mi][ni]) = make_double2(c[mi][ni][0], c[mi][ni][1]);
        }
      }
      // ---- 3b. stream the two finished 16-blocks to the factor store
      //          (the in-block triangles are the packed inverses in P)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        double* Lb = fac + (long long)(2 * K + b) * 2 * NB * LD;
        double* Ub = Lb + NB * LD;
        const int o = 16 * b;
        for (int c = warp; c < NB; c += LU_THREADS / 32) {
          for (int sidx = lane; sidx < LD; sidx += 32) {
            // L column o+c: rows o+c+1+sidx (inverse entries inside the block)
            Lb[c * LD + sidx] = sidx == W ? 0.0 : P[(o + c + 1 + sidx) * LDP + o + c];
            const int col = o + c + sidx;
            Ub[c * LD + sidx] = col < NBF ? P[(o + c) * LDP + col] : U[(o + c) * LDU + col - NBF];
          }
        }
      }
      // ---- 3c. entries entering the window for panel K+1 (slots of panel K)
      {
        const int base = k0 + NBF + W;             // first new index
        const int band = 2 * s.nc;
        for (int t = warp; t < NBF; t += LU_THREADS / 32) {  // new rows
          const RowInfo r = row_info(s, JD, base + t);
          int prow = ks + t; prow -= prow >= WS ? WS : 0;
          double* dst = win + (long long)prow * WS;
          for (int c = lane; c < W + NBF; c += 32) {
            int pc = ks + NBF + c; pc -= pc >= WS ? WS : 0; pc -= pc >= WS ? WS : 0;
            const int j = k0 + NBF + c, d = j - r.i;
            dst[pc] = (d > band || d < -band) ? 0.0 : entry(s, r, j, off);
          }
        }
        for (int rr = warp; rr < W; rr += LU_THREADS / 32) {  // new columns
          const int i = k0 + NBF + rr, j = base + lane, d = j - i;
          int pr = ks + NBF + rr; pr -= pr >= WS ? WS : 0; pr -= pr >= WS ? WS : 0;
          int pcol = ks + lane; pcol -= pcol >= WS ? WS : 0;
          double v = 0.0;
          if (d <= band) v = entry(s, row_info(s, JD, i), j, off);
          win[(long long)pr * WS + pcol] = v;
        }
      }
      __syncthreads();
      if (bad) break;
      ks += NBF;
      ks -= ks >= WS ? WS : 0;
    }
    if (tid == 0) status[sid] = bad;
    __syncthreads();
  }
}

int factor_smem_bytes(int W) {
  return (int)sizeof(double) * ((W + NBF) * LDP + NBF * (W + 4));
}

}  // namespace ocp
