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
//      16x16 block in registers (shuffles, no block barrier); the rest are
//      independent 16-wide triangular solves, all threads in parallel:
//        LU(A_aa);  U_ab = La^-1 A_ab, L_ba = A_ba Ua^-1, X_a = A21_a Ua^-1,
//        Y_a = La^-1 A12_a;  S = A_bb - L_ba U_ab, LU(S)  (warp 0) while the
//        other warps form A21_b - X_a U_ab and A12_b - L_ba Y_a;  then
//        X_b = (.) Uc^-1, Y_b = Lc^-1 (.)       (L21 = [X_a X_b], U12 = [Y_a; Y_b]);
//   3. rank-32 trailing update of the W x W window on the FP64 tensor cores
//      (DMMA m8n8k4, 16x16 warp tiles; measured 37.1 TFLOP/s vs 34.2 for
//      DFMA on this B200, tools/dmma_peak.cu); the window is a circular
//      (W+32)^2 buffer in a per-CTA global scratch that stays L2-resident
//      (0.5 B of L2 traffic per FMA).  Entries no panel has updated yet are
//      never stored: they are generated from the Jacobian diagonals where
//      they are first read.  One warp forms the 16x16 triangular inverses the
//      solve kernel uses (off the serial path), then all warps stream the
//      finished 16-blocks to the factor store.
//
// Factor store, per 32-block K (the unit the solve kernel streams):
//   [L: 32 x (W+1)  L[k0+c+1+s][k0+c], s < W][U: 32 x (W+1)  U[k0+c][k0+c+s]]
// with the in-block triangles replaced by their inverses: L entries with
// c+1+s < 32 hold (L11^{-1})[c+1+s][c], U entries with c+s < 32 hold
// (U11^{-1})[c][c+s].
#include "ocp_kernels.cuh"

namespace ocp {

// optional per-phase cycle counters (build with -DOCP_PHASE_TIMING; tools/phase_dbg.py)
#ifdef OCP_PHASE_TIMING
__device__ unsigned long long g_phase[8];
#define PHASE_START() long long t_last = clock64()
#define PHASE_MARK(k)                                                                   \
  do {                                                                                  \
    if (tid == 0) {                                                                     \
      const long long now = clock64();                                                  \
      atomicAdd(&g_phase[k], (unsigned long long)(now - t_last));                       \
      t_last = now;                                                                     \
    }                                                                                   \
  } while (0)
#else
#define PHASE_START() (void)0
#define PHASE_MARK(k) (void)0
#endif
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

// Reciprocal without the IEEE slow path (no call => nothing spills around it):
// MUFU seed + two Newton steps, ~1 ulp; pivots here are O(1/h^2) normal numbers.
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// One warp factors the 16x16 block at P[(o+i)*LDP + o+j] in place (no
// pivoting; L strict lower, U upper) and stores 1/U[i][i] in rd[i].
// Compact on purpose: the step loop is not unrolled (the kernel's hot loop
// must stay small for the instruction cache); lane r < 16 owns row r, loads
// the pivot row and its own row into registers, updates, stores.
__device__ __noinline__ void warp_lu16(double* P, int o, int lane, double* rd, int* bad) {
  __syncwarp();
  const int r = lane & 15;
  double* prow = P + (o + r) * LDP + o;
#pragma unroll 1
  for (int c = 0; c < 16; ++c) {
    const double* pc = P + (o + c) * LDP + o;
    double pv[16], a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) { pv[j] = pc[j]; a[j] = prow[j]; }
    const double piv = pc[c];
    const double rp = fast_rcp(piv);
    if (lane == 0) {
      rd[c] = rp;
      if (!(piv != 0.0 && isfinite(piv))) *bad = 1;
    }
    __syncwarp();
    if (lane < 16 && r > c) {
      const double l = prow[c] * rp;
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] = j > c ? fma(-l, pv[j], a[j]) : (j == c ? l : a[j]);
#pragma unroll
      for (int j = 0; j < 16; ++j) prow[j] = a[j];
    }
    __syncwarp();
  }
}

// row task: x U = a for the upper factor U at P block (o, o), in place on row[0..16)
__device__ __forceinline__ void row_solve_u(double* row, const double* P, int o, const double* rd) {
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = row[k];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    a[c] *= rd[c];
#pragma unroll
    for (int j = c + 1; j < 16; ++j) a[j] = fma(-a[c], P[(o + c) * LDP + o + j], a[j]);
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) row[k] = a[k];
}

// column task: L y = a for the unit lower factor L at P block (o, o), in place on col[t*ld]
__device__ __forceinline__ void col_solve_l(double* col, int ld, const double* P, int o) {
  double a[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) a[t] = col[t * ld];
#pragma unroll
  for (int k = 0; k < 16; ++k)
#pragma unroll
    for (int t = k + 1; t < 16; ++t) a[t] = fma(-P[(o + t) * LDP + o + k], a[k], a[t]);
#pragma unroll
  for (int t = 0; t < 16; ++t) col[t * ld] = a[t];
}

// lane j < 16: column j of the unit-lower inverse of L at block (o, o);
// lane 16 + j: column j of the inverse of U.  Result entry i in x[i].
__device__ __forceinline__ void tri_inverse_lane(const double* P, int o, int lane, const double* rd,
                                                 double* x) {
  const int j = lane & 15;
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
      x[i] = i <= j ? acc * rd[i] : 0.0;
    }
  }
}

__global__ void __launch_bounds__(LU_THREADS, 2)
k_band_factor(const SubInfo* subs, const int* list, int cnt, Phys P_, const double* JDpool,
              double* fac_pool, double* scratch, long long ws_stride, int* status) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int bad;
  __shared__ double rd[2][16];  // reciprocal pivots of U_aa, U_cc
  __shared__ double Pn[16 * LDP];   // next panel's A_aa, factored ahead (lookahead)
  __shared__ double rdn[16];
  __shared__ int tile_ctr;          // dynamic tile scheduler of the update phase
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = LU_THREADS / 32;
  constexpr int SIDE = NW - 1;  // forms the block inverses at the start of the update phase
  constexpr int LAW = 0;        // lookahead warp: factors the next panel's A_aa during the update
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
    __syncthreads();
    const int nblk = NP / NBF;
    int ks = 0;  // k0 mod WS
    for (int K = 0; K < nblk; ++K) {
      const int k0 = K * NBF;
      PHASE_START();
      // ---- 1. panel + U row block -> shared (warp per row, lanes along columns).
      //         An entry (i, j) has been touched by an earlier panel update iff
      //         K > 0 and max(i, j) < k0 + W; all others still hold their
      //         original value and are generated here instead of stored.
      //         Loads are issued in batches before any use (latency overlap).
      {
        const int fresh = K == 0 ? k0 : k0 + W;   // indices >= fresh are untouched
        int pcol = ks + lane; pcol -= pcol >= WS ? WS : 0;
        constexpr int PB = 8;
        for (int r0 = warp; r0 < W + NBF; r0 += PB * NW) {
          double v[PB];
#pragma unroll
          for (int q = 0; q < PB; ++q) {
            const int r = r0 + q * NW;
            int pr = ks + r; pr -= pr >= WS ? WS : 0; pr -= pr >= WS ? WS : 0;
            v[q] = (r < W + NBF && k0 + r < fresh && k0 + lane < fresh)
                       ? win[(long long)pr * WS + pcol] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < PB; ++q) {
            const int r = r0 + q * NW, i = k0 + r;
            if (r < W + NBF) {
              if (i >= fresh || k0 + lane >= fresh) v[q] = entry(s, row_info(s, JD, i), k0 + lane, off);
              if (K > 0 && r < 16 && lane < 16) v[q] = Pn[r * LDP + lane];  // factored ahead
              P[r * LDP + lane] = v[q];
            }
          }
        }
        for (int t = warp; t < NBF; t += NW) {
          const int i = k0 + t;
          int pr = ks + t; pr -= pr >= WS ? WS : 0;
          const double* src = win + (long long)pr * WS;
          double v[8];
          int pc = ks + NBF + lane; pc -= pc >= WS ? WS : 0; pc -= pc >= WS ? WS : 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = lane + 32 * q, j = k0 + NBF + c;
            v[q] = (c < W && j < fresh && i < fresh) ? src[pc] : 0.0;
            pc += 32;
            pc -= pc >= WS ? WS : 0;
          }
          const RowInfo ri = row_info(s, JD, i);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = lane + 32 * q, j = k0 + NBF + c;
            if (c < W) U[t * LDU + c] = (j >= fresh || i >= fresh) ? entry(s, ri, j, off) : v[q];
          }
        }
      }
      __syncthreads();
      // ---- 2a. LU(A_aa) (warp 0); from the second panel on it was factored
      //          during the previous update phase (lookahead warp)
      if (K == 0) {
        if (warp == 0) warp_lu16(P, 0, lane, rd[0], &bad);
      } else if (tid < 16) {
        rd[0][tid] = rdn[tid];
      }
      __syncthreads();
      PHASE_MARK(2);
      // ---- 2b/2c. warp 0: L_ba, U_ab (the 16x16 blocks next to A_aa), then
      //          S = A_bb - L_ba U_ab and LU(S), announcing L_ba/U_ab on named
      //          barrier 1 before the serial LU(S);
      //          warps 1..7: X_a (rows 32..) against U_aa, Y_a (U rows 0..15)
      //          against L_aa, then (after barrier 1) A21_b -= X_a U_ab and
      //          A12_b -= L_ba Y_a, overlapped with LU(S)
      if (warp == 0) {
        if (lane < 16) row_solve_u(P + (16 + lane) * LDP, P, 0, rd[0]);
        else col_solve_l(P + lane, LDP, P, 0);
        __syncwarp();
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
        asm volatile("bar.arrive 1, %0;" :: "n"(LU_THREADS) : "memory");
        warp_lu16(P, 16, lane, rd[1], &bad);
      } else {
        for (int task = tid - 32; task < 2 * W; task += LU_THREADS - 32) {
          if (task < W) row_solve_u(P + (NBF + task) * LDP, P, 0, rd[0]);
          else col_solve_l(U + (task - W), LDU, P, 0);
        }
        asm volatile("bar.sync 1, %0;" :: "n"(LU_THREADS) : "memory");
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
      PHASE_MARK(4);
      // ---- 2d. X_b solve against U_cc (rows 32..), Y_b against L_cc (U rows 16..31)
      if (tid == 0) tile_ctr = 1;   // tile 0 belongs to the lookahead warp
      for (int task = tid; task < 2 * W; task += LU_THREADS) {
        if (task < W) row_solve_u(P + (NBF + task) * LDP + 16, P, 16, rd[1]);
        else col_solve_l(U + 16 * LDU + (task - W), LDU, P, 16);
      }
      __syncthreads();
      PHASE_MARK(5);
      // ---- 3a. side warp: the 32x32 inverses of L11 and U11 (the solve kernel
      //          applies them as mat-vecs), written in place of the in-block
      //          triangles of the factor store:
      //            L11^-1 = [[La^-1, 0], [X, Lc^-1]],  X = -Lc^-1 L_ba La^-1
      //            U11^-1 = [[Ua^-1, Y], [0, Uc^-1]],  Y = -Ua^-1 U_ab Uc^-1
      if (warp == SIDE) {
        double* Lb = fac + (long long)K * 2 * NBF * LD;
        double* Ub = Lb + NBF * LD;
        const int j = lane & 15;
        double x[16], z[16];
        tri_inverse_lane(P, 0, lane, rd[0], x);    // La^-1 / Ua^-1 column j
        tri_inverse_lane(P, 16, lane, rd[1], z);   // Lc^-1 / Uc^-1 column j
        if (lane < 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i > j) __stcs(Lb + j * LD + i - j - 1, x[i]);                 // La^-1
            if (i > j) __stcs(Lb + (16 + j) * LD + i - j - 1, z[i]);          // Lc^-1
          }
          // X[:, j] = Lc^-1 (-L_ba La^-1[:, j]): forward substitution with unit Lc
          double t[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = fma(-P[(16 + i) * LDP + k], x[k], acc);
            t[i] = acc;
          }
#pragma unroll
          for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int i = k + 1; i < 16; ++i) t[i] = fma(-P[(16 + i) * LDP + 16 + k], t[k], t[i]);
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcs(Lb + j * LD + (16 + i) - j - 1, t[i]);   // X[i][j]
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i <= j) __stcs(Ub + i * LD + j - i, x[i]);                    // Ua^-1
            if (i <= j) __stcs(Ub + (16 + i) * LD + j - i, z[i]);             // Uc^-1
          }
          // Y[:, j] = Ua^-1 (-U_ab Uc^-1[:, j]): back substitution with Ua
          double t[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 16; ++k) acc = fma(-P[i * LDP + 16 + k], z[k], acc);
            t[i] = acc;
          }
#pragma unroll
          for (int k = 15; k >= 0; --k) {
            t[k] *= rd[0][k];
#pragma unroll
            for (int i = 0; i < k; ++i) t[i] = fma(-P[i * LDP + k], t[k], t[i]);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcs(Ub + i * LD + (16 + j) - i, t[i]);   // Y[i][j]
        }
      }
      // ---- 3b. rank-32 trailing update on [k0+32, k0+32+W)^2 with DMMA,
      //          32x16 warp tiles (4x2 m8n8k4 tiles, 8 independent accumulators)
      {
        const int g = lane >> 2, t4 = lane & 3;
        const int TR = (W + 31) >> 5, TC = W >> 4;     // last tile row may be 16 rows
        const int fresh = K == 0 ? k0 : k0 + W;        // indices >= fresh never updated
        // dynamic tile scheduling: the lookahead warp takes tile 0 first, the
        // side warp starts with the inverses; everybody then pulls tiles
        int wt = warp == LAW ? 0 : -1;
        for (;;) {
          if (wt < 0) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&tile_ctr, 1);
            wt = __shfl_sync(0xffffffffu, t, 0);
          }
          if (wt >= TR * TC) break;
          const int tr = wt / TC, tc = wt - tr * TC;
          const int R0 = 32 * tr, C0 = 16 * tc;
          const int mrows = (W - R0) >= 32 ? 4 : 2;    // 8-row slabs in this tile
          double c[4][2][2];
          long long addr[4][2];
          const bool gen = K == 0 || R0 + 32 > W - NBF || C0 + 16 > W - NBF;
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            int pr = ks + NBF + R0 + 8 * mi + g; pr -= pr >= WS ? WS : 0; pr -= pr >= WS ? WS : 0;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
              int pc = ks + NBF + C0 + 8 * ni + 2 * t4; pc -= pc >= WS ? WS : 0; pc -= pc >= WS ? WS : 0;
              addr[mi][ni] = (long long)pr * WS + pc;
              c[mi][ni][0] = c[mi][ni][1] = 0.0;
              if (mi < mrows) {
                const double2 v = *reinterpret_cast<const double2*>(win + addr[mi][ni]);
                c[mi][ni][0] = v.x;
                c[mi][ni][1] = v.y;
              }
            }
          }
          if (gen) {   // overwrite the entries that are still original with generated values
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              const int i = k0 + NBF + R0 + 8 * mi + g;
              if (mi < mrows) {
                const RowInfo ri = row_info(s, JD, i);
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) {
                  const int j = k0 + NBF + C0 + 8 * ni + 2 * t4;
                  if (i >= fresh || j >= fresh) c[mi][ni][0] = entry(s, ri, j, off);
                  if (i >= fresh || j + 1 >= fresh) c[mi][ni][1] = entry(s, ri, j + 1, off);
                }
              }
            }
          }
          const double* ap = P + (NBF + R0 + g) * LDP + t4;
          const double* bp = U + t4 * LDU + C0 + g;
#pragma unroll
          for (int kk = 0; kk < NBF; kk += 4) {
            const double b0 = bp[kk * LDU], b1 = bp[kk * LDU + 8];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              if (mi < mrows) {
                const double am = -ap[8 * mi * LDP + kk];
                dmma_884(c[mi][0][0], c[mi][0][1], am, b0);
                dmma_884(c[mi][1][0], c[mi][1][1], am, b1);
              }
            }
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
              if (mi < mrows)
                *reinterpret_cast<double2*>(win + addr[mi][ni]) = make_double2(c[mi][ni][0], c[mi][ni][1]);
          if (warp == LAW && wt == 0 && K + 1 < nblk) {
            // tile 0 holds the next panel's A_aa (rows/cols [k0+32, k0+48)),
            // now final: factor it here, overlapped with the other warps' update
            __syncwarp();
            for (int e = lane; e < 256; e += 32) {
              const int r = e >> 4, cc = e & 15;
              int pr = ks + NBF + r; pr -= pr >= WS ? WS : 0;
              int pc = ks + NBF + cc; pc -= pc >= WS ? WS : 0;
              Pn[r * LDP + cc] = win[(long long)pr * WS + pc];
            }
            warp_lu16(Pn, 0, lane, rdn, &bad);
          }
          wt = -1;
        }
      }
      // ---- 3c. the rest of the finished 32-block -> factor store
      //          (streaming stores: the 8 GB store must not evict the L2-resident windows)
      for (int c = warp; c < NBF; c += NW) {
        double* Lb = fac + (long long)K * 2 * NBF * LD;
        double* Ub = Lb + NBF * LD;
        const int lfirst = NBF - 1 - c;  // first L entry below the block
        for (int sidx = lfirst + lane; sidx < LD; sidx += 32)
          __stcs(Lb + c * LD + sidx, sidx == W ? 0.0 : P[(c + 1 + sidx) * LDP + c]);
        const int ufirst = NBF - c;      // first U entry right of the block
        for (int sidx = ufirst + lane; sidx < LD; sidx += 32)
          __stcs(Ub + c * LD + sidx, U[c * LDU + c + sidx - NBF]);
      }
      __syncthreads();
      PHASE_MARK(6);
      if (bad) break;
      ks += NBF;
      ks -= ks >= WS ? WS : 0;
    }
    if (tid == 0) status[sid] = bad;
    __syncthreads();
  }
}

#ifdef OCP_PHASE_TIMING
void read_phase(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_phase, 8 * sizeof(unsigned long long)); }
#endif
int factor_smem_bytes(int W) {
  return (int)sizeof(double) * ((W + NBF) * LDP + NBF * (W + 4));
}

}  // namespace ocp
