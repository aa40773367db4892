// Block-tridiagonal ("block-Thomas") factorisation of the local Jacobians and
// the matching stored-factor solve (sm_100a, FP64 tensor cores).
//
// In band order (k = a*n + t, n = 2 nc, t = 2b + f) the local pair Jacobian
// (schwarz.py:166-171, system.py:135-144) is block tridiagonal along the long
// side: diagonal blocks D_a (one grid line: diag, y<->p coupling, +-1
// neighbours in the line) and off-diagonal blocks off*I (the a +- 1 lines).
// Its LU without pivoting, grouped by lines, is
//     S_0 = D_0,   S_a = D_a - off^2 S_{a-1}^{-1},
// and a solve is
//     forward   w_a = S_a^{-1} (r_a - off w_{a-1})
//     backward  x_a = w_a - off S_a^{-1} x_{a+1}.
// P J is symmetric (P swaps the y / p unknowns of every point: J = [[K, B12],
// [B21, K]] with K = A + diag(phi') symmetric and B12, B21 diagonal), so
// J^T = P J P, every Schur complement keeps S_a^T = P S_a P, and
// W_a = S_a^{-1} P = M_a^{-1} with M_a = P S_a symmetric.  The factor store
// keeps, per line, -W_a as the upper triangle of 16x16 tiles (NPS =
// round16(n), identity on the padding; layout in ocp_kernels.cuh): 55 of 100
// tiles at NPS = 160.
//
// k_block_factor: one persistent CTA per SM (12 warps) takes subdomains from
// a cost-sorted queue; M stays resident in shared memory (NPB <= 160; larger
// blocks keep their last rows in a per-CTA global scratch, L2-resident).  Per
// line the E phase writes the previous line's -W to the store from the rows
// it loads and rebuilds M_a = P D_a - off^2 P W_{a-1} P in place; then a
// symmetric block sweep (Goodnight's sweep operator, 32-wide pivot panels,
// result -M^{-1}) inverts it:
//     P1  A^{-1} of the 32x32 pivot block (Gauss-Jordan, 2x2 pivots)
//     P2  M[p, j] = A^{-1} M[p, j]                      (DMMA, row block)
//     P3a M[i, j] -= M[i, p] M[p, j], upper tiles only (DMMA), mirrored
//     P3b M[i, p] = M[p, i]^T, M[p, p] = -A^{-1}        (register transpose)
// P1 of panel p+1 runs on warps 0..3 (lookahead) while the other warps finish
// P3a and P3b of panel p; P1 of panel 0 runs under the E phase of rows 32+.
// Every flop except the pivot inverses is a DMMA (mma.sync.m8n8k4.f64) on
// shared-memory operands.
//
// k_block_solve<MODE>: one CTA per subdomain, a producer warp streaming
// tile-column pairs of each line through a ring of TMA bulk copies (+ an L2
// prefetch of the next line) and two consumer threads per row accumulating
// the full symmetric row (stored tiles + the transposed column above the
// diagonal tile).  MODE 0: inner-Newton solve (pool to pool); MODE 1: the
// backward sweep stops at the first owned line (schwarz.py:344); MODE 2: the
// fused JVP; MODE 3: the fused RAS apply.
#include "ocp_kernels.cuh"
#include "ocp_tma.cuh"

namespace ocp {

#ifndef OCP_BF_THREADS
#define OCP_BF_THREADS 384
#endif
constexpr int BF_THREADS = OCP_BF_THREADS;   // factor CTA: 12 warps (measured: 8 warps 5 % slower, 16 warps 1 % slower)

#ifdef OCP_PHASE_TIMING
__device__ unsigned long long g_bphase[8];
#define BPH_START() long long t_last = clock64()
#define BPH_MARK(k)                                                                     \
  do {                                                                                  \
    if (threadIdx.x == 0) {                                                             \
      const long long now = clock64();                                                  \
      atomicAdd(&g_bphase[k], (unsigned long long)(now - t_last));                      \
      t_last = now;                                                                     \
    }                                                                                   \
  } while (0)
__device__ long long g_subt[1024][3];   // per subdomain: start clock, end clock, SM id
void read_bphase(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_bphase, 8 * sizeof(unsigned long long));
}
void read_subt(long long* out, int n) {
  cudaMemcpyFromSymbol(out, g_subt, (size_t)3 * (n < 1024 ? n : 1024) * sizeof(long long));
}
#else
#define BPH_START() (void)0
#define BPH_MARK(k) (void)0
#endif
#ifdef OCP_P1_SERIAL
constexpr bool P1_SERIAL = true;
#else
constexpr bool P1_SERIAL = false;
#endif
constexpr int BF_JL_POINTS = 112;   // points per line whose diagonals fit the shared JL slot
constexpr int BS_STAGES = 4;     // TMA ring depth of the solve
#ifndef OCP_BS_PF_EARLY
#define OCP_BS_PF_EARLY 0
#endif
// the solve prefetches line a+1 into L2 at stage nst-1-BS_PF_EARLY of line a (< 0: off)
constexpr int BS_PF_EARLY = OCP_BS_PF_EARLY;
constexpr int BS_MAX_THREADS = 480;   // 2 threads per row + a producer warp, NPS <= 224

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// entry (i, j) of the diagonal block D_a; JL = the line's Jacobian diagonals
// (4 per point, copied to shared memory), padding: identity
__device__ __forceinline__ double d_entry(const SubInfo& s, const double* JL, int i, int j,
                                          double off) {
  const int n = 2 * s.nc;
  if (i >= n || j >= n) return i == j ? 1.0 : 0.0;
  const int bi = i >> 1, fi = i & 1, bj = j >> 1, fj = j & 1;
  if (bi == bj) {
    if (fi == fj) return JL[4 * bi];                   // 4/h^2 + phi'(y)
    return fi == 0 ? JL[4 * bi + 1] : JL[4 * bi + 2];  // b12 (y row), b21 (p row)
  }
  if (fi == fj && (bi - bj == 1 || bj - bi == 1)) return off;
  return 0.0;
}

// reciprocal without the IEEE slow path (no call => nothing spills around
// it): MUFU seed + two Newton steps, ~1 ulp; pivots are O(1/h^2) normals
__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// P1: in-place Gauss-Jordan inverse of the 32x32 block at S[p0.., p0..] by
// PW warps (named barrier 2).  Thread (w, lane) keeps rows R w .. R w + R - 1
// (R = 32 / PW) of column `lane` in registers; every pivot step reads the pivot column / row
// from one of two ping-pong 32x33 buffers and writes its updated entries to
// the other, so a step costs one barrier.  No shuffles: inside a
// warp-uniform branch the compiler wraps each shfl in a convergence check.
constexpr int WLD = 33;
#ifndef OCP_LAW
#define OCP_LAW 4
#endif
constexpr int LAW = OCP_LAW;   // lookahead warps (0 .. LAW-1): the next pivot inverse while the others update
// kmax: pivots kmax .. 31 of this block lie in the identity padding past the
// line's n unknowns (decoupled: zero rows / columns outside the diagonal), so
// their Gauss-Jordan steps are exact no-ops and are skipped - the last panel
// of a 72-unknown line (NPB 96) takes 4 steps instead of 16.
// bw: rows / columns of the block that exist in storage (32, or 16 for the
// half-width last panel of a line padded to 16: the rest is identity, held
// in registers only).
template <int PW>
__device__ __noinline__ void pivot_inverse32(double* B, int lds, double* W0, double* W1, int wsub,
                                             int lane, int* bad, int kmax, int bw = 32) {
  // Gauss-Jordan with 2x2 pivot blocks: 16 dependent steps instead of 32.
  // Step s eliminates rows/columns K = {k, k+1}, k = 2s:
  //   S[K,K] <- P^{-1};  S[K,j] <- P^{-1} S[K,j];  S[i,K] <- -S[i,K] P^{-1};
  //   S[i,j] <- S[i,j] - S[i,K] (P^{-1} S[K,j])
  constexpr int R = 32 / PW;
  double c[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int row = R * wsub + i;
    c[i] = (row < bw && lane < bw) ? B[row * lds + lane] : (row == lane ? 1.0 : 0.0);
    W0[row * WLD + lane] = c[i];
  }
  asm volatile("bar.sync 2, %0;" ::"n"(32 * PW) : "memory");
  bool ok = true;
#ifdef OCP_PHASE_TIMING
  const long long t_piv = clock64();
#endif
#pragma unroll 1
  for (int k = 0; k < kmax; k += 2) {
    const double* Wr = (k & 2) ? W1 : W0;
    double* Ww = (k & 2) ? W0 : W1;
    const double p00 = Wr[k * WLD + k], p01 = Wr[k * WLD + k + 1];
    const double p10 = Wr[(k + 1) * WLD + k], p11 = Wr[(k + 1) * WLD + k + 1];
    const double b0 = Wr[k * WLD + lane], b1 = Wr[(k + 1) * WLD + lane];   // S[K, lane]
    double f0[R], f1[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      f0[i] = Wr[(R * wsub + i) * WLD + k];
      f1[i] = Wr[(R * wsub + i) * WLD + k + 1];
    }
    const double det = fma(p00, p11, -p01 * p10);
    ok = ok && det != 0.0 && isfinite(det);
    const double rd = rcp64(det);
    const double q00 = p11 * rd, q01 = -p01 * rd, q10 = -p10 * rd, q11 = p00 * rd;   // P^{-1}
    const int t = lane - k;                        // 0 / 1: this column is in K
    const bool inK = t == 0 || t == 1;
    // new S[K, lane]: P^{-1} column t for lanes in K, P^{-1} S[K, lane] otherwise
    const double m0 = inK ? (t == 0 ? q00 : q01) : fma(q00, b0, q01 * b1);
    const double m1 = inK ? (t == 0 ? q10 : q11) : fma(q10, b0, q11 * b1);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = R * wsub + i;
      double v;
      if (row == k) v = m0;
      else if (row == k + 1) v = m1;
      else v = fma(-f0[i], m0, fma(-f1[i], m1, inK ? 0.0 : c[i]));
      c[i] = v;
      // publish what the next step reads: its pivot rows and columns
      if (row == k + 2 || row == k + 3 || lane == k + 2 || lane == k + 3) Ww[row * WLD + lane] = v;
    }
    asm volatile("bar.sync 2, %0;" ::"n"(32 * PW) : "memory");
  }
#ifdef OCP_PHASE_TIMING
  if (P1_SERIAL && wsub == 0 && lane == 0) atomicAdd(&g_bphase[0], (unsigned long long)(clock64() - t_piv));
#endif
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (R * wsub + i < bw && lane < bw) B[(R * wsub + i) * lds + lane] = c[i];
  if (!ok) *bad = 1;
}
// real pivots of the 32x32 pivot block at p0 (n even: 2x2 pivot pairs stay whole)
__device__ __forceinline__ int pivot_kmax(int n, int p0) {
  const int k = n - p0;
  return k < 32 ? (k > 0 ? k : 0) : 32;
}

// one DMMA tile of 8 MI rows x 16 columns over KK pivot columns:
//   C (+)= sgn * A[8 MI x KK] * B[KK x 16]
//   A element (m, k) at A + m*lda + k ; B element (k, n) at B + k*ldb + n
// (MI, KK) = (4, 32) everywhere except the half-width last panel of a line
// padded to 16 (narrow lines: 72 unknowns at NPB = 80), where the row tile
// has 16 rows (MI = 2) and / or the pivot panel 16 columns (KK = 16).
#ifdef OCP_DFMA_ONLY
// A/B build (tools/build_variant.py dfma -DOCP_DFMA_ONLY): the same tiles,
// register layout and shared-memory operands, multiplied with DFMA instead of
// DMMA - each lane accumulates its outputs from one A element per row and
// double2 B loads per k.  Justifies the DMMA choice with a measurement
// (profiles/r2_dmma_vs_dfma.md).
template <int MI, int KK>
__device__ __forceinline__ void tile_mk(const double* A, int lda, const double* B, int ldb,
                                        double c[4][2][2], int lane, double sgn) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll 4
  for (int k = 0; k < KK; ++k) {
    const double2 b0 = *reinterpret_cast<const double2*>(B + k * ldb + 2 * t4);
    const double2 b1 = *reinterpret_cast<const double2*>(B + k * ldb + 8 + 2 * t4);
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const double am = sgn * A[(8 * mi + g) * lda + k];
      c[mi][0][0] = fma(am, b0.x, c[mi][0][0]);
      c[mi][0][1] = fma(am, b0.y, c[mi][0][1]);
      c[mi][1][0] = fma(am, b1.x, c[mi][1][0]);
      c[mi][1][1] = fma(am, b1.y, c[mi][1][1]);
    }
  }
}
#else
template <int MI, int KK>
__device__ __forceinline__ void tile_mk(const double* A, int lda, const double* B, int ldb,
                                        double c[4][2][2], int lane, double sgn) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int kk = 0; kk < KK; kk += 4) {
    const double b0 = B[(kk + t4) * ldb + g];
    const double b1 = B[(kk + t4) * ldb + 8 + g];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const double am = sgn * A[(8 * mi + g) * lda + kk + t4];
      dmma(c[mi][0][0], c[mi][0][1], am, b0);
      dmma(c[mi][1][0], c[mi][1][1], am, b1);
    }
  }
}
#endif
__device__ __forceinline__ void tile_32x16(const double* A, int lda, const double* B, int ldb,
                                           double c[4][2][2], int lane, double sgn) {
  tile_mk<4, 32>(A, lda, B, ldb, c, lane, sgn);
}

// C tile (8 MI x 16) at base (row stride lds) -> registers / back
template <int MI = 4>
__device__ __forceinline__ void load_c(const double* base, int lds, double c[4][2][2], int lane) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(base + (8 * mi + g) * lds + 8 * ni + 2 * t4);
      c[mi][ni][0] = v.x;
      c[mi][ni][1] = v.y;
    }
}
template <int MI = 4>
__device__ __forceinline__ void store_c(double* base, int lds, const double c[4][2][2], int lane) {
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
      *reinterpret_cast<double2*>(base + (8 * mi + g) * lds + 8 * ni + 2 * t4) =
          make_double2(c[mi][ni][0], c[mi][ni][1]);
}

// P3b strip: out[16 x 32] = -A[16 x 32] P  (A and out at the same place)
__device__ __forceinline__ void strip_16x32(double* A, const double* P, int lds, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  double c[2][4][2] = {};
#ifdef OCP_DFMA_ONLY
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    double2 b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = *reinterpret_cast<const double2*>(P + k * lds + 8 * ni + 2 * t4);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double am = -A[(8 * mi + g) * lds + k];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        c[mi][ni][0] = fma(am, b[ni].x, c[mi][ni][0]);
        c[mi][ni][1] = fma(am, b[ni].y, c[mi][ni][1]);
      }
    }
  }
  __syncwarp();   // every lane has read its A rows before they are overwritten
#else
#pragma unroll
  for (int kk = 0; kk < 32; kk += 4) {
    double b[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = P[(kk + t4) * lds + 8 * ni + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double am = -A[(8 * mi + g) * lds + kk + t4];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(c[mi][ni][0], c[mi][ni][1], am, b[ni]);
    }
  }
#endif
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(A + (8 * mi + g) * lds + 8 * ni + 2 * t4) =
          make_double2(c[mi][ni][0], c[mi][ni][1]);
}

// Row storage of the Schur block.  Normally every row is in shared memory;
// blocks larger than the shared capacity keep rows [0, r0) there and the
// rest in a per-CTA global scratch (L2-resident).  Row tiles are 32-row
// aligned and r0 is a multiple of 32, so a tile never straddles the split.
template <bool SPLIT>
struct Rows {
  double* s;
  double* g;
  int r0, lds;
  __device__ __forceinline__ double* row(int i) const {
    if (!SPLIT) return s + i * lds;
    return i < r0 ? s + i * lds : g + (i - r0) * lds;
  }
};

// HALF: NPB is an odd multiple of 16 (narrow-line instance only): the last
// panel is 16 wide.  HALF = false compiles the 32-wide-panel code alone.
template <bool SPLIT, bool HALF = false>
__device__ __forceinline__ void factor_one(const SubInfo& s, const double* JD, double off,
                                           const Rows<SPLIT> R, double* fac, int* bad, double* W0,
                                           double* W1, double* JL) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BF_THREADS / 32;
  const int NPB = s.pad_, NPS = s.NPS, n = 2 * s.nc, nr = s.nr, lds = R.lds;
  // NPB is a multiple of 32, or (narrow lines, ocp_block_narrow.cu) of 16: the
  // last panel is then 16 wide - one column tile, 16-row tiles, 16 pivot columns
  const int npan = (NPB + 31) / 32, nct = NPB / 16;
  auto pwid = [&](int p) { return HALF && p == npan - 1 ? 16 : 32; };
  constexpr bool ALLP1 = LAW == BF_THREADS / 32;   // every warp is a pivot warp (needs the serial schedule)
  static_assert(!ALLP1 || P1_SERIAL, "LAW == warps per CTA needs OCP_P1_SERIAL");
  const double off2 = off * off;
  const long long lsz = block_line_doubles(NPS);   // stored doubles per line
  BPH_START();
  // the Jacobian diagonals of the next line are loaded one line ahead
  // (registers) and staged in shared memory (JL) at the start of its E phase
  const int nq = 4 * s.nc;
  // lines of up to 2 BF_THREADS diagonal entries are prefetched in registers;
  // wider ones (short side > 192) are copied at the start of their E phase
  const bool jreg = nq <= 2 * BF_THREADS;
  double jn0 = jreg && tid < nq ? JD[tid] : 0.0;
  double jn1 = jreg && tid + BF_THREADS < nq ? JD[tid + BF_THREADS] : 0.0;
  // -W of a line goes to the factor store by TMA bulk stores (issued by warp
  // 0): the copies run on the TMA engine, so no global store traffic sits in
  // the load/store queues of the compute phases.  The shared block is
  // symmetric, so column j of the upper tile triangle (rows 0 .. 16c+15,
  // c = j / 16) is the head of shared row j: one copy per column.
  auto store_block = [&](int line) {
    double* dst = fac + (long long)line * lsz;
    const int rs = SPLIT ? (R.r0 < NPS ? R.r0 : NPS) : NPS;   // rows held in shared memory
    const int cpb = NPS / 16;
    auto col_off = [cpb](int j) {
      const int c = j >> 4;
      return block_col_off(c, cpb) + (long long)(j - 16 * c) * (16 * c + 18);
    };
    if (warp == 0) {
      for (int j = lane; j < rs; j += 32)
        bulk_s2g(dst + col_off(j), R.row(j), (uint32_t)((16 * (j >> 4) + 16) * sizeof(double)));
      bulk_commit();
    }
    if (SPLIT)
      for (int j = rs + warp; j < NPS; j += NW) {
        const int m16 = 16 * (j >> 4) + 16;
        for (int r = lane; r < m16; r += 32) __stcs(dst + col_off(j) + r, R.row(j)[r]);
      }
    if (warp == 0) bulk_wait_read();
    __syncthreads();
  };
  for (int a = 0; a < nr; ++a) {
    if (jreg) {
      if (tid < nq) JL[tid] = jn0;
      if (tid + BF_THREADS < nq) JL[tid + BF_THREADS] = jn1;
      if (a + 1 < nr) {
        const double* nx = JD + (long long)(a + 1) * nq;
        jn0 = tid < nq ? nx[tid] : 0.0;
        jn1 = tid + BF_THREADS < nq ? nx[tid + BF_THREADS] : 0.0;
      }
    } else {
      for (int t = tid; t < nq; t += BF_THREADS) JL[t] = JD[(long long)a * nq + t];
    }
    __syncthreads();   // JL complete: both warp groups read all of it in E2
    BPH_MARK(6);
    // ---- E1. M = -off^2 P W_{a-1} P = off^2 (-W_{a-1})[i^1][j^1] on the real
    //      block (the shared block holds -W_{a-1}), identity on the padding
    //      (warp per row pair, double2 columns; a pair's loads are issued
    //      before its stores: new row i is old row i^1 with swapped columns).
    //      The loaded rows also go to the factor store: by symmetry stored
    //      column i of line a-1 is the head of row i (coalesced streaming
    //      stores; the shared block is read only once).
    double* dstl = fac + (long long)(a - 1) * lsz;
    // warps 0..LAW-1 build rows 0..31 and invert the first pivot block while
    // the other warps build the remaining rows (3 % faster than E for all
    // rows, then the first pivot inverse on 8 warps)
    const bool grpA = warp < LAW;
    const int e_lo = grpA ? 0 : 32, e_hi = grpA && !ALLP1 && NPB > 32 ? 32 : NPB;
    const int e_w = grpA ? warp : warp - LAW, e_nw = grpA ? LAW : NW - LAW;
    // (rows wider than 256 columns are processed in chunks of 256; PACK - lines
    // of at most 128 columns, the narrow instance - puts two row pairs in the
    // four column slots of a lane, so twice the loads are in flight per warp)
    constexpr bool PACK = HALF;
    for (int i0 = e_lo + 2 * e_w; i0 < e_hi; i0 += 2 * e_nw * (PACK ? 2 : 1))
      for (int cb = 0; cb < NPB; cb += 256) {
        double2 v[2][4];
        auto rowof = [&](int u) { return i0 + (PACK ? 2 * e_nw * (u >> 1) : 0); };   // first row of slot u's pair
        auto colof = [&](int u) { return cb + 2 * lane + 64 * (PACK ? (u & 1) : u); };
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = colof(u);
            v[r][u] = (a > 0 && j < NPB && rowof(u) < e_hi)
                          ? *reinterpret_cast<const double2*>(R.row(rowof(u) + r) + j)
                          : make_double2(0.0, 0.0);
          }
        if (a > 0)
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (!PACK && u > 0) break;   // (one row pair: its column slots are handled below)
              if (PACK && (u & 1)) continue;
              const int i = rowof(u) + r, m16 = 16 * (i >> 4) + 16;
              if (i >= NPS || rowof(u) >= e_hi) continue;
              double2* col = reinterpret_cast<double2*>(dstl + block_col_off(i >> 4, NPS / 16) +
                                                        (long long)(i & 15) * (m16 + 2));
#pragma unroll
              for (int u2 = 0; u2 < (PACK ? 2 : 4); ++u2) {
                const int j = colof(u + u2);
                if (j < m16) __stcs(col + (j >> 1), v[r][u + u2]);
              }
            }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = rowof(u) + r, j = colof(u);
            if (j >= NPB || rowof(u) >= e_hi) continue;
            double2 w;
            if (i < n && j < n) {
              w.x = off2 * v[1 - r][u].y;
              w.y = off2 * v[1 - r][u].x;
            } else {
              w.x = i == j ? 1.0 : 0.0;
              w.y = i == j + 1 ? 1.0 : 0.0;
            }
            *reinterpret_cast<double2*>(R.row(i) + j) = w;
          }
      }
    if (grpA) asm volatile("bar.sync 2, %0;" ::"n"(32 * LAW) : "memory");
    else asm volatile("bar.sync 3, %0;" ::"n"(BF_THREADS - 32 * LAW) : "memory");
    BPH_MARK(7);
    {
      const int n_hi = e_hi < n ? e_hi : n;
      for (int e = 7 * e_lo + 32 * e_w + lane; e < 7 * n_hi; e += 32 * e_nw) {
        const int i = e / 7, j = i + (e - 7 * i) - 3;
        if (j >= 0 && j < n) R.row(i)[j] += d_entry(s, JL, i ^ 1, j, off);
      }
    }
    if (grpA) {
      asm volatile("bar.sync 2, %0;" ::"n"(32 * LAW) : "memory");
      pivot_inverse32<LAW>(R.row(0), lds, W0, W1, warp, lane, bad, pivot_kmax(n, 0), pwid(0));
    }
    __syncthreads();
    BPH_MARK(1);
    // ---- Symmetric block sweep of M in place (Goodnight's sweep operator with
    //      32-wide pivot panels: every intermediate stays symmetric and the
    //      result is -M^{-1} = -W_a).  For pivot block A = M[p][p]:
    //        P2   M[p][j] = A^{-1} M[p][j]            (row block, DMMA)
    //        P3a  M[i][j] -= M[i][p] M[p][j]           upper 32x16 tiles only (DMMA);
    //             strictly-upper tiles are mirrored into the lower triangle
    //        P3b  M[i][p] = M[p][i]^T (transposed copy), M[p][p] = -A^{-1}
    //      P1 (the 32x32 pivot inverse) of panel 0 ran on warps 0..LAW-1 under
    //      the E phase; P1 of panel p+1 runs on the same warps (lookahead) as
    //      soon as warps 0, 1 have updated the next pivot block, concurrently
    //      with the other trailing tiles.
    BPH_MARK(5);
    for (int p = 0; p < npan; ++p) {
      const int p0 = 32 * p;
      double* Prow = R.row(p0);                 // the pivot row block
      const double* Pinv = Prow + p0;
      // ---- P2: row block S[p, j] = Pinv S[p, j] (column tiles of 16 outside p)
      const int pw = pwid(p), pc = pw / 16;   // this panel's width and column tiles
      for (int tI = warp; tI < nct - pc; tI += NW) {
        const int j0 = 16 * (tI + (tI >= 2 * p ? pc : 0));
        if (j0 >= NPS) continue;   // identity padding: M[p, j] = 0 stays 0
        double c[4][2][2] = {};
        if (pw == 32) {
          tile_mk<4, 32>(Pinv, lds, Prow + j0, lds, c, lane, 1.0);
          store_c<4>(Prow + j0, lds, c, lane);
        } else {
          tile_mk<2, 16>(Pinv, lds, Prow + j0, lds, c, lane, 1.0);
          store_c<2>(Prow + j0, lds, c, lane);
        }
      }
      __syncthreads();
      BPH_MARK(2);
      // ---- P3a: M[i, j] -= M[i, p] M[p, j] on the upper tiles (i, j outside p)
      {
        // compact numbering of the upper 32x16 tiles (ct >= 2 rt) outside
        // panel p, row tile by row tile
        auto upper = [&](int tI, int& rt, int& ct) {
          for (rt = 0; rt < npan; ++rt) {
            if (rt == p) continue;
            const int cnt = nct - 2 * rt - (p > rt ? pc : 0);
            if (tI < cnt) {
              ct = 2 * rt + tI;
              if (p > rt && ct >= 2 * p) ct += pc;
              return true;
            }
            tI -= cnt;
          }
          return false;
        };
        const int total = p * (nct - pc) - p * (p - 1) +
                          (npan - 1 - p) * nct - (npan - 1 - p) * (npan + p);
        const bool la = p + 1 < npan;
        const int g = lane >> 2, t4 = lane & 3;
        auto tile = [&](int tI) {
          int rt, ct;
          upper(tI, rt, ct);
          if (16 * ct >= NPS) return;   // padding columns: M[p, j] = 0, no update
          double* Ci = R.row(32 * rt);
          double c[4][2][2];
          const int rw = pwid(rt);   // rows of this row tile
          if (rw == 32 && pw == 32) {
            load_c<4>(Ci + 16 * ct, lds, c, lane);
            tile_mk<4, 32>(Ci + p0, lds, Prow + 16 * ct, lds, c, lane, -1.0);
            store_c<4>(Ci + 16 * ct, lds, c, lane);
          } else if (rw == 32) {
            load_c<4>(Ci + 16 * ct, lds, c, lane);
            tile_mk<4, 16>(Ci + p0, lds, Prow + 16 * ct, lds, c, lane, -1.0);
            store_c<4>(Ci + 16 * ct, lds, c, lane);
          } else {   // (the half-width panel is the last one: the pivot panel is a full one)
            load_c<2>(Ci + 16 * ct, lds, c, lane);
            tile_mk<2, 32>(Ci + p0, lds, Prow + 16 * ct, lds, c, lane, -1.0);
            store_c<2>(Ci + 16 * ct, lds, c, lane);
          }
          if (ct >= 2 * rt + 2) {   // strictly upper: mirror into the lower triangle
            // (a 16-row tile is never strictly upper: the half-width panel is the last one)
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                  R.row(16 * ct + 8 * ni + 2 * t4 + k)[32 * rt + 8 * mi + g] = c[mi][ni][k];
          }
        };
        // ---- P3b: column block M[i, p] = M[p, i]^T (the new row block is
        //      A^{-1} M[p][i]; by symmetry the new column block is its
        //      transpose), pivot block -A^{-1}.  Register transpose: task
        //      (row tile rt outside p, column half): lane l gathers
        //      M[p0 + 16h + c][32rt + l], c < 16 (coalesced row reads) and
        //      writes them as 16 contiguous entries of row 32rt + l.  It must
        //      follow every P3a tile (they read the old column block).
        auto p3b = [&](int rank, int nw) {   // rank: this warp's index among the nw doing it
          for (int task = rank; task < pc * (npan - 1); task += nw) {
            int rt = task >> (pc - 1);   // pc is 1 or 2
            const int c0 = 16 * (task - (rt << (pc - 1))), i = 32 * (rt + (rt >= p ? 1 : 0)) + lane;
            rt += rt >= p ? 1 : 0;
            if (i >= NPB) continue;   // (half-width last row tile)
            double v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = Prow[(c0 + c) * lds + i];
            double* dst = R.row(i) + p0 + c0;
#pragma unroll
            for (int c = 0; c < 16; c += 2)
              *reinterpret_cast<double2*>(dst + c) = make_double2(v[c], v[c + 1]);
          }
          for (int e = 32 * rank + lane; e < 32 * pw; e += 32 * nw) {   // pivot block -> -A^{-1}
            if ((e & 31) >= pw) continue;
            double* q = Prow + (e >> 5) * lds + p0 + (e & 31);
            *q = -*q;
          }
        };
        if (!la) {
          for (int tI = warp; tI < total; tI += NW) tile(tI);
          __syncthreads();
          BPH_MARK(3);
          p3b(warp, NW);
        } else {
          // the two tiles of the next pivot block (row tile p+1, column tiles
          // 2p+2, 2p+3) come first in row p+1 of the compact numbering; the
          // lookahead warps then invert that block while the others finish
          // the trailing tiles and do P3b (barrier 5: all P3a tiles done)
          const int la0 = p * (nct - 2) - p * (p - 1);
          // (lookahead warps 0 and 4, one SM sub-partition, measured 13 % slower)
          const bool law = warp < LAW;
          const int lrank = warp, trank = warp - LAW;
#ifdef OCP_P1_SERIAL
          // no overlap (A/B on wide lines; the narrow-line instance, where
          // every warp is a pivot warp): every warp does trailing tiles, then
          // warps 0..LAW-1 invert the next pivot block with the FP64 pipe to
          // themselves
          for (int tI = warp; tI < total; tI += NW) tile(tI);
          __syncthreads();
          BPH_MARK(3);
          if (law)
            pivot_inverse32<LAW>(R.row(p0 + 32) + p0 + 32, lds, W0, W1, lrank, lane, bad,
                                 pivot_kmax(n, p0 + 32), pwid(p + 1));
          if (ALLP1) {
            __syncthreads();
            p3b(warp, NW);
          } else if (!law) {
            p3b(trank, NW - LAW);
          }
          __syncthreads();
          BPH_MARK(5);
          if (false) {
#else
          if (law) {
#endif
#ifdef OCP_PHASE_TIMING
            const long long tla = clock64();
#endif
            if (lrank < pwid(p + 1) / 16) tile(la0 + lrank);   // the lookahead tiles (next pivot block)
            asm volatile("bar.arrive 5, %0;" ::"n"(BF_THREADS) : "memory");
            asm volatile("bar.sync 2, %0;" ::"n"(32 * LAW) : "memory");
            pivot_inverse32<LAW>(R.row(p0 + 32) + p0 + 32, lds, W0, W1, lrank, lane, bad,
                                 pivot_kmax(n, p0 + 32), pwid(p + 1));
#ifdef OCP_PHASE_TIMING
            if (tid == 0) atomicAdd(&g_bphase[0], (unsigned long long)(clock64() - tla));
#endif
          } else if (!P1_SERIAL) {
            for (int tI = trank; tI < total; tI += NW - LAW)
              if (tI < la0 || tI >= la0 + pwid(p + 1) / 16) tile(tI);
            asm volatile("bar.sync 5, %0;" ::"n"(BF_THREADS) : "memory");
            p3b(trank, NW - LAW);
          }
          __syncthreads();
          BPH_MARK(3);
        }
      }
      __syncthreads();
      BPH_MARK(4);
    }
    if (*bad) return;
  }
  // the last S^{-1}; the factor store must be complete when the kernel ends
  store_block(nr - 1);
  if (warp == 0) bulk_wait_all();
}

#ifndef OCP_BF_MINB
#define OCP_BF_MINB 1
#endif
__global__ void __launch_bounds__(BF_THREADS, OCP_BF_MINB)
k_block_factor(const SubInfo* subs, const int* list, int cnt, Phys P, const double* JDpool,
               double* fac_pool, double* gscratch, long long gs_stride, int* status) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int bad, next;
  // dynamic distribution: CTAs take the next subdomain of the (cost-sorted)
  // list from a counter stored at list[cnt] (zeroed by the host)
  int* counter = const_cast<int*>(list) + cnt;
  for (;;) {
    if (threadIdx.x == 0) next = atomicAdd(counter, 1);
    __syncthreads();
    const int li = next;
    if (li >= cnt) break;
    const int sid = list[li];
    const SubInfo s = subs[sid];
    const double* JD = JDpool + 2 * s.loc;
    double* fac = fac_pool + s.fac;
    const int lds = s.pad_ + 4;
    if (threadIdx.x == 0) bad = 0;
#ifdef OCP_PHASE_TIMING
    long long t_sub = clock64();
#endif
    __syncthreads();
    // shared memory: [S rows: SMEM_S doubles][W0, W1: 32 x 33][JL]
    constexpr int SMEM_S = BF_SMEM_MAX_NPB * (BF_SMEM_MAX_NPB + 4);
    double* W0 = sm + SMEM_S;
    double* W1 = W0 + 32 * WLD;
    double* JL = W1 + 32 * WLD;
    // lines wider than the shared JL slot (short side > BF_JL_POINTS) keep
    // their diagonals after the scratch rows of this CTA
    if (s.nc > BF_JL_POINTS) JL = gscratch + (long long)blockIdx.x * gs_stride + (long long)s.pad_ * lds;
    if (s.pad_ <= BF_SMEM_MAX_NPB) {
#ifdef OCP_NARROW_INSTANCE
      if (s.pad_ & 16)
        factor_one<false, true>(s, JD, P.off, Rows<false>{sm, nullptr, s.pad_, lds}, fac, &bad, W0, W1, JL);
      else
#endif
      factor_one<false>(s, JD, P.off, Rows<false>{sm, nullptr, s.pad_, lds}, fac, &bad, W0, W1, JL);
    } else {
      const int r0 = (SMEM_S / lds) / 32 * 32;   // rows that fit in shared memory
      factor_one<true>(s, JD, P.off,
                       Rows<true>{sm, gscratch + (long long)blockIdx.x * gs_stride, r0, lds}, fac,
                       &bad, W0, W1, JL);
    }
    __syncthreads();
#ifdef OCP_PHASE_TIMING
    if (threadIdx.x == 0 && sid < 1024) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_subt[sid][0] = t_sub;
      g_subt[sid][1] = clock64();
      g_subt[sid][2] = smid;
    }
#endif
    if (threadIdx.x == 0) status[sid] = bad;
    __syncthreads();
  }
}

int block_factor_threads() { return BF_THREADS; }

#ifndef OCP_NARROW_INSTANCE
// ---------------------------------------------------------------------------
// k_block_factor_mc: the same factorisation, bitwise, for FEW WIDE subdomains
// (coarse decompositions, the monolithic direct solve): K CTAs per subdomain
// share its Schur block, which lives in global memory (L2).  Every phase of
// the line / panel schedule of factor_one is split into independent items
// (row pairs of the E phase, 32x16 DMMA tiles of P2 and P3a, transpose tasks
// of P3b, stored columns) dealt round-robin to all warps of the K CTAs, with
// a split arrival-counter barrier per subdomain between dependent phases:
//   E | P1(0) | P2(0) | P3a(0) | P3b(0) + P1(1) | P2(1) | ... | P3b(last) |
// (P1(p+1) touches only the pivot block p+1, P3b(p) only column block p).
// Each item is computed exactly as factor_one computes it, so the stored
// -W_a are identical to the single-CTA path's; only the schedule differs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mc_barrier(unsigned long long* ctr, unsigned long long& target,
                                           int K) {
  __syncthreads();
  target += K;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(BF_THREADS, 1)
k_block_factor_mc(const SubInfo* subs, const int* list, int K, Phys P, const double* JDpool,
                  double* fac_pool, double* mscratch, long long ms_stride, int* status,
                  unsigned long long* bars) {
  __shared__ double W0[32 * WLD], W1[32 * WLD];
  __shared__ int bad;
  const int li = blockIdx.x / K, rank = blockIdx.x - li * K;
  const int sid = list[li];
  const SubInfo s = subs[sid];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BF_THREADS / 32;
  const int gw = rank * NW + warp, GW = K * NW;   // this warp among all warps of the subdomain
  const int NPB = s.pad_, NPS = s.NPS, n = 2 * s.nc, nr = s.nr, lds = NPB + 4;
  const int npan = NPB / 32, nct = NPB / 16, cpb = NPS / 16;
  const double off = P.off, off2 = off * off;
  const long long lsz = block_line_doubles(NPS);
  const int nq = 4 * s.nc;
  const double* JD = JDpool + 2 * s.loc;
  double* fac = fac_pool + s.fac;
  double* M = mscratch + (long long)li * ms_stride;
  auto row = [&](int i) { return M + (long long)i * lds; };
  unsigned long long* ctr = bars + 16 * li;   // one 128-byte line per subdomain
  unsigned long long target = 0;
  if (tid == 0) bad = 0;
  __syncthreads();
  auto col_off = [cpb](int j) {
    const int c = j >> 4;
    return block_col_off(c, cpb) + (long long)(j - 16 * c) * (16 * c + 18);
  };
  const int g = lane >> 2, t4 = lane & 3;
  for (int a = 0; a < nr; ++a) {
    const double* JL = JD + (long long)a * nq;   // this line's diagonals (global)
    double* dstl = fac + (long long)(a - 1) * lsz;
    // ---- E: row pairs (store line a-1's -W, rebuild M = P D_a - off^2 P W P)
    for (int pi = gw; pi < NPB / 2; pi += GW) {
      const int i0 = 2 * pi;
      for (int cb = 0; cb < NPB; cb += 256) {
        double2 v[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = cb + 2 * lane + 64 * u;
            v[r][u] = (a > 0 && j < NPB) ? *reinterpret_cast<const double2*>(row(i0 + r) + j)
                                         : make_double2(0.0, 0.0);
          }
        if (a > 0)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int i = i0 + r, m16 = 16 * (i >> 4) + 16;
            if (i >= NPS) continue;
            double2* col = reinterpret_cast<double2*>(dstl + block_col_off(i >> 4, cpb) +
                                                      (long long)(i & 15) * (m16 + 2));
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = cb + 2 * lane + 64 * u;
              if (j < m16) __stcs(col + (j >> 1), v[r][u]);
            }
          }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int i = i0 + r;
          double* rw = row(i);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = cb + 2 * lane + 64 * u;
            if (j >= NPB) continue;
            double2 w;
            if (i < n && j < n) {
              w.x = off2 * v[1 - r][u].y;
              w.y = off2 * v[1 - r][u].x;
            } else {
              w.x = i == j ? 1.0 : 0.0;
              w.y = i == j + 1 ? 1.0 : 0.0;
            }
            *reinterpret_cast<double2*>(rw + j) = w;
          }
        }
      }
      __syncwarp();
      if (lane < 14) {   // the seven diagonals of P D_a on the pair's two rows
        const int i = i0 + lane / 7, j = i + lane % 7 - 3;
        if (i < n && j >= 0 && j < n) row(i)[j] += d_entry(s, JL, i ^ 1, j, off);
      }
    }
    mc_barrier(ctr, target, K);
    // ---- P1 of panel 0
    if (rank == 0 && warp < LAW)
      pivot_inverse32<LAW>(row(0), lds, W0, W1, warp, lane, &bad, pivot_kmax(n, 0));
    mc_barrier(ctr, target, K);
    for (int p = 0; p < npan; ++p) {
      const int p0 = 32 * p;
      double* Prow = row(p0);
      const double* Pinv = Prow + p0;
      // ---- P2: row block tiles
      for (int tI = gw; tI < nct - 2; tI += GW) {
        const int j0 = 16 * (tI + (tI >= 2 * p ? 2 : 0));
        if (j0 >= NPS) continue;
        double c[4][2][2] = {};
        tile_32x16(Pinv, lds, Prow + j0, lds, c, lane, 1.0);
        store_c(Prow + j0, lds, c, lane);
      }
      mc_barrier(ctr, target, K);
      // ---- P3a: upper tiles outside panel p (factor_one's compact numbering)
      {
        const int total = p * (nct - 2) - p * (p - 1) + (npan - 1 - p) * nct -
                          (npan - 1 - p) * (npan + p);
        for (int tI = gw; tI < total; tI += GW) {
          int rt, ct, t = tI;
          for (rt = 0; rt < npan; ++rt) {
            if (rt == p) continue;
            const int cnt = nct - 2 * rt - (p > rt ? 2 : 0);
            if (t < cnt) {
              ct = 2 * rt + t;
              if (p > rt && ct >= 2 * p) ct += 2;
              break;
            }
            t -= cnt;
          }
          if (16 * ct >= NPS) continue;
          double* Ci = row(32 * rt);
          double c[4][2][2];
          load_c(Ci + 16 * ct, lds, c, lane);
          tile_32x16(Ci + p0, lds, Prow + 16 * ct, lds, c, lane, -1.0);
          store_c(Ci + 16 * ct, lds, c, lane);
          if (ct >= 2 * rt + 2) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                  row(16 * ct + 8 * ni + 2 * t4 + k)[32 * rt + 8 * mi + g] = c[mi][ni][k];
          }
        }
      }
      mc_barrier(ctr, target, K);
      // ---- P3b of panel p (column block = row block transposed, pivot -A^{-1})
      //      and P1 of panel p + 1 (disjoint data)
      if (p + 1 < npan && rank == (p + 1) % K && warp < LAW)
        pivot_inverse32<LAW>(row(p0 + 32) + p0 + 32, lds, W0, W1, warp, lane, &bad,
                             pivot_kmax(n, p0 + 32));
      for (int task = gw; task < 2 * (npan - 1); task += GW) {
        int rt = task >> 1;
        rt += rt >= p ? 1 : 0;
        const int c0 = 16 * (task & 1), i = 32 * rt + lane;
        double v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = Prow[(c0 + c) * lds + i];
        double* dst = row(i) + p0 + c0;
#pragma unroll
        for (int c = 0; c < 16; c += 2)
          *reinterpret_cast<double2*>(dst + c) = make_double2(v[c], v[c + 1]);
      }
      for (int e = gw * 32 + lane; e < 32 * 32; e += GW * 32) {
        double* q = Prow + (e >> 5) * lds + p0 + (e & 31);
        *q = -*q;
      }
      mc_barrier(ctr, target, K);
    }
  }
  // the last line's -W: stored column j is the head of row j
  double* dst = fac + (long long)(nr - 1) * lsz;
  for (int j = gw; j < NPS; j += GW) {
    const int m16 = 16 * (j >> 4) + 16;
    for (int r = lane; r < m16; r += 32) __stcs(dst + col_off(j) + r, row(j)[r]);
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(&status[sid], 1);
}

cudaError_t launch_block_factor_mc(int cnt, int K, cudaStream_t st, const SubInfo* subs,
                                   const int* list, const Phys* P, const double* JDpool,
                                   double* fac_pool, double* mscratch, long long ms_stride,
                                   int* status, unsigned long long* bars) {
  Phys p = *P;
  void* args[] = {(void*)&subs, (void*)&list, (void*)&K, (void*)&p, (void*)&JDpool,
                  (void*)&fac_pool, (void*)&mscratch, (void*)&ms_stride, (void*)&status,
                  (void*)&bars};
  return cudaLaunchCooperativeKernel((void*)k_block_factor_mc, cnt * K, BF_THREADS, args, 0, st);
}
#endif

int block_factor_smem_bytes(int max_npb) {
  (void)max_npb;   // fixed layout: [S: 160 x 164][W0, W1: 32 x 33][JL: 4 x 112]
  return (int)sizeof(double) * (BF_SMEM_MAX_NPB * (BF_SMEM_MAX_NPB + 4) + 2 * 32 * WLD + 4 * BF_JL_POINTS);
}

// ---------------------------------------------------------------------------
// solve with the stored S_a^{-1}
// ---------------------------------------------------------------------------
// One stage of the solve ring holds two tile columns of a line, c and
// cpb-1-c (the middle one alone when cpb is odd), so every stage carries the
// same bytes (~90-100 KB in flight per CTA).  Stages are sized for pairs up
// to cpb = 11 (config 4's corner: two CTAs per SM still fit); a subdomain
// whose pairs do not fit streams one tile column per stage.
__host__ __device__ inline int bs_stage_doubles(int max_nps) {
  const int cpb = max_nps / 16, pc = cpb < 11 ? cpb : 11;
  const int pair = 256 * pc + 320, single = (int)block_col_doubles(cpb - 1);
  return pair > single ? pair : single;
}
// two threads per row (one warp per tile row) + one producer warp
__host__ __device__ inline int bs_threads(int max_nps) { return 2 * max_nps + 32; }

// Solve with the stored W_a.  Thread (i, h) (warp ti = i / 16, lane = 16h +
// i % 16) accumulates two halves of row i of the FULL symmetric W_a v':
//   row part     W[i][16c + 8h + k] v'[16c + 8h + k]   stored tiles (ti, c), c >= ti
//   column part  W[r][i] v'[r], r < 16 ti, r = 4q + 2h + {0, 1}  (= W[i][r])
// so every thread does 8 cpb FMAs per line whatever its tile, no cross-thread
// reductions are needed (one shuffle joins the halves), and each stored
// element is read from shared memory twice (once per product).  Warps move
// through the ring independently: a producer warp refills a slot once every
// consumer warp has released it (empty mbarriers), and the consumers meet
// once per line (named barrier 1) because line a+1 needs all of line a.
// JVP right-hand side of local point t (= 2b + f) of oriented line a: the
// coupling to the outside of the rectangle, e = A_ext d (schwarz.py:341-342),
// in k_jvp_rhs's operation order (zero for points with no outside neighbour)
__device__ __forceinline__ double jvp_rhs(const SubInfo& s, const double* d, int gn, double off,
                                          int a, int t) {
  const int b = t >> 1, f = t & 1;
  int i, j;
  local_to_global(s, a, b, i, j);
  const long long Ntot = (long long)gn * gn;
  const int di[4] = {-1, 0, 0, 1};
  const int dj[4] = {0, -1, 1, 0};
  double e = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ii = i + di[u], jj = j + dj[u];
    if (ii < 0 || ii >= gn || jj < 0 || jj >= gn || in_rect(s, ii, jj)) continue;
    e = add(e, mul(off, d[f * Ntot + (long long)ii * gn + jj]));
  }
  return e;
}

// RAS-apply right-hand side: the global v restricted to local point t of line a
__device__ __forceinline__ double ras_rhs(const SubInfo& s, const double* v, int gn, int a, int t) {
  int i, j;
  local_to_global(s, a, t >> 1, i, j);
  return v[(long long)(t & 1) * gn * gn + (long long)i * gn + j];
}

template <int MODE>
__global__ void __launch_bounds__(BS_MAX_THREADS, 2)
k_block_solve(const SubInfo* subs, const int* list, const double* fac_pool, const double* in_pool,
              double scale, double* out_pool, double off, int max_npb, const double* dglob,
              double* oglob, int gn) {
  // MODE 0: solve pool -> pool.  MODE 1: the backward sweep stops at the first
  // owned line.  MODE 2: the fused JVP (schwarz.py:327-345): MODE 1 with the
  // right-hand side A_ext d computed from the global d and out[own] =
  // -(d + x)[own] written straight to the global vector.  MODE 3: the fused
  // RAS apply (schwarz.py:221-239): right-hand side v restricted to the
  // rectangle, out[own] = x[own].
  extern __shared__ __align__(16) double sm[];
  const SubInfo s = subs[list[blockIdx.x]];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NPS = s.NPS, n = 2 * s.nc, nr = s.nr;   // stored block size (multiple of 16)
  const int SBS = bs_stage_doubles(max_npb);
  double* stage = sm;                                 // [BS_STAGES][SBS]
  double* vp = sm + BS_STAGES * SBS;                  // [2][max_npb]: P vin, double-buffered by line
  __shared__ __align__(8) uint64_t full[BS_STAGES], empty[BS_STAGES];
  const double* fac = fac_pool + s.fac;
  const double* in = in_pool + s.loc;
  double* out = out_pool + s.loc;
  const long long lsz = block_line_doubles(NPS);
  const int cpb = NPS / 16;                           // tile columns per line = consumer warps
  const bool paired = 256 * cpb + 320 <= SBS;
  const int nst = paired ? (cpb + 1) / 2 : cpb;       // stages per line
  int a_stop = 0;
  if (MODE >= 1) a_stop = s.orient == 0 ? s.or0 - s.r0 : s.oc0 - s.c0;
  const int nback = nr - 1 - a_stop > 0 ? nr - 1 - a_stop : 0;   // lines a = nr-2 .. a_stop
  const int nlines = nr + nback, total = nlines * nst;
  if (tid == 0) {
    for (int i = 0; i < BS_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], cpb);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // line 0 input, stored permuted: vp[t ^ 1] = vin[t]
  for (int t = tid; t < NPS; t += blockDim.x)
    vp[t ^ 1] = t < n ? (MODE == 2 ? jvp_rhs(s, dglob, gn, off, 0, t)
                         : MODE == 3 ? ras_rhs(s, dglob, gn, 0, t) : scale * in[t]) : 0.0;
  __syncthreads();
  if (warp == (int)(blockDim.x >> 5) - 1) {
    // ---- producer: stage t = (line blk, k) into slot t % BS_STAGES
    if (lane == 0) {
      // the next line is prefetched into L2 as one bulk range while the
      // ring issues the last BS_PF_EARLY+1 stages of the current line
      auto line_of = [&](int b) { return b < nr ? b : nr - 2 - (b - nr); };
      const int kpf = nst - 1 - BS_PF_EARLY > 0 ? nst - 1 - BS_PF_EARLY : 0;
      int blk = 0, k = 0;
      for (int t = 0; t < total; ++t) {
        const int st = t % BS_STAGES;
        if (t >= BS_STAGES) mbar_wait(&empty[st], ((t / BS_STAGES) - 1) & 1);
        const int a = line_of(blk);
        const int k2 = paired ? cpb - 1 - k : k;
        const double* src = fac + a * lsz;
        // a pair (k, cpb-1-k) is contiguous in the store
        const uint32_t bytes = (uint32_t)(8 * (block_col_doubles(k) + (k2 != k ? block_col_doubles(k2) : 0)));
        mbar_expect_tx(&full[st], bytes);
        // (one copy per tile column measured ~1 % faster than one per pair)
        bulk_g2s(stage + st * SBS, src + block_col_off(k, cpb), (uint32_t)(8 * block_col_doubles(k)),
                 &full[st]);
        if (k2 != k)
          bulk_g2s(stage + st * SBS + block_col_doubles(k), src + block_col_off(k2, cpb),
                   (uint32_t)(8 * block_col_doubles(k2)), &full[st]);
        if (BS_PF_EARLY >= 0 && k == kpf && blk + 1 < nlines)
          bulk_prefetch_l2(fac + line_of(blk + 1) * lsz, (uint32_t)(8 * lsz));
        if (++k == nst) { k = 0; ++blk; }
      }
    }
    return;
  }
  if (warp >= cpb) return;   // consumer warps beyond this subdomain's tile rows
  const int ti = warp, jj = lane & 15, h = lane >> 4, i = 16 * ti + jj;
  int st = 0;
  uint32_t ph = 0;
  for (int blk = 0; blk < nlines; ++blk) {
    const bool fwd = blk < nr;
    const int a = fwd ? blk : nr - 2 - (blk - nr);
    const double* v = vp + (blk & 1) * max_npb;
    double* vnext = vp + ((blk + 1) & 1) * max_npb;
    // prefetch of this row's combine operand (in_{a+1} forward, w_a backward)
    double nxt = 0.0;
    if (h == 0 && i < n) {
      if (fwd) {
        if (a + 1 < nr)
          nxt = MODE == 2 ? jvp_rhs(s, dglob, gn, off, a + 1, i)
                : MODE == 3 ? ras_rhs(s, dglob, gn, a + 1, i) : in[(long long)(a + 1) * n + i];
      } else {
        nxt = out[(long long)a * n + i];
      }
    }
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    auto tile_column = [&](const double* cb, int c) {
      const int ld2 = 16 * c + 18;
      if (c >= ti) {   // row part: this row's 8 columns of tile (ti, c)
        const double* w = cb + 8 * h * ld2 + i;
        const double2* vv = reinterpret_cast<const double2*>(v + 16 * c + 8 * h);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 x = vv[k >> 1];
          p0 = fma(w[k * ld2], x.x, p0);
          p1 = fma(w[(k + 1) * ld2], x.y, p1);
        }
      }
      if (c == ti) {   // column part: stored column i above the diagonal tile
        const double* cj = cb + jj * ld2 + 2 * h;
        const double* vr = v + 2 * h;
#pragma unroll 4
        for (int r = 0; r < 16 * c; r += 4) {
          const double2 x = *reinterpret_cast<const double2*>(cj + r);
          const double2 y = *reinterpret_cast<const double2*>(vr + r);
          p2 = fma(x.x, y.x, p2);
          p3 = fma(x.y, y.y, p3);
        }
      }
    };
    for (int k = 0; k < nst; ++k) {
      const int k2 = paired ? cpb - 1 - k : k;
      mbar_wait(&full[st], ph);
      const double* ch = stage + st * SBS;
      tile_column(ch, k);
      if (k2 != k) tile_column(ch + block_col_doubles(k), k2);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == BS_STAGES) { st = 0; ph ^= 1; }
    }
    double y = -((p0 + p1) + (p2 + p3));        // the store holds -W
    y += __shfl_xor_sync(0xffffffffu, y, 16);   // (S_a^{-1} vin)[i]
    if (h == 0) {
      double x = 0.0;   // x_a where this line is final (backward, or the last line)
      if (fwd) {
        // w_a = y; next input = scale in_{a+1} - off w_a (the last line starts
        // the backward sweep with x_{nr-1} = w_{nr-1})
        const double w = i < n ? y : 0.0;
        if (i < n && (MODE < 2 || a + 1 < nr)) out[(long long)a * n + i] = w;
        vnext[i ^ 1] = (a + 1 < nr) ? (i < n ? fma(-off, w, scale * nxt) : 0.0) : w;
        x = w;
      } else {
        // x_a = w_a - off y ; next input = x_a
        x = i < n ? fma(-off, y, nxt) : 0.0;
        if (MODE < 2 && i < n) out[(long long)a * n + i] = x;
        vnext[i ^ 1] = x;
      }
      if (MODE >= 2 && (!fwd || a + 1 == nr) && i < n) {
        // out[own] = -(d_loc + x)[own] (JVP, k_jvp_out's rounding) or x[own] (RAS)
        int gi, gj;
        local_to_global(s, a, i >> 1, gi, gj);
        if (gi >= s.or0 && gi < s.or1 && gj >= s.oc0 && gj < s.oc1) {
          const long long g = (long long)(i & 1) * gn * gn + (long long)gi * gn + gj;
          oglob[g] = MODE == 2 ? -add(dglob[g], x) : x;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * cpb) : "memory");
  }
}

// ---------------------------------------------------------------------------
// k_block_solve_wide: the same solve for lines wider than the fast kernel's
// limit (NPS > 224, i.e. a short side above 112 points: coarse
// decompositions and the monolithic direct solve of newton[-eps]).
// Warp w < NWC owns tile rows w, w + NWC, ... (TR of them, NWC <= 31);
// the producer streams each tile column in units of G of its 16 columns
// (G * (16c + 18) doubles <= WIDE_SBS; G = 16 up to cpb = 32), so any width
// fits the ring.  Row
// and column parts are those of k_block_solve; tile columns are visited in
// order 0 .. cpb-1 (two accumulators per row).
// ---------------------------------------------------------------------------
constexpr int WIDE_SBS = 8192;   // doubles per ring stage (64 KB): whole tile columns up to cpb = 32
constexpr int WIDE_STAGES = 3;

__host__ __device__ inline int wide_group(int cpb) {   // columns per unit
  int g = 16;
  while (g > 1 && (long long)g * (16 * (cpb - 1) + 18) > WIDE_SBS) g >>= 1;
  return g;
}

template <int MODE, int TR>
__global__ void __launch_bounds__(1024, 1)
k_block_solve_wide(const SubInfo* subs, const int* list, const double* fac_pool,
                   const double* in_pool, double scale, double* out_pool, double off, int max_nps,
                   const double* dglob, double* oglob, int gn) {
  extern __shared__ __align__(16) double sm[];
  const SubInfo s = subs[list[blockIdx.x]];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NPS = s.NPS, n = 2 * s.nc, nr = s.nr, cpb = NPS / 16;
  const int NWC = (cpb + TR - 1) / TR;                // consumer warps of this subdomain
  const int G = wide_group(cpb), upc = 16 / G, nunits = cpb * upc;
  double* stage = sm;                                 // [WIDE_STAGES][WIDE_SBS]
  double* vp = sm + WIDE_STAGES * WIDE_SBS;             // [2][max_nps]
  __shared__ __align__(8) uint64_t full[WIDE_STAGES], empty[WIDE_STAGES];
  const double* fac = fac_pool + s.fac;
  const double* in = in_pool + s.loc;
  double* out = out_pool + s.loc;
  const long long lsz = block_line_doubles(NPS);
  int a_stop = 0;
  if (MODE >= 1) a_stop = s.orient == 0 ? s.or0 - s.r0 : s.oc0 - s.c0;
  const int nback = nr - 1 - a_stop > 0 ? nr - 1 - a_stop : 0;
  const int nlines = nr + nback;
  if (tid == 0) {
    for (int i = 0; i < WIDE_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < NPS; t += blockDim.x)
    vp[t ^ 1] = t < n ? (MODE == 2 ? jvp_rhs(s, dglob, gn, off, 0, t)
                         : MODE == 3 ? ras_rhs(s, dglob, gn, 0, t) : scale * in[t]) : 0.0;
  __syncthreads();
  auto line_of = [&](int b) { return b < nr ? b : nr - 2 - (b - nr); };
  if (warp == (int)(blockDim.x >> 5) - 1) {
    if (lane == 0) {
      const long long total = (long long)nlines * nunits;
      for (long long t = 0; t < total; ++t) {
        const int st = (int)(t % WIDE_STAGES);
        if (t >= WIDE_STAGES) mbar_wait(&empty[st], (uint32_t)(((t / WIDE_STAGES) - 1) & 1));
        const int blk = (int)(t / nunits), u = (int)(t % nunits);
        const int c = u / upc, q0 = (u % upc) * G, ld2 = 16 * c + 18;
        const double* src = fac + line_of(blk) * lsz + block_col_off(c, cpb) + (long long)q0 * ld2;
        const uint32_t bytes = (uint32_t)(8 * G * ld2);
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(stage + st * WIDE_SBS, src, bytes, &full[st]);
        if (u == 0 && blk + 1 < nlines)   // the whole next line into L2 (short TMA latency)
          bulk_prefetch_l2(fac + line_of(blk + 1) * lsz, (uint32_t)(8 * lsz));
      }
    }
    return;
  }
  if (warp >= NWC) return;
  const int jj = lane & 15, h = lane >> 4;
  int st = 0;
  uint32_t ph = 0;
  for (int blk = 0; blk < nlines; ++blk) {
    const bool fwd = blk < nr;
    const int a = line_of(blk);
    const double* v = vp + (blk & 1) * max_nps;
    double* vnext = vp + ((blk + 1) & 1) * max_nps;
    double acc[TR][2];
#pragma unroll
    for (int r = 0; r < TR; ++r) acc[r][0] = acc[r][1] = 0.0;
    for (int u = 0; u < nunits; ++u) {
      const int c = u / upc, q0 = (u % upc) * G, ld2 = 16 * c + 18;
      mbar_wait(&full[st], ph);
      const double* cb = stage + st * WIDE_SBS;   // columns q0 .. q0+G-1 of tile column c
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        const int ti = warp + NWC * r;
        if (ti >= cpb) continue;
        const int i = 16 * ti + jj;
        if (c >= ti) {   // row part: columns 8h .. 8h+7 of tile (ti, c) inside this unit
          const int k0 = max(8 * h, q0), k1 = min(8 * h + 8, q0 + G);
          for (int q = k0; q < k1; ++q) acc[r][q & 1] = fma(cb[(q - q0) * ld2 + i], v[16 * c + q], acc[r][q & 1]);
        }
        if (c == ti && jj >= q0 && jj < q0 + G) {   // column part: stored column i above the diagonal tile
          const double* cj = cb + (jj - q0) * ld2 + 2 * h;
          const double* vr = v + 2 * h;
          for (int rr = 0; rr < 16 * c; rr += 4) {
            const double2 x = *reinterpret_cast<const double2*>(cj + rr);
            const double2 y = *reinterpret_cast<const double2*>(vr + rr);
            acc[r][0] = fma(x.x, y.x, acc[r][0]);
            acc[r][1] = fma(x.y, y.y, acc[r][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == WIDE_STAGES) { st = 0; ph ^= 1; }
    }
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int ti = warp + NWC * r;
      if (ti >= cpb) continue;
      const int i = 16 * ti + jj;
      double y = -(acc[r][0] + acc[r][1]);        // the store holds -W
      y += __shfl_xor_sync(0xffffffffu, y, 16);
      if (h == 0) {
        double nxt = 0.0;
        if (i < n) {
          if (fwd) {
            if (a + 1 < nr)
              nxt = MODE == 2 ? jvp_rhs(s, dglob, gn, off, a + 1, i)
                    : MODE == 3 ? ras_rhs(s, dglob, gn, a + 1, i) : in[(long long)(a + 1) * n + i];
          } else {
            nxt = out[(long long)a * n + i];
          }
        }
        double x = 0.0;
        if (fwd) {
          const double w = i < n ? y : 0.0;
          if (i < n && (MODE < 2 || a + 1 < nr)) out[(long long)a * n + i] = w;
          vnext[i ^ 1] = (a + 1 < nr) ? (i < n ? fma(-off, w, scale * nxt) : 0.0) : w;
          x = w;
        } else {
          x = i < n ? fma(-off, y, nxt) : 0.0;
          if (MODE < 2 && i < n) out[(long long)a * n + i] = x;
          vnext[i ^ 1] = x;
        }
        if (MODE >= 2 && (!fwd || a + 1 == nr) && i < n) {
          int gi, gj;
          local_to_global(s, a, i >> 1, gi, gj);
          if (gi >= s.or0 && gi < s.or1 && gj >= s.oc0 && gj < s.oc1) {
            const long long g = (long long)(i & 1) * gn * gn + (long long)gi * gn + gj;
            oglob[g] = MODE == 2 ? -add(dglob[g], x) : x;
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * NWC) : "memory");
  }
}

size_t block_solve_wide_smem_bytes(int max_nps) {
  return sizeof(double) * ((size_t)WIDE_STAGES * WIDE_SBS + 2 * (size_t)max_nps);
}

template <int MODE>
static cudaError_t launch_wide_mode(int grid, cudaStream_t st, const SubInfo* subs, const int* list,
                                    const double* fac, const double* in, double scale,
                                    double* out_pool, double off, int max_nps, const double* dglob,
                                    double* oglob, int gn) {
  const int cpb = max_nps / 16;
  const size_t smem = block_solve_wide_smem_bytes(max_nps);
  int tr = 1;
  while ((cpb + tr - 1) / tr > 31) tr *= 2;
  const int nt = 32 * ((cpb + tr - 1) / tr + 1);
#define OCP_WIDE(TRV)                                                                           \
  do {                                                                                          \
    cudaError_t e = raise_smem_limit((const void*)k_block_solve_wide<MODE, TRV>, (int)smem);    \
    if (e != cudaSuccess) return e;                                                             \
    k_block_solve_wide<MODE, TRV><<<grid, nt, smem, st>>>(subs, list, fac, in, scale, out_pool, \
                                                          off, max_nps, dglob, oglob, gn);      \
  } while (0)
  if (tr == 1) OCP_WIDE(1);
  else if (tr == 2) OCP_WIDE(2);
  else if (tr == 4) OCP_WIDE(4);
  else if (tr == 8) OCP_WIDE(8);
  else return cudaErrorInvalidConfiguration;   // NPS > 3968: short side above 1984 points
#undef OCP_WIDE
  return cudaGetLastError();
}

int block_solve_max_nps() { return 16 * 31 * 8; }

#ifndef OCP_NARROW_INSTANCE
size_t block_solve_mc_smem_bytes(int max_nps);
#endif

#ifndef OCP_NARROW_INSTANCE
// ---------------------------------------------------------------------------
// k_block_solve_mc: the block solve for FEW WIDE subdomains, K CTAs per
// subdomain (cooperative).  The stored tile columns of a line are split in
// units of 8 columns, dealt round-robin to the K CTAs; each CTA streams its
// units (TMA ring) and forms, for every row i, its partial of (-W_a v)[i]
// (row parts of its columns, column parts of the stored columns it holds).
// The partials go to a per-subdomain buffer, one arrival barrier per line,
// and every CTA sums the K partials of all rows in rank order
// (deterministic) and continues the forward / backward recurrence; rank 0
// writes the outputs.  Rows: two threads each (one warp per tile row) + a
// producer warp, so NPS <= 496.
// ---------------------------------------------------------------------------
constexpr int MC_UNIT_COLS = 8;
constexpr int MC_SBS = 8 * (16 * 30 + 18) + 32;   // one unit of the widest tile column (NPS 496)
constexpr int MC_STAGES = 6;

template <int MODE>
__global__ void __launch_bounds__(1024, 1)
k_block_solve_mc(const SubInfo* subs, const int* list, int K, const double* fac_pool,
                 const double* in_pool, double scale, double* out_pool, double off, int max_nps,
                 const double* dglob, double* oglob, int gn, double* partials,
                 unsigned long long* bars) {
  extern __shared__ __align__(16) double sm[];
  const int li = blockIdx.x / K, rank = blockIdx.x - li * K;
  const SubInfo s = subs[list[li]];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NPS = s.NPS, n = 2 * s.nc, nr = s.nr, cpb = NPS / 16;
  const int upc = 16 / MC_UNIT_COLS, nunits = cpb * upc;
  const int mine = nunits > rank ? (nunits - rank + K - 1) / K : 0;   // units of this CTA per line
  double* stage = sm;                                  // [MC_STAGES][MC_SBS]
  double* vp = sm + MC_STAGES * MC_SBS;                // [2][max_nps]
  __shared__ __align__(8) uint64_t full[MC_STAGES], empty[MC_STAGES];
  const double* fac = fac_pool + s.fac;
  const double* in = in_pool + s.loc;
  double* out = out_pool + s.loc;
  const long long lsz = block_line_doubles(NPS);
  double* part = partials + (long long)li * 2 * K * max_nps;   // [2][K][max_nps]
  unsigned long long* ctr = bars + 16 * li;
  unsigned long long target = 0;
  int a_stop = 0;
  if (MODE >= 1) a_stop = s.orient == 0 ? s.or0 - s.r0 : s.oc0 - s.c0;
  const int nback = nr - 1 - a_stop > 0 ? nr - 1 - a_stop : 0;
  const int nlines = nr + nback;
  if (tid == 0) {
    for (int i = 0; i < MC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], cpb);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < NPS; t += blockDim.x)
    vp[t ^ 1] = t < n ? (MODE == 2 ? jvp_rhs(s, dglob, gn, off, 0, t)
                         : MODE == 3 ? ras_rhs(s, dglob, gn, 0, t) : scale * in[t]) : 0.0;
  __syncthreads();
  auto line_of = [&](int b) { return b < nr ? b : nr - 2 - (b - nr); };
  const int nwarps = (int)(blockDim.x >> 5);
  const bool producer = warp == nwarps - 1 && lane == 0;
  long long tp = 0;   // producer's unit counter (ring slot = tp % MC_STAGES)
  auto issue_line = [&](int blk) {   // this CTA's units of line blk (mine <= MC_STAGES / 2)
    for (int k = 0; k < mine; ++k, ++tp) {
      const int st = (int)(tp % MC_STAGES);
      if (tp >= MC_STAGES) mbar_wait(&empty[st], (uint32_t)(((tp / MC_STAGES) - 1) & 1));
      const int u = rank + K * k;
      const int c = u / upc, q0 = (u % upc) * MC_UNIT_COLS, ld2 = 16 * c + 18;
      const double* src = fac + line_of(blk) * lsz + block_col_off(c, cpb) + (long long)q0 * ld2;
      const uint32_t bytes = (uint32_t)(8 * MC_UNIT_COLS * ld2);
      mbar_expect_tx(&full[st], bytes);
      bulk_g2s(stage + st * MC_SBS, src, bytes, &full[st]);
    }
  };
  if (producer) issue_line(0);
  const bool consumer = warp < cpb;
  const int ti = warp, jj = lane & 15, h = lane >> 4, i = 16 * ti + jj;
  int st = 0;
  uint32_t ph = 0;
  for (int blk = 0; blk < nlines; ++blk) {
    const bool fwd = blk < nr;
    const int a = line_of(blk);
    const double* v = vp + (blk & 1) * max_nps;
    double* vnext = vp + ((blk + 1) & 1) * max_nps;
    // this row's combine operand, read before the line's barrier (backward:
    // rank 0 overwrites out[a] with x_a after it)
    double nxt = 0.0;
    if (consumer && h == 0 && i < n) {
      if (fwd) {
        if (a + 1 < nr)
          nxt = MODE == 2 ? jvp_rhs(s, dglob, gn, off, a + 1, i)
                : MODE == 3 ? ras_rhs(s, dglob, gn, a + 1, i) : in[(long long)(a + 1) * n + i];
      } else {
        nxt = out[(long long)a * n + i];
      }
    }
    if (producer && blk + 1 < nlines) issue_line(blk + 1);
    double p0 = 0.0, p1 = 0.0;
    if (consumer) {
      for (int k = 0; k < mine; ++k) {
        const int u = rank + K * k;
        const int c = u / upc, q0 = (u % upc) * MC_UNIT_COLS, ld2 = 16 * c + 18;
        mbar_wait(&full[st], ph);
        const double* cb = stage + st * MC_SBS;   // columns q0 .. q0+7 of tile column c
        if (c >= ti && q0 == MC_UNIT_COLS * h) {   // row part: this thread's 8 columns
#pragma unroll
          for (int q = 0; q < MC_UNIT_COLS; q += 2) {
            p0 = fma(cb[q * ld2 + i], v[16 * c + q0 + q], p0);
            p1 = fma(cb[(q + 1) * ld2 + i], v[16 * c + q0 + q + 1], p1);
          }
        }
        if (c == ti && jj >= q0 && jj < q0 + MC_UNIT_COLS) {   // column part
          const double* cj = cb + (jj - q0) * ld2 + 2 * h;
          const double* vr = v + 2 * h;
          for (int r = 0; r < 16 * c; r += 4) {
            const double2 x = *reinterpret_cast<const double2*>(cj + r);
            const double2 y = *reinterpret_cast<const double2*>(vr + r);
            p0 = fma(x.x, y.x, p0);
            p1 = fma(x.y, y.y, p1);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == MC_STAGES) { st = 0; ph ^= 1; }
      }
      double y = p0 + p1;
      y += __shfl_xor_sync(0xffffffffu, y, 16);
      if (h == 0) part[((long long)(blk & 1) * K + rank) * max_nps + i] = y;
    }
    mc_barrier(ctr, target, K);
    if (consumer && h == 0) {
      double y = 0.0;
      for (int r = 0; r < K; ++r) y += __ldcg(part + ((long long)(blk & 1) * K + r) * max_nps + i);
      y = -y;   // the store holds -W
      double x = 0.0;
      if (fwd) {
        const double w = i < n ? y : 0.0;
        if (rank == 0 && i < n && (MODE < 2 || a + 1 < nr)) out[(long long)a * n + i] = w;
        vnext[i ^ 1] = (a + 1 < nr) ? (i < n ? fma(-off, w, scale * nxt) : 0.0) : w;
        x = w;
      } else {
        x = i < n ? fma(-off, y, nxt) : 0.0;
        if (rank == 0 && MODE < 2 && i < n) out[(long long)a * n + i] = x;
        vnext[i ^ 1] = x;
      }
      if (rank == 0 && MODE >= 2 && (!fwd || a + 1 == nr) && i < n) {
        int gi, gj;
        local_to_global(s, a, i >> 1, gi, gj);
        if (gi >= s.or0 && gi < s.or1 && gj >= s.oc0 && gj < s.oc1) {
          const long long g = (long long)(i & 1) * gn * gn + (long long)gi * gn + gj;
          oglob[g] = MODE == 2 ? -add(dglob[g], x) : x;
        }
      }
    }
    __syncthreads();   // vnext complete; (backward) out[a] read before the next line writes
  }
}
#endif

size_t block_solve_smem_bytes(int max_npb) {
  return sizeof(double) * ((size_t)BS_STAGES * bs_stage_doubles(max_npb) + 2 * (size_t)max_npb);
}

cudaError_t launch_block_solve(int mode, int grid, cudaStream_t st, const SubInfo* subs,
                               const int* list, const double* fac, const double* in, double scale,
                               double* out_pool, double off, int max_npb, const double* dglob,
                               double* oglob, int gn) {
  const size_t smem = block_solve_smem_bytes(max_npb);
  const int nt = bs_threads(max_npb);
  if (nt > BS_MAX_THREADS) {   // short side above 112 points
    if (mode == 0) return launch_wide_mode<0>(grid, st, subs, list, fac, in, scale, out_pool, off, max_npb, dglob, oglob, gn);
    if (mode == 1) return launch_wide_mode<1>(grid, st, subs, list, fac, in, scale, out_pool, off, max_npb, dglob, oglob, gn);
    if (mode == 2) return launch_wide_mode<2>(grid, st, subs, list, fac, in, scale, out_pool, off, max_npb, dglob, oglob, gn);
    return launch_wide_mode<3>(grid, st, subs, list, fac, in, scale, out_pool, off, max_npb, dglob, oglob, gn);
  }
  if (mode == 0)
    k_block_solve<0><<<grid, nt, smem, st>>>(subs, list, fac, in, scale, out_pool, off, max_npb,
                                             dglob, oglob, gn);
  else if (mode == 1)
    k_block_solve<1><<<grid, nt, smem, st>>>(subs, list, fac, in, scale, out_pool, off, max_npb,
                                             dglob, oglob, gn);
  else if (mode == 2)
    k_block_solve<2><<<grid, nt, smem, st>>>(subs, list, fac, in, scale, out_pool, off, max_npb,
                                             dglob, oglob, gn);
  else
    k_block_solve<3><<<grid, nt, smem, st>>>(subs, list, fac, in, scale, out_pool, off, max_npb,
                                             dglob, oglob, gn);
  return cudaGetLastError();
}

cudaError_t set_block_kernel_smem(int factor_bytes, int solve_bytes) {
  cudaError_t e = raise_smem_limit((const void*)k_block_factor, factor_bytes);
  if (e != cudaSuccess) return e;
  e = raise_smem_limit((const void*)k_block_solve<0>, solve_bytes);
  if (e != cudaSuccess) return e;
  e = raise_smem_limit((const void*)k_block_solve<1>, solve_bytes);
  if (e != cudaSuccess) return e;
  e = raise_smem_limit((const void*)k_block_solve<2>, solve_bytes);
  if (e != cudaSuccess) return e;
  return raise_smem_limit((const void*)k_block_solve<3>, solve_bytes);
}

#ifndef OCP_NARROW_INSTANCE
size_t block_solve_mc_smem_bytes(int max_nps) {
  return sizeof(double) * ((size_t)MC_STAGES * MC_SBS + 2 * (size_t)max_nps);
}

// K CTAs per subdomain; partials: [cnt][2][K][max_nps] doubles, bars: 16 per subdomain (zeroed)
cudaError_t launch_block_solve_mc(int mode, int cnt, int K, cudaStream_t st, const SubInfo* subs,
                                  const int* list, const double* fac, const double* in,
                                  double scale, double* out_pool, double off, int max_nps,
                                  const double* dglob, double* oglob, int gn, double* partials,
                                  unsigned long long* bars) {
  const int cpb = max_nps / 16;
  const int nt = 32 * (cpb + 1);
  if (nt > 1024) return cudaErrorInvalidConfiguration;
  const size_t smem = block_solve_mc_smem_bytes(max_nps);
  void* fn = mode == 0 ? (void*)k_block_solve_mc<0> : mode == 1 ? (void*)k_block_solve_mc<1>
           : mode == 2 ? (void*)k_block_solve_mc<2> : (void*)k_block_solve_mc<3>;
  cudaError_t e = raise_smem_limit((const void*)fn, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&subs, (void*)&list, (void*)&K, (void*)&fac, (void*)&in, (void*)&scale,
                  (void*)&out_pool, (void*)&off, (void*)&max_nps, (void*)&dglob, (void*)&oglob,
                  (void*)&gn, (void*)&partials, (void*)&bars};
  return cudaLaunchCooperativeKernel(fn, cnt * K, nt, args, smem, st);
}
#endif

}  // namespace ocp
