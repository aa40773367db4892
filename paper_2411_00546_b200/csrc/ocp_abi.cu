// C ABI + host driver of the RASPEN hot path (declared in include/ocp_gpu.h).
//
// The batched inner Newton below is Algorithm 1 (newton.py:133-181) run for
// all subdomains at once with per-subdomain state (active / converged /
// failed, iteration count, frozen threshold, line-search alpha).  All
// decisions are made here on the host from device-reduced norms, in double,
// with the reference's exact comparisons; only vectors live on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ocp_gpu.h"
#include "ocp_kernels.cuh"

using namespace ocp;
namespace ocp_nw { void read_bphase(unsigned long long* out); }
namespace ocp { void read_bphase(unsigned long long* out);
                void read_aphase(unsigned long long* out); void read_subt(long long* out, int n); }

namespace {

thread_local std::string g_global_err;

struct Event {
  cudaEvent_t a, b;
  int cls;
  double flops, bytes;
};

enum { CLS_FACTOR = 0, CLS_SOLVE = 1, CLS_SWEEP = 2, CLS_JVP = 3, CLS_INNER_SOLVE = 4, CLS_MGS = 5,
       CLS_RESID = 6, NCLS = 7 };

}  // namespace

struct ocp_ctx {
  int n = 0, s1 = 0, s2 = 0, m = 0, I = 0;
  long long N = 0;
  Phys P{};
  std::vector<SubInfo> subs;
  std::vector<double> sub_flops;    // algorithmic band-LU flops per subdomain
  std::vector<double> sub_fbytes;   // algorithmic factor bytes of a full solve per subdomain
  std::vector<double> sub_jbytes;   // algorithmic factor bytes of a JVP solve (owned rows only)
  std::vector<long long> sub_dofs;  // 2 R C
  SubInfo* d_subs = nullptr;
  long long pool_len = 0, fac_len = 0, ref_len = 0, dof_total = 0;
  int maxW = 0, maxNP = 0;
  double *d_f = nullptr, *d_yd = nullptr;
  double *V = nullptr, *R = nullptr, *D = nullptr, *B = nullptr, *JD = nullptr;
  int *d_list_all = nullptr, *d_list = nullptr, *d_status = nullptr, *d_flags = nullptr;
  double *d_alpha = nullptr, *d_rpart = nullptr;   // d_rpart: per (subdomain, residual CTA) squared-norm partial
  unsigned long long* d_rbad = nullptr;   // per (subdomain, residual CTA) first bad phi'/phi
  int res_chunks = 1;
  int res_smem = 0;           // dynamic shared memory of k_residual
  long long* d_bad = nullptr;
  int maxNPB = 0, maxNPS = 0;
  int* d_flist = nullptr;      // block format: factor list ordered by decreasing cost
  int* d_solve_order = nullptr;   // launch order of full-list block solves
  int* h_flist = nullptr;
  double* bscratch = nullptr;  // block format: global Schur blocks too large for shared memory
  long long bs_stride = 0;
  int bf_grid = 1;
  bool bf_narrow = false;     // narrow-line factor instance (ocp_block_narrow.cu)
  int mc_K = 0;               // > 1: K CTAs per subdomain (k_block_factor_mc, few wide subdomains)
  double* mscratch = nullptr; // their Schur blocks
  long long ms_stride = 0;
  unsigned long long* d_mcbars = nullptr;
  int mc_Ks = 0;              // > 1: K CTAs per subdomain in the block solves (k_block_solve_mc)
  double* mc_partials = nullptr;
  int num_sms = 148;
  double *red_partials = nullptr, *d_h = nullptr, *d_result = nullptr;
  unsigned int* red_counter = nullptr;
  unsigned long long* arn_bar = nullptr;   // split grid barrier of the Arnoldi kernel
  double* arn_partials = nullptr;          // [2][2048] block partials of the Arnoldi kernel
  unsigned long long arn_epoch = 0;        // arrivals so far on arn_bar
  double* gm_Q = nullptr;      // persistent GMRES basis (grow-only), ocp_raspen_gmres
  long long gm_n = 0;          // vector length the basis columns were sized for
  double* gm_w = nullptr;
  long long gm_cols = 0;
  double* gm_dh = nullptr;     // two device slots of Arnoldi coefficients (pipelined GMRES)
  double* gm_hh = nullptr;     // their pinned host copies
  int gm_hcap = 0;             // entries per slot
  cudaEvent_t gm_ev[2] = {nullptr, nullptr};
  double* gm_t = nullptr;      // J q_j of the preconditioned (linear-RAS) operator
  double* st_buf = nullptr;    // state-equation CG: dg, r, p, Ap (4 N doubles)
  double* st_sc = nullptr;     // CG scalars (rr, pAp, alpha, beta)
  double* st_hist = nullptr;   // CG r.r history (device) ...
  double* st_hhist = nullptr;  // ... and its pinned host copy
  int st_hcap = 0;
  unsigned long long* d_gbad = nullptr;   // first nonfinite phi'/phi'' of the global Jacobian
  int h_cap = 0;
  cudaStream_t stream = nullptr;
  // narrow-line factor: the few subdomains beyond its shared block run the
  // 12-warp kernel on a second stream beside the many small ones
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // pinned host staging
  double* h_norm2 = nullptr;   // squared residual norms per subdomain (finish_residual)
  double* h_rpart = nullptr;   // pinned: per-CTA partials of the last residual
  unsigned long long* h_rbad = nullptr;
  std::vector<long long> res_bad;   // first nonfinite phi'/phi'' key of the last residual with Jacobian diagonals
  int* h_status = nullptr;
  long long* h_bad = nullptr;
  int* h_list = nullptr;
  double* h_alpha = nullptr;
  double* h_small = nullptr;
  int* h_flags = nullptr;
  std::string err;
  // instrumentation
  bool prof = false;
  long long launches = 0;
  std::vector<Event> pending;
  std::vector<cudaEvent_t> free_events;
  double stat_ms[NCLS] = {};
  double stat_cnt[NCLS] = {};
  double stat_flops = 0, stat_bytes = 0, stat_dof = 0, stat_rbytes = 0;
  double resid_bytes_all = 0;   // algorithmic bytes of one full-set residual
  cudaEvent_t marks[16] = {};
};

namespace {

// The GMRES basis of a destroyed context (stream-ordered pool memory, its
// stream idle) is kept for the next context of the process: a fresh context
// of the same problem size then solves without growing a multi-GB basis by
// doubling (each growth a new pool block + copy; fragmented pool blocks made
// some growths map new physical memory in the middle of a solve).
std::mutex g_spare_mu;
double* g_spare_Q = nullptr;
size_t g_spare_bytes = 0;

void spare_put(double* q, size_t bytes, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_spare_mu);
  if (bytes > g_spare_bytes) std::swap(q, g_spare_Q), std::swap(bytes, g_spare_bytes);
  if (q) cudaFreeAsync(q, st);
}

double* spare_take(size_t min_bytes, size_t* bytes) {
  std::lock_guard<std::mutex> lk(g_spare_mu);
  if (!g_spare_Q || g_spare_bytes < min_bytes) return nullptr;
  double* q = g_spare_Q;
  *bytes = g_spare_bytes;
  g_spare_Q = nullptr;
  g_spare_bytes = 0;
  return q;
}

// Guard-zone allocator (OCP_GUARD=1 in the environment): every device buffer
// of the library gets GUARD_BYTES of a fill pattern on both sides, and
// ocp_check_guards counts pattern bytes that kernels overwrote - an
// out-of-bounds write detector that runs at full speed on any pool (the
// GPU pool refuses compute-sanitizer).  The interior is filled with the same
// pattern, so a read of never-written memory yields garbage, not zeros.
constexpr size_t GUARD_BYTES = 64 << 10;
constexpr unsigned char GUARD_FILL = 0xA5;
std::mutex g_guard_mu;
std::map<void*, std::pair<char*, size_t>> g_guards;   // user pointer -> (base, bytes)
bool guard_on() {
  static const bool on = [] {
    const char* v = getenv("OCP_GUARD");
    return v && v[0] == '1';
  }();
  return on;
}
cudaError_t guard_malloc(void** p, size_t bytes) {
  if (!guard_on()) return cudaMalloc(p, bytes);
  char* base = nullptr;
  cudaError_t e = cudaMalloc(&base, bytes + 2 * GUARD_BYTES);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, GUARD_FILL, bytes + 2 * GUARD_BYTES);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();   // before any non-blocking stream uses it
  if (e != cudaSuccess) return e;
  *p = base + GUARD_BYTES;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guards[*p] = {base, bytes};
  return cudaSuccess;
}
long long g_guard_freed_bad = 0;   // corrupted guard bytes of buffers already freed
std::string g_guard_first;
long long count_guard(const char* base, size_t bytes, std::string* first) {
  std::vector<unsigned char> h(GUARD_BYTES);
  long long bad = 0;
  for (int side = 0; side < 2; ++side) {
    const char* g = side ? base + GUARD_BYTES + bytes : base;
    if (cudaMemcpy(h.data(), g, GUARD_BYTES, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (size_t k = 0; k < GUARD_BYTES; ++k)
      if (h[k] != GUARD_FILL) {
        if (first && first->empty()) {
          char buf[160];
          snprintf(buf, sizeof buf, "buffer of %zu bytes: %s guard byte %zu overwritten", bytes,
                   side ? "tail" : "head", k);
          *first = buf;
        }
        ++bad;
      }
  }
  return bad;
}
cudaError_t guard_free(void* p) {
  if (!p) return cudaSuccess;
  if (guard_on()) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guards.find(p);
    if (it != g_guards.end()) {
      char* base = it->second.first;
      cudaDeviceSynchronize();   // the buffer's last kernels have finished
      const long long bad = count_guard(base, it->second.second, &g_guard_first);
      if (bad > 0) g_guard_freed_bad += bad;
      g_guards.erase(it);
      return cudaFree(base);
    }
  }
  return cudaFree(p);
}
template <class T>
cudaError_t gmalloc(T** p, size_t bytes) {
  void* v = nullptr;
  const cudaError_t e = guard_malloc(&v, bytes);
  *p = static_cast<T*>(v);
  return e;
}
cudaError_t gfree(void* p) { return guard_free(p); }

int fail(ocp_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf; else g_global_err = buf;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(ctx, OCP_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                             \
  } while (0)

#define CKL()                                                                      \
  do {                                                                             \
    ++ctx->launches;                                                               \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return fail(ctx, OCP_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                             \
  } while (0)

cudaEvent_t get_event(ocp_ctx* ctx) {
  if (!ctx->free_events.empty()) {
    cudaEvent_t e = ctx->free_events.back();
    ctx->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Timer {
  ocp_ctx* ctx;
  Event ev{};
  bool on;
  Timer(ocp_ctx* c, int cls, double flops = 0, double bytes = 0) : ctx(c), on(c && c->prof) {
    if (!on) return;
    ev.a = get_event(ctx);
    ev.b = get_event(ctx);
    ev.cls = cls;
    ev.flops = flops;
    ev.bytes = bytes;
    cudaEventRecord(ev.a, ctx->stream);
  }
  ~Timer() {
    if (!on) return;
    cudaEventRecord(ev.b, ctx->stream);
    ctx->pending.push_back(ev);
  }
};

void drain_events(ocp_ctx* ctx) {
  if (ctx->pending.empty()) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    ctx->stat_ms[e.cls] += ms;
    ctx->stat_cnt[e.cls] += 1;
    if (e.cls == CLS_FACTOR) ctx->stat_flops += e.flops;
    if (e.cls == CLS_SOLVE) ctx->stat_bytes += e.bytes;
    if (e.cls == CLS_RESID) ctx->stat_rbytes += e.bytes;
    ctx->free_events.push_back(e.a);
    ctx->free_events.push_back(e.b);
  }
  ctx->pending.clear();
}

std::vector<std::pair<int, int>> tile_edges(int n, int parts, bool& ok) {
  std::vector<std::pair<int, int>> out;
  const int base = n / parts, rem = n % parts;
  ok = base > 0;
  if (!ok) return out;
  for (int k = 0; k < parts; ++k) out.push_back({k * base, k * base + base + (k == parts - 1 ? rem : 0)});
  return out;
}

// exact band-LU flop count: sum_k m_k (1 + 2 u_k), m_k = u_k = min(w, N-1-k)
double band_lu_flops(long long N, long long w) {
  double tot = 0.0;
  for (long long k = 0; k < N; ++k) {
    const double m = (double)std::min(w, N - 1 - k);
    tot += m * (1.0 + 2.0 * m);
  }
  return tot;
}


// local residual (+ per-subdomain squared norms) of `cnt` listed subdomains
int launch_residual(ocp_ctx* ctx, const int* d_list, int cnt, const double* x, const double* V,
                    const double* D, const double* alpha, double eps, double* R, bool jd = false) {
  if (cnt == 0) return OCP_OK;
  // full-set residual evaluations are timed for the stencil roofline
  // (48 B per local point: read y,p,f,y_d, write r1,r2 - SURVEY.md 8d; with
  // the fused Jacobian diagonals 80 B: + the (dg, b12, b21, 0) write)
  {
  Timer t(cnt == ctx->I && !D ? ctx : nullptr, CLS_RESID, 0,
          ctx->resid_bytes_all * (jd ? 80.0 / 48.0 : 1.0));
  const dim3 grid(cnt, ctx->res_chunks);
  // every list is an ascending subset of the subdomains, so a full-count
  // list is the identity: the kernel then skips the list indirection
  if (!D)   // no staged direction: the compact L1-read path
    k_residual<true><<<grid, RES_THREADS, 0, ctx->stream>>>(
        ctx->d_subs, cnt == ctx->I ? nullptr : d_list, ctx->P, x, V, D, alpha, ctx->d_f, ctx->d_yd, eps, R,
        ctx->d_rpart, jd ? ctx->JD : nullptr, ctx->d_rbad);
  else
  k_residual<false><<<grid, RES_THREADS, ctx->res_smem, ctx->stream>>>(
      ctx->d_subs, cnt == ctx->I ? nullptr : d_list, ctx->P, x, V, D, alpha, ctx->d_f, ctx->d_yd, eps, R,
      ctx->d_rpart, jd ? ctx->JD : nullptr, ctx->d_rbad);
  CKL();
  }
  // the per-CTA partials come back with the copy the caller waits for anyway
  const size_t np = (size_t)ctx->I * ctx->res_chunks;
  CK(cudaMemcpyAsync(ctx->h_rpart, ctx->d_rpart, np * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (jd)
    CK(cudaMemcpyAsync(ctx->h_rbad, ctx->d_rbad, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
  return OCP_OK;
}

// after the stream synchronisation that follows launch_residual: squared norms
// of the listed subdomains (partials added in CTA order: deterministic) and,
// for a residual with Jacobian diagonals, their first nonfinite phi' / phi'' key
void finish_residual(ocp_ctx* ctx, const int* list, int cnt, bool jd) {
  const int ny = ctx->res_chunks;
  for (int k = 0; k < cnt; ++k) {
    const int i = list ? list[k] : k;
    double v = 0.0;
    for (int y = 0; y < ny; ++y) v += ctx->h_rpart[(size_t)i * ny + y];
    ctx->h_norm2[i] = v;
    if (jd) {
      unsigned long long b = ~0ull;
      for (int y = 0; y < ny; ++y) b = std::min(b, ctx->h_rbad[(size_t)i * ny + y]);
      ctx->res_bad[i] = b == ~0ull ? -1ll : (long long)b;
    }
  }
}

int upload_list(ocp_ctx* ctx, const std::vector<int>& list) {
  std::copy(list.begin(), list.end(), ctx->h_list);
  CK(cudaMemcpyAsync(ctx->d_list, ctx->h_list, list.size() * sizeof(int), cudaMemcpyHostToDevice,
                     ctx->stream));
  return OCP_OK;
}

int launch_factor(ocp_ctx* ctx, const int* d_list, const std::vector<int>& list, double* fac) {
  const int cnt = (int)list.size();
  if (cnt == 0) return OCP_OK;
  double flops = 0;
  for (int i : list) flops += ctx->sub_flops[i];
  Timer t(ctx, CLS_FACTOR, flops);
  {
    // persistent CTAs take subdomains in list order: largest work first
    // (global-memory Schur blocks, then nr * NPB^3), so the tail is short
    if (!ctx->d_flist) {   // lists + the work counters of the persistent CTAs
      CK(gmalloc(&ctx->d_flist, (ctx->I + 2) * sizeof(int)));
      CK(cudaMallocHost(&ctx->h_flist, (ctx->I + 2) * sizeof(int)));
    }
    CK(cudaStreamSynchronize(ctx->stream));   // h_flist may still feed a previous copy
    std::vector<int> ord(list);
    const int smem_npb = ctx->bf_narrow ? narrow_factor_max_npb() : BF_SMEM_MAX_NPB;
    auto cost = [&](int i) {
      const SubInfo& su = ctx->subs[i];
      const double c = (double)su.nr * su.pad_ * su.pad_ * su.pad_;
      return su.pad_ > smem_npb ? 4.0 * c : c;
    };
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return cost(x) > cost(y); });
    // narrow instance: [wide subdomains][counter][the others][counter]
    int nwide = 0;
    if (ctx->bf_narrow && ctx->mc_K <= 1) {
      std::stable_partition(ord.begin(), ord.end(), [&](int i) { return ctx->subs[i].pad_ > smem_npb; });
      while (nwide < cnt && ctx->subs[ord[nwide]].pad_ > smem_npb) ++nwide;
    }
    int* hl = ctx->h_flist;
    for (int i = 0; i < nwide; ++i) hl[i] = ord[i];
    const int off2 = nwide ? nwide + 1 : 0;   // second list (all of it when there is no wide one)
    if (nwide) hl[nwide] = 0;
    for (int i = nwide; i < cnt; ++i) hl[off2 + i - nwide] = ord[i];
    hl[off2 + cnt - nwide] = 0;
    CK(cudaMemcpyAsync(ctx->d_flist, hl, (cnt + (nwide ? 2 : 1)) * sizeof(int), cudaMemcpyHostToDevice,
                       ctx->stream));
    const int grid = std::min(cnt, ctx->bf_grid);
    if (ctx->mc_K > 1) {   // few wide subdomains: K CTAs each (status / barriers zeroed first)
      CK(cudaMemsetAsync(ctx->d_status, 0, ctx->I * sizeof(int), ctx->stream));
      CK(cudaMemsetAsync(ctx->d_mcbars, 0, (size_t)16 * ctx->I * sizeof(unsigned long long),
                         ctx->stream));
      cudaError_t e = launch_block_factor_mc(cnt, ctx->mc_K, ctx->stream, ctx->d_subs, ctx->d_flist,
                                             &ctx->P, ctx->JD, fac, ctx->mscratch, ctx->ms_stride,
                                             ctx->d_status, ctx->d_mcbars);
      if (e == cudaErrorCooperativeLaunchTooLarge) {   // SMs taken: one CTA per subdomain from now on
        cudaGetLastError();
        ctx->mc_K = ctx->mc_Ks = 0;
        return launch_factor(ctx, d_list, list, fac);
      }
      CK(e);
    } else if (ctx->bf_narrow) {
      if (nwide) {   // first, on the second stream: they take an SM each beside the narrow CTAs
        if (!ctx->stream2) {
          CK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        }
        CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->stream2, ctx->ev_fork, 0));
        k_block_factor<<<std::min(nwide, ctx->num_sms), block_factor_threads(),
                         block_factor_smem_bytes(ctx->maxNPB), ctx->stream2>>>(
            ctx->d_subs, ctx->d_flist, nwide, ctx->P, ctx->JD, fac, ctx->bscratch, ctx->bs_stride,
            ctx->d_status);
        CKL();
        CK(cudaEventRecord(ctx->ev_join, ctx->stream2));
      }
      if (cnt > nwide)
        CK(launch_narrow_factor(std::min(cnt - nwide, ctx->bf_grid), ctx->stream, ctx->d_subs,
                                ctx->d_flist + off2, cnt - nwide, &ctx->P, ctx->JD, fac, ctx->bscratch,
                                ctx->bs_stride, ctx->d_status));
      if (nwide) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
    } else {
      k_block_factor<<<grid, block_factor_threads(), block_factor_smem_bytes(ctx->maxNPB),
                       ctx->stream>>>(ctx->d_subs, ctx->d_flist, cnt, ctx->P, ctx->JD, fac,
                                      ctx->bscratch, ctx->bs_stride, ctx->d_status);
    }
    CKL();
    return OCP_OK;
  }
}

// every block solve goes through here: K CTAs per subdomain for few wide
// subdomains (k_block_solve_mc), else one CTA per subdomain
cudaError_t solve_dispatch(ocp_ctx* ctx, int mode, int cnt, const int* d_list, const double* fac,
                           const double* in, double scale, double* out_pool, const double* dglob,
                           double* oglob) {
  if (ctx->mc_Ks > 1) {
    cudaError_t e = cudaMemsetAsync(ctx->d_mcbars, 0, (size_t)16 * ctx->I * sizeof(unsigned long long),
                                    ctx->stream);
    if (e != cudaSuccess) return e;
    e = launch_block_solve_mc(mode, cnt, ctx->mc_Ks, ctx->stream, ctx->d_subs, d_list, fac, in,
                              scale, out_pool, ctx->P.off, ctx->maxNPS, dglob, oglob, ctx->P.n,
                              ctx->mc_partials, ctx->d_mcbars);
    if (e != cudaErrorCooperativeLaunchTooLarge) return e;
    cudaGetLastError();   // SMs taken: one CTA per subdomain from now on
    ctx->mc_Ks = 0;
  }
  return launch_block_solve(mode, cnt, ctx->stream, ctx->d_subs, d_list, fac, in, scale, out_pool,
                            ctx->P.off, ctx->maxNPS, dglob, oglob, ctx->P.n);
}

cudaError_t any_solve(ocp_ctx* ctx, int mode, int cnt, const int* d_list, const double* fac,
                      const double* in, double scale, double* out) {
  return solve_dispatch(ctx, mode, cnt, cnt == ctx->I ? ctx->d_solve_order : d_list, fac, in, scale,
                        out, nullptr, nullptr);
}

int launch_solve(ocp_ctx* ctx, const int* d_list, const std::vector<int>& list, const double* fac,
                 const double* in, double scale, double* out, int cls) {
  const int cnt = (int)list.size();
  if (cnt == 0) return OCP_OK;
  double bytes = 0;
  for (int i : list) bytes += ctx->sub_fbytes[i];
  Timer t(ctx, cls, 0, bytes);
  CK(any_solve(ctx, 0, cnt, d_list, fac, in, scale, out));
  ++ctx->launches;
  return OCP_OK;
}

inline int ew_grid(long long n) {
  long long g = (n + 255) / 256;
  return (int)std::max(1LL, std::min<long long>(g, 148LL * 16));
}

std::string fmt_e3(double v) {
  char buf[64];
  snprintf(buf, sizeof buf, "%.3e", v);
  return buf;
}

}  // namespace

extern "C" {

const char* ocp_last_error(const ocp_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_global_err.c_str();
}

int ocp_ctx_create(int n, int s1, int s2, int overlap, double nu, double mu, int phi_kind,
                   double kappa, const double* f_host, const double* y_d_host, ocp_ctx** out) {
  ocp_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, OCP_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (n < 1) return fail(nullptr, OCP_ERR_ARG, "grid needs at least one interior point per dimension");
  const bool grid_only = (s1 == 0 && s2 == 0);   // whole-grid operators only, no subdomains
  if (!grid_only && (s1 < 1 || s2 < 1))
    return fail(nullptr, OCP_ERR_ARG, "need at least one tile per dimension");
  if (overlap < 0) return fail(nullptr, OCP_ERR_ARG, "overlap must be nonnegative");
  if (!(nu > 0.0) || !(mu > 0.0)) return fail(nullptr, OCP_ERR_ARG, "nu and mu must be positive");
  if (phi_kind < 0 || phi_kind > 2) return fail(nullptr, OCP_ERR_ARG, "unknown phi kind %d", phi_kind);
  bool ok1 = true, ok2 = true;
  std::vector<std::pair<int, int>> rt, ct;
  if (!grid_only) {
    rt = tile_edges(n, s1, ok1);
    if (!ok1) return fail(nullptr, OCP_ERR_ARG, "cannot tile %d points into %d nonempty parts", n, s1);
    ct = tile_edges(n, s2, ok2);
    if (!ok2) return fail(nullptr, OCP_ERR_ARG, "cannot tile %d points into %d nonempty parts", n, s2);
  }
  auto minw = [](const std::vector<std::pair<int, int>>& t) {
    int m = INT_MAX;
    for (auto& e : t) m = std::min(m, e.second - e.first);
    return m;
  };
  if (s1 > 1 && overlap > minw(rt))
    return fail(nullptr, OCP_ERR_ARG, "overlap exceeds neighbor tile in the row direction");
  if (s2 > 1 && overlap > minw(ct))
    return fail(nullptr, OCP_ERR_ARG, "overlap exceeds neighbor tile in the column direction");
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return fail(nullptr, OCP_ERR_NO_DEVICE, "no CUDA device visible");

  ctx = new ocp_ctx();
  ctx->n = n; ctx->s1 = s1; ctx->s2 = s2; ctx->m = overlap;
  ctx->N = (long long)n * n;
  const double h = 1.0 / (n + 1);
  const double h2 = h * h;  // Python h ** 2 (correctly rounded square)
  ctx->P.n = n;
  ctx->P.phi_kind = phi_kind;
  ctx->P.diag = 4.0 / h2;
  ctx->P.off = -1.0 / h2;
  ctx->P.nu = nu;
  ctx->P.mu = mu;
  ctx->P.rnu = 1.0 / nu;   // correctly rounded on the host (dvd_const)
  ctx->P.rmu = 1.0 / mu;
  ctx->P.kappa = kappa;
  ctx->P.kappa2 = kappa * kappa;
  long long loc = 0, fac = 0, ref = 0;
  for (auto& r : rt) {
    for (auto& c : ct) {
      SubInfo s{};
      s.r0 = std::max(0, r.first - overlap);
      s.r1 = std::min(n, r.second + overlap);
      s.c0 = std::max(0, c.first - overlap);
      s.c1 = std::min(n, c.second + overlap);
      s.or0 = r.first; s.or1 = r.second; s.oc0 = c.first; s.oc1 = c.second;
      const int R = s.r1 - s.r0, C = s.c1 - s.c0;
      s.orient = C <= R ? 0 : 1;
      s.nr = std::max(R, C);
      s.nc = std::min(R, C);
      s.w = 2 * s.nc;
      // padded half-bandwidth: a multiple of 16, and at least one factor block
      // (the 32x32 in-block inverses are stored inside the band columns)
      s.W = std::max(((s.w + NB - 1) / NB) * NB, NBF);
      s.N = 2 * R * C;
      s.NP = ((s.N + NBF - 1) / NBF) * NBF;
      s.pad_ = ((2 * s.nc + 31) / 32) * 32;   // NPB (Gauss-Jordan panels of 32)
      s.NPS = ((2 * s.nc + 15) / 16) * 16;    // stored S_a^{-1} (solve chunks of 16 rows)
      s.loc = loc;
      s.fac = fac;
      s.ref = ref;
      loc += s.NP;
      ref += s.N;
      ctx->subs.push_back(s);
      ctx->sub_flops.push_back(band_lu_flops(s.N, s.w));
      // the JVP needs x only on the ownership block: the backward sweep stops
      // at its first oriented line (MODE 1 of both solve kernels)
      const int a_own = s.orient == 0 ? s.or0 - s.r0 : s.oc0 - s.c0;
      {
        // the upper 16-tile triangle of W_a = S_a^{-1} P per line (block_line_doubles):
        // forward reads all nr, backward nr-1-a_stop of them
        const double blk = 8.0 * (double)block_line_doubles(s.NPS);
        fac += (long long)s.nr * block_line_doubles(s.NPS);
        ctx->sub_fbytes.push_back(blk * (2.0 * s.nr - 1.0));
        ctx->sub_jbytes.push_back(blk * (s.nr + std::max(0, s.nr - 1 - a_own)));
      }
      ctx->maxNPB = std::max(ctx->maxNPB, s.pad_);
      ctx->maxNPS = std::max(ctx->maxNPS, s.NPS);
      ctx->sub_dofs.push_back(s.N);
      ctx->maxW = std::max(ctx->maxW, s.W);
      ctx->maxNP = std::max(ctx->maxNP, s.NP);
    }
  }
  ctx->I = (int)ctx->subs.size();
  ctx->pool_len = loc;
  ctx->fac_len = fac;
  ctx->ref_len = ref;
  auto cleanup_fail = [&](int code) {
    g_global_err = ctx->err;
    ocp_ctx_destroy(ctx);
    return code;
  };
#define CKC(call)                                                                       \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      fail(ctx, OCP_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));                \
      return cleanup_fail(OCP_ERR_CUDA);                                                \
    }                                                                                   \
  } while (0)
  int dev = 0;
  CKC(cudaGetDevice(&dev));
  CKC(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev));
  CKC(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  {
    // the GMRES basis (up to GBs, grown by doubling) comes from the device's
    // stream-ordered memory pool: growth needs no host synchronisation, and
    // the pool keeps the pages for the next context instead of unmapping them
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
      unsigned long long thr = 16ULL << 30;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  const int I = ctx->I;
  CKC(gmalloc(&ctx->d_subs, I * sizeof(SubInfo)));
  CKC(cudaMemcpy(ctx->d_subs, ctx->subs.data(), I * sizeof(SubInfo), cudaMemcpyHostToDevice));
  const size_t nbytes = ctx->N * sizeof(double);
  CKC(gmalloc(&ctx->d_f, nbytes));
  CKC(gmalloc(&ctx->d_yd, nbytes));
  CKC(cudaMemcpy(ctx->d_f, f_host, nbytes, cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(ctx->d_yd, y_d_host, nbytes, cudaMemcpyHostToDevice));
  const size_t pbytes = ctx->pool_len * sizeof(double);
  for (double** p : {&ctx->V, &ctx->R, &ctx->D, &ctx->B}) {
    CKC(gmalloc(p, pbytes));
    // (on the context's stream: it is non-blocking, so a legacy-default-stream
    // memset would not be ordered before the first kernels that use the buffer)
    CKC(cudaMemsetAsync(*p, 0, pbytes, ctx->stream));
  }
  CKC(gmalloc(&ctx->JD, 2 * pbytes));
  CKC(cudaMemsetAsync(ctx->JD, 0, 2 * pbytes, ctx->stream));
  CKC(gmalloc(&ctx->d_list_all, I * sizeof(int)));
  CKC(gmalloc(&ctx->d_list, I * sizeof(int)));
  CKC(gmalloc(&ctx->d_status, I * sizeof(int)));
  CKC(gmalloc(&ctx->d_alpha, I * sizeof(double)));
  {
    // residual grid: one CTA per RQ consecutive local points, staging the
    // points plus one local row either side in dynamic shared memory
    int maxt = 1, max_nc = 1;
    for (auto& sub : ctx->subs) {
      maxt = std::max(maxt, (sub.nr * sub.nc + RQ - 1) / RQ);
      max_nc = std::max(max_nc, sub.nc);
    }
    ctx->res_chunks = maxt;
    ctx->res_smem = (int)residual_smem_bytes(max_nc);
    CKC(raise_smem_limit((const void*)k_residual<false>, ctx->res_smem));
  }
  CKC(gmalloc(&ctx->d_rpart, (size_t)I * ctx->res_chunks * sizeof(double)));
  CKC(gmalloc(&ctx->d_rbad, (size_t)I * ctx->res_chunks * sizeof(unsigned long long)));
  CKC(gmalloc(&ctx->d_bad, I * sizeof(long long)));
  CKC(gmalloc(&ctx->d_flags, 4 * sizeof(int)));
  {
    std::vector<int> all(I);
    for (int i = 0; i < I; ++i) all[i] = i;
    CKC(cudaMemcpy(ctx->d_list_all, all.data(), I * sizeof(int), cudaMemcpyHostToDevice));
    // launch order of full-list block solves: with 2 CTAs per SM the first
    // num_sms CTAs take one SM each and the next ones pair up with the first
    // SMs, so the SMs at positions [I - num_sms, num_sms) keep a single CTA.
    // The subdomains with the most solve bytes (the last tile row / column,
    // ~30 % above an interior one) go there: a CTA alone on its SM streams
    // faster, and the slowest chains bound the launch.
    std::vector<int> ord(all);
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int x, int y) { return ctx->sub_jbytes[x] > ctx->sub_jbytes[y]; });
    std::vector<int> sol(ord);
    const int sms = ctx->num_sms;
    if (I > sms && I < 2 * sms) {
      const int lo = I - sms, hi = sms;   // positions whose SM keeps one CTA
      int pos = 0;
      for (int k = lo; k < hi; ++k) sol[k] = ord[pos++];   // heaviest: alone on an SM
      for (int k = 0; k < lo; ++k) sol[k] = ord[pos++];
      for (int k = hi; k < I; ++k) sol[k] = ord[pos++];
    }
    CKC(gmalloc(&ctx->d_solve_order, I * sizeof(int)));
    CKC(cudaMemcpy(ctx->d_solve_order, sol.data(), I * sizeof(int), cudaMemcpyHostToDevice));
  }
  // narrow lines (config 5): a 6-warp factor CTA, two per SM, when there
  // are enough subdomains to fill them and nearly every line fits its
  // 96-unknown shared-memory block (ocp_block_narrow.cu)
  if (I >= 2 * ctx->num_sms) {
    // (an instance whose block size is an odd multiple of 16 factors lines padded
    // to 16 with a half-width last panel: such lines get pad_ = NPS)
    const int nmax = narrow_factor_max_npb();
    const bool half = (nmax & 16) != 0;
    int fit = 0;
    for (auto& sub : ctx->subs) fit += (half ? sub.NPS : sub.pad_) <= nmax;
    ctx->bf_narrow = 10LL * fit >= 9LL * I;
    if (ctx->bf_narrow && half) {
      ctx->maxNPB = 0;
      for (auto& sub : ctx->subs) {
        if (sub.NPS <= nmax && (sub.NPS & 16) && sub.NPS >= 48) sub.pad_ = sub.NPS;
        ctx->maxNPB = std::max(ctx->maxNPB, sub.pad_);
      }
      CKC(cudaMemcpy(ctx->d_subs, ctx->subs.data(), I * sizeof(SubInfo), cudaMemcpyHostToDevice));
    }
  }
  const int bf_per_sm = ctx->bf_narrow ? narrow_factor_ctas_per_sm() : 1;
  const int bf_max_npb = ctx->bf_narrow ? narrow_factor_max_npb() : BF_SMEM_MAX_NPB;
  ctx->bf_grid = std::max(1, std::min(I, bf_per_sm * ctx->num_sms));
  if (ctx->maxNPS > block_solve_max_nps()) {
    fail(ctx, OCP_ERR_UNSUPPORTED, "local short side %d exceeds the block solve's limit %d",
         ctx->maxNPS / 2, block_solve_max_nps() / 2);
    return cleanup_fail(OCP_ERR_UNSUPPORTED);
  }
  // few subdomains wider than the shared block: K CTAs per subdomain share its
  // Schur block in global memory (k_block_factor_mc; OCP_FACTOR_MC=0 disables)
  if (ctx->maxNPB > bf_max_npb && 2 * I <= ctx->num_sms) {
    const char* e = getenv("OCP_FACTOR_MC");
    if (!(e && e[0] == '0')) {
      ctx->mc_K = std::min(32, ctx->num_sms / I);
      ctx->ms_stride = (long long)ctx->maxNPB * (ctx->maxNPB + 4);
      CKC(gmalloc(&ctx->mscratch, (size_t)I * ctx->ms_stride * sizeof(double)));
      CKC(gmalloc(&ctx->d_mcbars, (size_t)16 * I * sizeof(unsigned long long)));
      // the solves too when the lines are wider than the fast solve's 224 and
      // fit k_block_solve_mc (NPS <= 496; at most 3 units of 8 columns per CTA)
      const int units = 2 * (ctx->maxNPS / 16);
      const int ks = std::min(ctx->mc_K, units);
      if (ctx->maxNPS > 224 && ctx->maxNPS <= 496 && 3 * ks >= units) {
        ctx->mc_Ks = ks;
        CKC(gmalloc(&ctx->mc_partials, (size_t)I * 2 * ks * ctx->maxNPS * sizeof(double)));
      }
    }
  }
  if (ctx->maxNPB > bf_max_npb) {
    // rows beyond the shared block, then (short side > 112) the line's
    // Jacobian diagonals (k_block_factor)
    ctx->bs_stride = (long long)ctx->maxNPB * (ctx->maxNPB + 4) + 2LL * ctx->maxNPB;
    CKC(gmalloc(&ctx->bscratch, ctx->bf_grid * ctx->bs_stride * sizeof(double)));
  }
  CKC(gmalloc(&ctx->red_partials, RED_BLOCKS * sizeof(double)));
  CKC(gmalloc(&ctx->red_counter, sizeof(unsigned int)));
  CKC(cudaMemsetAsync(ctx->red_counter, 0, sizeof(unsigned int), ctx->stream));
  CKC(gmalloc(&ctx->arn_bar, sizeof(unsigned long long)));
  CKC(gmalloc(&ctx->arn_partials, 2 * 2048 * sizeof(double)));
  CKC(cudaMemsetAsync(ctx->arn_bar, 0, sizeof(unsigned long long), ctx->stream));
  CKC(gmalloc(&ctx->d_result, 8 * sizeof(double)));
  ctx->h_cap = 4096;
  CKC(gmalloc(&ctx->d_h, ctx->h_cap * sizeof(double)));
  CKC(cudaMallocHost(&ctx->h_norm2, I * sizeof(double)));
  // (one pinned allocation for both: cudaMallocHost / cudaFreeHost cost milliseconds)
  CKC(cudaMallocHost(&ctx->h_rpart, 2 * (size_t)I * ctx->res_chunks * sizeof(double)));
  ctx->h_rbad = reinterpret_cast<unsigned long long*>(ctx->h_rpart + (size_t)I * ctx->res_chunks);
  ctx->res_bad.assign(I, -1ll);
  CKC(cudaMallocHost(&ctx->h_status, I * sizeof(int)));
  CKC(cudaMallocHost(&ctx->h_bad, I * sizeof(long long)));
  CKC(cudaMallocHost(&ctx->h_list, I * sizeof(int)));
  CKC(cudaMallocHost(&ctx->h_alpha, I * sizeof(double)));
  CKC(cudaMallocHost(&ctx->h_small, 8192 * sizeof(double)));
  CKC(cudaMallocHost(&ctx->h_flags, 4 * sizeof(int)));
  {
    int optin = 0;
    CKC(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    {
      // (lines wider than 224 unknowns use k_block_solve_wide, which sets its own limit)
      const int fb = block_factor_smem_bytes(ctx->maxNPB),
                sb = (int)block_solve_smem_bytes(std::min(ctx->maxNPS, 224));
      if (fb + 1024 > optin || sb + 1024 > optin) {
        fail(ctx, OCP_ERR_UNSUPPORTED, "block factor needs more shared memory than the device offers");
        return cleanup_fail(OCP_ERR_UNSUPPORTED);
      }
      CKC(set_block_kernel_smem(fb, sb));
      if (ctx->bf_narrow) CKC(narrow_set_factor_smem());
    }
  }
#undef CKC
  for (auto& s : ctx->subs) {
    ctx->dof_total += s.N;
    ctx->resid_bytes_all += 48.0 * (double)s.nr * s.nc;
  }
  *out = ctx;
  return OCP_OK;
}

void ocp_ctx_destroy(ocp_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->gm_Q && ctx->stream)   // kept for the next context (or back to the memory pool)
    spare_put(ctx->gm_Q, (size_t)ctx->gm_cols * ctx->gm_n * sizeof(double), ctx->stream);
  ctx->gm_Q = nullptr;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (void* p : {(void*)ctx->d_subs, (void*)ctx->d_f, (void*)ctx->d_yd, (void*)ctx->V, (void*)ctx->R,
                  (void*)ctx->D, (void*)ctx->B, (void*)ctx->JD, (void*)ctx->d_list_all,
                  (void*)ctx->d_list, (void*)ctx->d_status, (void*)ctx->d_alpha,
                  (void*)ctx->d_bad, (void*)ctx->d_rpart, (void*)ctx->d_rbad, (void*)ctx->d_flags, (void*)ctx->mscratch, (void*)ctx->d_mcbars, (void*)ctx->mc_partials,
                  (void*)ctx->red_partials, (void*)ctx->red_counter, (void*)ctx->arn_bar, (void*)ctx->arn_partials, (void*)ctx->d_result,
                  (void*)ctx->gm_Q, (void*)ctx->gm_w, (void*)ctx->gm_dh, (void*)ctx->gm_t,
                  (void*)ctx->st_buf, (void*)ctx->st_sc, (void*)ctx->st_hist,
                  (void*)ctx->d_gbad, (void*)ctx->bscratch, (void*)ctx->d_flist, (void*)ctx->d_solve_order,
                  (void*)ctx->d_h})
    if (p) gfree(p);
  for (void* p : {(void*)ctx->h_norm2, (void*)ctx->h_rpart, (void*)ctx->h_status, (void*)ctx->h_bad, (void*)ctx->h_list,
                  (void*)ctx->h_alpha, (void*)ctx->h_small, (void*)ctx->h_flags,
                  (void*)ctx->gm_hh, (void*)ctx->st_hhist, (void*)ctx->h_flist})
    if (p) cudaFreeHost(p);
  for (auto e : ctx->gm_ev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  for (auto e : ctx->marks) if (e) cudaEventDestroy(e);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int ocp_ctx_info(const ocp_ctx* ctx, long long* info) {
  if (!ctx || !info) return OCP_ERR_ARG;
  info[0] = ctx->I;
  info[1] = ctx->pool_len;
  info[2] = ctx->fac_len;
  info[3] = ctx->maxW;
  info[4] = NB;
  info[5] = ctx->dof_total;
  info[6] = ctx->ref_len;
  return OCP_OK;
}

int ocp_subdomain_table(const ocp_ctx* ctx, int* rects) {
  if (!ctx || !rects) return OCP_ERR_ARG;
  for (int i = 0; i < ctx->I; ++i) {
    const SubInfo& s = ctx->subs[i];
    const int v[11] = {s.r0, s.r1, s.c0, s.c1, s.or0, s.or1, s.oc0, s.oc1, s.orient, s.nr, s.nc};
    std::memcpy(rects + 11 * i, v, sizeof v);
  }
  return OCP_OK;
}

int ocp_malloc(size_t bytes, void** dev) {
  ocp_ctx* ctx = nullptr;
  if (!dev) return OCP_ERR_ARG;
  CK(gmalloc(dev, std::max<size_t>(bytes, 16)));
  return OCP_OK;
}

int ocp_free(void* dev) {
  ocp_ctx* ctx = nullptr;
  if (dev) CK(gfree(dev));
  return OCP_OK;
}

int ocp_h2d(ocp_ctx* ctx, void* dev, const void* host, size_t bytes) {
  CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return OCP_OK;
}

int ocp_d2h(ocp_ctx* ctx, void* host, const void* dev, size_t bytes) {
  CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return OCP_OK;
}

int ocp_d2d(ocp_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return OCP_OK;
}

int ocp_memset0(ocp_ctx* ctx, void* dev, size_t bytes) {
  CK(cudaMemsetAsync(dev, 0, bytes, ctx->stream));
  return OCP_OK;
}

int ocp_sync(ocp_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  return OCP_OK;
}

// ---------------------------------------------------------------------------
// the RAS sweep (raspen_residual, schwarz.py:285-324)
// ---------------------------------------------------------------------------
// The batched inner Newton of every subdomain in `only` (all when only < 0),
// then - for the whole set - the refactorisation at eps_fac and f_val.
static int sweep_impl(ocp_ctx* ctx, const double* x, double* fac, double eps_fac, double eps0,
                      double gamma, double eps_min, double tol, int max_outer, double sigma,
                      int max_halvings, double* fval, int* inner_iters, int* failed_sub, int only) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  if (!ctx || !x || !fac || (only < 0 && !fval)) return fail(ctx, OCP_ERR_ARG, "null argument");
  if (only >= ctx->I) return fail(ctx, OCP_ERR_ARG, "subdomain %d out of range", only);
  const int I = ctx->I;
  cudaStream_t st = ctx->stream;
  Timer sweep_timer(ctx, CLS_SWEEP);
  enum { ACTIVE = 0, DONE = 1, FAILED = 2 };
  struct Failure {
    int code;
    std::string msg;
  };
  std::vector<int> state(I, ACTIVE), iters(I, 0);
  std::vector<double> nrm(I), thr(I), alpha(I, 1.0);
  std::vector<Failure> why(I);
  int lowest = INT_MAX;
  auto mark_fail = [&](int i, int code, const std::string& msg) {
    state[i] = FAILED;
    why[i] = {code, msg};
    lowest = std::min(lowest, i);
  };

  k_gather<<<I, 256, 0, st>>>(ctx->d_subs, ctx->d_list_all, ctx->P, x, ctx->V);
  CKL();
  double eps = eps0;
  // the first residual also produces the Jacobian diagonals at eps0
  if (int rc = launch_residual(ctx, ctx->d_list_all, I, x, ctx->V, nullptr, nullptr, eps, ctx->R, true))
    return rc;
  CK(cudaStreamSynchronize(st));
  finish_residual(ctx, nullptr, I, true);
  for (int i = 0; i < I; ++i) {
    if (only >= 0 && i != only) {   // local_correction: subdomain `only` alone
      state[i] = DONE;
      continue;
    }
    nrm[i] = std::sqrt(ctx->h_norm2[i]);
    if (!std::isfinite(nrm[i])) {
      mark_fail(i, OCP_ERR_NONFINITE_INIT, "nonfinite residual at the initial guess");
      continue;
    }
    thr[i] = std::max(tol, tol * nrm[i]);  // newton.py:148
  }

  std::vector<int> act, pend, acc, next;
  while (true) {
    act.clear();
    for (int i = 0; i < I && i < lowest; ++i) {
      if (state[i] != ACTIVE) continue;
      if (nrm[i] <= thr[i] && eps == eps_min) {  // newton.py:153
        state[i] = DONE;
      } else if (iters[i] >= max_outer) {
        char buf[128];
        snprintf(buf, sizeof buf, "no convergence within %d outer iterations", max_outer);
        mark_fail(i, OCP_ERR_LOCAL_SOLVE, buf);
      } else {
        act.push_back(i);
      }
    }
    // subdomains above a known failure cannot change the outcome
    act.erase(std::remove_if(act.begin(), act.end(), [&](int i) { return i > lowest; }), act.end());
    if (act.empty()) break;
    const int cnt = (int)act.size();
    if (int rc = upload_list(ctx, act)) return rc;
    // the Jacobian diagonals at (V, eps) came with the residual that accepted
    // the last step (or the first residual): every active subdomain was in it
    if (int rc = launch_factor(ctx, ctx->d_list, act, fac)) return rc;
    if (int rc = launch_solve(ctx, ctx->d_list, act, fac, ctx->R, -1.0, ctx->D, CLS_INNER_SOLVE)) return rc;
    CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, I * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    pend.clear();
    for (int i : act) {
      const long long b = ctx->res_bad[i];
      if (b >= 0) {
        char buf[160];
        snprintf(buf, sizeof buf, "%s@%lld", (b >> 32) ? "phi''(y)" : "phi'(y)", b & 0xffffffffLL);
        mark_fail(i, OCP_ERR_NONFINITE, buf);
      } else if (ctx->h_status[i]) {
        mark_fail(i, OCP_ERR_LOCAL_SOLVE,
                  "sparse factorization failed: singular local Jacobian (zero pivot in banded LU)");
      } else {
        pend.push_back(i);
        alpha[i] = 1.0;
      }
    }
    // relaxed backtracking (newton.py:96-112), all pending subdomains at once
    acc.clear();
    for (int h = 0; h <= max_halvings && !pend.empty(); ++h) {
      for (size_t k = 0; k < pend.size(); ++k) ctx->h_alpha[pend[k]] = alpha[pend[k]];
      CK(cudaMemcpyAsync(ctx->d_alpha, ctx->h_alpha, I * sizeof(double), cudaMemcpyHostToDevice, st));
      if (int rc = upload_list(ctx, pend)) return rc;
      if (int rc = launch_residual(ctx, ctx->d_list, (int)pend.size(), x, ctx->V, ctx->D,
                                   ctx->d_alpha, eps, nullptr)) return rc;
      CK(cudaStreamSynchronize(st));
      finish_residual(ctx, pend.data(), (int)pend.size(), false);
      next.clear();
      for (int i : pend) {
        const double trial = std::sqrt(ctx->h_norm2[i]);
        if (std::isfinite(trial) && trial <= sigma * nrm[i]) acc.push_back(i);
        else {
          alpha[i] *= 0.5;
          next.push_back(i);
        }
      }
      pend.swap(next);
    }
    for (int i : pend) {
      char buf[160];
      snprintf(buf, sizeof buf, "no admissible step within %d halvings (residual %s)", max_halvings,
               fmt_e3(nrm[i]).c_str());
      mark_fail(i, OCP_ERR_LOCAL_SOLVE, buf);
    }
    const double eps_next = (eps_min > gamma * eps) ? eps_min : gamma * eps;  // max(gamma*eps, eps_min)
    if (!acc.empty()) {
      std::sort(acc.begin(), acc.end());
      for (int i : acc) ctx->h_alpha[i] = alpha[i];
      CK(cudaMemcpyAsync(ctx->d_alpha, ctx->h_alpha, I * sizeof(double), cudaMemcpyHostToDevice, st));
      if (int rc = upload_list(ctx, acc)) return rc;
      const int na = (int)acc.size();
      k_update<<<na, 256, 0, st>>>(ctx->d_subs, ctx->d_list, ctx->V, ctx->D, ctx->d_alpha);
      CKL();
      if (int rc = launch_residual(ctx, ctx->d_list, na, x, ctx->V, nullptr, nullptr, eps_next, ctx->R,
                                   true))
        return rc;
      CK(cudaStreamSynchronize(st));
      finish_residual(ctx, acc.data(), na, true);
      for (int i : acc) {
        nrm[i] = std::sqrt(ctx->h_norm2[i]);
        iters[i] += 1;
        ctx->stat_dof += (double)ctx->sub_dofs[i];
      }
    }
    eps = eps_next;
  }
  if (inner_iters) for (int i = 0; i < I; ++i) inner_iters[i] = iters[i];
  if (lowest != INT_MAX) {
    if (failed_sub) *failed_sub = lowest;
    return fail(ctx, why[lowest].code, "%s", why[lowest].msg.c_str());
  }
  if (failed_sub) *failed_sub = -1;
  if (only >= 0) return OCP_OK;
  // refactorisation at the converged values, at eps (schwarz.py:305-315)
  std::vector<int> all(I);
  for (int i = 0; i < I; ++i) all[i] = i;
  k_jacdiag<<<I, 256, 0, st>>>(ctx->d_subs, ctx->d_list_all, ctx->P, ctx->V, eps_fac, ctx->JD,
                               ctx->d_bad);
  CKL();
  if (int rc = launch_factor(ctx, ctx->d_list_all, all, fac)) return rc;
  {
    dim3 grid(I, 8);
    k_scatter_fval<<<grid, 256, 0, st>>>(ctx->d_subs, ctx->P, ctx->V, x, fval);
    CKL();
  }
  CK(cudaMemcpyAsync(ctx->h_bad, ctx->d_bad, I * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, I * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int i = 0; i < I; ++i) {
    if (ctx->h_bad[i] >= 0) {
      const long long b = ctx->h_bad[i];
      if (failed_sub) *failed_sub = i;
      return fail(ctx, OCP_ERR_NONFINITE, "%s@%lld", (b >> 32) ? "phi''(y)" : "phi'(y)",
                  b & 0xffffffffLL);
    }
    if (ctx->h_status[i]) {
      if (failed_sub) *failed_sub = i;
      return fail(ctx, OCP_ERR_LOCAL_SOLVE,
                  "singular local Jacobian: zero pivot in banded LU");
    }
  }
  return OCP_OK;
}

int ocp_raspen_residual(ocp_ctx* ctx, const double* x, double* fac, double eps0, double gamma,
                        double eps_min, double tol, int max_outer, double sigma, int max_halvings,
                        double* fval, int* inner_iters, int* failed_sub) {
  return sweep_impl(ctx, x, fac, eps_min, eps0, gamma, eps_min, tol, max_outer, sigma, max_halvings,
                    fval, inner_iters, failed_sub, -1);
}

int ocp_raspen_residual_at(ocp_ctx* ctx, const double* x, double* fac, double eps, double eps0,
                           double gamma, double eps_min, double tol, int max_outer, double sigma,
                           int max_halvings, double* fval, int* inner_iters, int* failed_sub) {
  return sweep_impl(ctx, x, fac, eps, eps0, gamma, eps_min, tol, max_outer, sigma, max_halvings,
                    fval, inner_iters, failed_sub, -1);
}

int ocp_local_correction(ocp_ctx* ctx, const double* x, double* fac, int sub, double eps0,
                         double gamma, double eps_min, double tol, int max_outer, double sigma,
                         int max_halvings, int* inner_iters, int* failed_sub) {
  if (sub < 0) return fail(ctx, OCP_ERR_ARG, "subdomain %d out of range", sub);
  return sweep_impl(ctx, x, fac, eps_min, eps0, gamma, eps_min, tol, max_outer, sigma,
                    max_halvings, nullptr, inner_iters, failed_sub, sub);
}

int ocp_raspen_jvp(ocp_ctx* ctx, const double* fac, const double* d, double* out) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  if (!ctx || !fac || !d || !out) return fail(ctx, OCP_ERR_ARG, "null argument");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  Timer tj(ctx, CLS_JVP);
  // one fused launch: rhs from d, solve, out[own] = -(d + x)
  double bytes = 0;
  for (int i = 0; i < I; ++i) bytes += ctx->sub_jbytes[i];
  Timer t(ctx, CLS_SOLVE, 0, bytes);
  CK(solve_dispatch(ctx, 2, I, ctx->d_solve_order, fac, nullptr, 1.0, ctx->B, d, out));
  ++ctx->launches;
  return OCP_OK;
}

int ocp_local_values(ocp_ctx* ctx, double* values) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  k_band_to_ref<<<ctx->I, 256, 0, ctx->stream>>>(ctx->d_subs, ctx->V, values);
  CKL();
  return OCP_OK;
}

int ocp_local_residual(ocp_ctx* ctx, const double* x, const double* v_ref, double eps, double* r_ref) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  k_ref_to_band<<<I, 256, 0, st>>>(ctx->d_subs, v_ref, ctx->B);
  CKL();
  if (int rc = launch_residual(ctx, ctx->d_list_all, I, x, ctx->B, nullptr, nullptr, eps, ctx->D)) return rc;
  k_band_to_ref<<<I, 256, 0, st>>>(ctx->d_subs, ctx->D, r_ref);
  CKL();
  CK(cudaStreamSynchronize(st));
  return OCP_OK;
}

int ocp_local_residual_trial(ocp_ctx* ctx, const double* x, const double* v_ref, const double* d_ref,
                             const double* alpha_host, double eps, double* norm2_host) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  if (!alpha_host || !norm2_host) return fail(ctx, OCP_ERR_ARG, "null argument");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  k_ref_to_band<<<I, 256, 0, st>>>(ctx->d_subs, v_ref, ctx->B);
  CKL();
  k_ref_to_band<<<I, 256, 0, st>>>(ctx->d_subs, d_ref, ctx->D);
  CKL();
  for (int i = 0; i < I; ++i) ctx->h_alpha[i] = alpha_host[i];
  CK(cudaMemcpyAsync(ctx->d_alpha, ctx->h_alpha, I * sizeof(double), cudaMemcpyHostToDevice, st));
  if (int rc = launch_residual(ctx, ctx->d_list_all, I, x, ctx->B, ctx->D, ctx->d_alpha, eps, nullptr))
    return rc;
  CK(cudaStreamSynchronize(st));
  finish_residual(ctx, nullptr, I, false);
  for (int i = 0; i < I; ++i) norm2_host[i] = ctx->h_norm2[i];
  return OCP_OK;
}

int ocp_local_direction(ocp_ctx* ctx, const double* x, const double* v_ref, double eps, double* d_ref) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  double* fac = nullptr;
  CK(gmalloc(&fac, ctx->fac_len * sizeof(double)));
  k_ref_to_band<<<I, 256, 0, st>>>(ctx->d_subs, v_ref, ctx->B);
  CKL();
  if (int rc = launch_residual(ctx, ctx->d_list_all, I, x, ctx->B, nullptr, nullptr, eps, ctx->D)) return rc;
  k_jacdiag<<<I, 256, 0, st>>>(ctx->d_subs, ctx->d_list_all, ctx->P, ctx->B, eps, ctx->JD, ctx->d_bad);
  CKL();
  std::vector<int> all(I);
  for (int i = 0; i < I; ++i) all[i] = i;
  int rc = launch_factor(ctx, ctx->d_list_all, all, fac);
  if (!rc) rc = launch_solve(ctx, ctx->d_list_all, all, fac, ctx->D, -1.0, ctx->D, CLS_INNER_SOLVE);
  if (!rc) {
    k_band_to_ref<<<I, 256, 0, st>>>(ctx->d_subs, ctx->D, d_ref);
    CKL();
  }
  cudaStreamSynchronize(st);
  gfree(fac);
  if (rc) return rc;
  CK(cudaMemcpy(ctx->h_status, ctx->d_status, I * sizeof(int), cudaMemcpyDeviceToHost));
  for (int i = 0; i < I; ++i)
    if (ctx->h_status[i]) return fail(ctx, OCP_ERR_LOCAL_SOLVE, "zero pivot in subdomain %d", i);
  return OCP_OK;
}

// ---------------------------------------------------------------------------
// vector kernels
// ---------------------------------------------------------------------------
int ocp_vec_dot(ocp_ctx* ctx, long long n, const double* x, const double* y, double* out) {
  k_dot<<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(n, x, y, ctx->red_partials, ctx->red_counter,
                                                     ctx->d_result, 0);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_small, ctx->d_result, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *out = ctx->h_small[0];
  return OCP_OK;
}

int ocp_vec_nrm2(ocp_ctx* ctx, long long n, const double* x, double* out) {
  k_dot<<<RED_BLOCKS, RED_THREADS, 0, ctx->stream>>>(n, x, x, ctx->red_partials, ctx->red_counter,
                                                     ctx->d_result, 1);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_small, ctx->d_result, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *out = ctx->h_small[0];
  return OCP_OK;
}

int ocp_vec_add_scaled(ocp_ctx* ctx, long long n, const double* x, double alpha, const double* d,
                       double* out) {
  k_add_scaled<<<ew_grid(n), 256, 0, ctx->stream>>>(n, x, alpha, d, out);
  CKL();
  return OCP_OK;
}

int ocp_vec_scale(ocp_ctx* ctx, long long n, double a, const double* x, double* out) {
  k_scale<<<ew_grid(n), 256, 0, ctx->stream>>>(n, a, x, out);
  CKL();
  return OCP_OK;
}

int ocp_vec_div(ocp_ctx* ctx, long long n, const double* x, double s, double* out) {
  k_div<<<ew_grid(n), 256, 0, ctx->stream>>>(n, x, s, out);
  CKL();
  return OCP_OK;
}

static int run_flags(ocp_ctx* ctx, long long n, const double* x, const double* y, int* fl) {
  ctx->h_flags[0] = 1;
  ctx->h_flags[1] = 1;
  CK(cudaMemcpyAsync(ctx->d_flags, ctx->h_flags, 2 * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  k_flags<<<ew_grid(n), 256, 0, ctx->stream>>>(n, x, y, ctx->d_flags);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  fl[0] = ctx->h_flags[0];
  fl[1] = ctx->h_flags[1];
  return OCP_OK;
}

int ocp_vec_equal(ocp_ctx* ctx, long long n, const double* x, const double* y, int* equal) {
  int fl[2];
  if (int rc = run_flags(ctx, n, x, y, fl)) return rc;
  *equal = fl[0];
  return OCP_OK;
}

int ocp_vec_all_finite(ocp_ctx* ctx, long long n, const double* x, int* finite) {
  int fl[2];
  if (int rc = run_flags(ctx, n, x, nullptr, fl)) return rc;
  *finite = fl[1];
  return OCP_OK;
}

int ocp_mgs(ocp_ctx* ctx, long long n, const double* Q, long long ldq, int j, double* w, double* h_host) {
  if (j + 2 > ctx->h_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(gfree(ctx->d_h));
    ctx->h_cap = 2 * (j + 2);
    CK(gmalloc(&ctx->d_h, ctx->h_cap * sizeof(double)));
  }
  Timer t(ctx, CLS_MGS);
  cudaStream_t st = ctx->stream;
  for (int i = 0; i <= j; ++i) {
    k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, i > 0 ? Q + (long long)(i - 1) * ldq : nullptr,
                                                   i > 0 ? ctx->d_h + i - 1 : nullptr,
                                                   Q + (long long)i * ldq, ctx->red_partials,
                                                   ctx->red_counter, ctx->d_h + i);
    CKL();
  }
  k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, Q + (long long)j * ldq, ctx->d_h + j, nullptr,
                                                 ctx->red_partials, ctx->red_counter, ctx->d_h + j + 1);
  CKL();
  CK(cudaMemcpyAsync(h_host, ctx->d_h, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OCP_OK;
}

int ocp_arnoldi(ocp_ctx* ctx, long long n, double* Q, long long ldq, int j, const double* w_in,
                double* h_host) {
  if (j + 2 > ctx->h_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(gfree(ctx->d_h));
    ctx->h_cap = 2 * (j + 2);
    CK(gmalloc(&ctx->d_h, ctx->h_cap * sizeof(double)));
  }
  cudaStream_t st = ctx->stream;
  {
    Timer t(ctx, CLS_MGS);
    cudaError_t e = launch_arnoldi(st, ctx->num_sms, n, Q, ldq, j, w_in, ctx->arn_partials, ctx->d_h,
                                   ctx->arn_bar, &ctx->arn_epoch);
    if (e == cudaSuccess) {
      ++ctx->launches;
    } else if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      double* w = Q + (long long)(j + 1) * ldq;  // work in the next column
      CK(cudaMemcpyAsync(w, w_in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      for (int i = 0; i <= j; ++i) {
        k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(
            n, w, i > 0 ? Q + (long long)(i - 1) * ldq : nullptr, i > 0 ? ctx->d_h + i - 1 : nullptr,
            Q + (long long)i * ldq, ctx->red_partials, ctx->red_counter, ctx->d_h + i);
        CKL();
      }
      k_mgs_pass<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, w, Q + (long long)j * ldq, ctx->d_h + j,
                                                     nullptr, ctx->red_partials, ctx->red_counter,
                                                     ctx->d_h + j + 1);
      CKL();
      CK(cudaMemcpyAsync(ctx->h_small, ctx->d_h + j + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      k_div<<<ew_grid(n), 256, 0, st>>>(n, w, ctx->h_small[0], w);
      CKL();
    } else {
      return fail(ctx, OCP_ERR_CUDA, "cooperative Arnoldi launch: %s", cudaGetErrorString(e));
    }
  }
  CK(cudaMemcpyAsync(h_host, ctx->d_h, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OCP_OK;
}

// Linear-RAS Newton-Krylov (newton-ras-eps): whole-grid residual / Jacobian
// and the one-level RAS preconditioner built from the batched banded LU.
int ocp_global_residual(ocp_ctx* ctx, const double* x, double eps, double* r) {
  if (!ctx || !x || !r) return fail(ctx, OCP_ERR_ARG, "null argument");
  k_global_residual<<<ew_grid(ctx->N), 256, 0, ctx->stream>>>(ctx->P, x, ctx->d_f, ctx->d_yd, eps, r);
  CKL();
  return OCP_OK;
}

int ocp_global_jacobian(ocp_ctx* ctx, const double* x, double eps, double* jd) {
  if (!ctx || !x || !jd) return fail(ctx, OCP_ERR_ARG, "null argument");
  cudaStream_t st = ctx->stream;
  if (!ctx->d_gbad) CK(gmalloc(&ctx->d_gbad, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(ctx->d_gbad, 0xff, sizeof(unsigned long long), st));
  k_global_jacdiag<<<ew_grid(ctx->N), 256, 0, st>>>(ctx->P, x, eps, reinterpret_cast<double4*>(jd),
                                                     ctx->d_gbad);
  CKL();
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->d_gbad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad != ~0ull)
    return fail(ctx, OCP_ERR_NONFINITE, "%s@%lld", (bad >> 32) ? "phi''(y)" : "phi'(y)",
                (long long)(bad & 0xffffffffull));
  return OCP_OK;
}

int ocp_global_jvp(ocp_ctx* ctx, const double* jd, const double* d, double* out) {
  if (!ctx || !jd || !d || !out) return fail(ctx, OCP_ERR_ARG, "null argument");
  k_global_jvp<<<ew_grid(ctx->N), 256, 0, ctx->stream>>>(ctx->P, reinterpret_cast<const double4*>(jd),
                                                          d, out);
  CKL();
  return OCP_OK;
}

// local Jacobians at x restricted to every subdomain, factored into fac
// (ras_preconditioner, schwarz.py:221-232)
int ocp_ras_factor(ocp_ctx* ctx, const double* x, double eps, double* fac, int* failed_sub) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  if (!ctx || !x || !fac) return fail(ctx, OCP_ERR_ARG, "null argument");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  if (failed_sub) *failed_sub = -1;
  k_gather<<<I, 256, 0, st>>>(ctx->d_subs, ctx->d_list_all, ctx->P, x, ctx->B);
  CKL();
  k_jacdiag<<<I, 256, 0, st>>>(ctx->d_subs, ctx->d_list_all, ctx->P, ctx->B, eps, ctx->JD, ctx->d_bad);
  CKL();
  std::vector<int> all(I);
  for (int i = 0; i < I; ++i) all[i] = i;
  if (int rc = launch_factor(ctx, ctx->d_list_all, all, fac)) return rc;
  CK(cudaMemcpyAsync(ctx->h_bad, ctx->d_bad, I * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, I * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int i = 0; i < I; ++i) {
    if (ctx->h_bad[i] >= 0) {
      const long long b = ctx->h_bad[i];
      if (failed_sub) *failed_sub = i;
      return fail(ctx, OCP_ERR_NONFINITE, "%s@%lld", (b >> 32) ? "phi''(y)" : "phi'(y)",
                  b & 0xffffffffLL);
    }
    if (ctx->h_status[i]) {
      if (failed_sub) *failed_sub = i;
      return fail(ctx, OCP_ERR_LOCAL_SOLVE,
                  "singular local block: zero pivot in banded LU");
    }
  }
  return OCP_OK;
}

// out = sum_i P~_i J_i^{-1} R_i v  (the apply closure, schwarz.py:234-239)
int ocp_ras_apply(ocp_ctx* ctx, const double* fac, const double* v, double* out) {
  if (ctx && ctx->I == 0) return fail(ctx, OCP_ERR_ARG, "grid-only context has no subdomains");
  if (!ctx || !fac || !v || !out) return fail(ctx, OCP_ERR_ARG, "null argument");
  cudaStream_t st = ctx->stream;
  const int I = ctx->I;
  // one fused launch: rhs gathered per line, out[own] = x[own]
  double bytes = 0;
  for (int i = 0; i < I; ++i) bytes += ctx->sub_jbytes[i];
  Timer t(ctx, CLS_SOLVE, 0, bytes);
  CK(solve_dispatch(ctx, 3, I, ctx->d_solve_order, fac, nullptr, 1.0, ctx->B, v, out));
  ++ctx->launches;
  return OCP_OK;
}

// ---- state equation of the manufactured problems (system.py:181-197) ----
int ocp_state_residual(ocp_ctx* ctx, const double* y, const double* rhs, double* out) {
  if (!ctx || !y || !rhs || !out) return fail(ctx, OCP_ERR_ARG, "null argument");
  k_state_residual<<<ew_grid(ctx->N), 256, 0, ctx->stream>>>(ctx->P, y, rhs, out);
  CKL();
  return OCP_OK;
}

int ocp_manufacture_yd(ocp_ctx* ctx, const double* ybar, const double* pbar, double* yd) {
  if (!ctx || !ybar || !pbar || !yd) return fail(ctx, OCP_ERR_ARG, "null argument");
  k_manufacture_yd<<<ew_grid(ctx->N), 256, 0, ctx->stream>>>(ctx->P, ybar, pbar, yd);
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  return OCP_OK;
}

// (A + diag(phi'(y))) x = b by conjugate gradients from x = 0 until
// ||r|| <= rel_tol ||b|| (the matrix is SPD for the phi families used:
// phi' >= 0).  Scalars stay on the device; the host polls the r.r history
// every CG_POLL iterations (the few extra iterations only tighten x).
int ocp_state_cg(ocp_ctx* ctx, const double* y, const double* b, double rel_tol, int max_iters,
                 double* x, int* iters_out, double* resid_out, int* conv_out) {
  if (!ctx || !y || !b || !x || max_iters < 1) return fail(ctx, OCP_ERR_ARG, "bad argument");
  constexpr int CG_POLL = 16;
  cudaStream_t st = ctx->stream;
  const long long N = ctx->N;
  if (!ctx->st_buf) {
    CK(gmalloc(&ctx->st_buf, 4 * (size_t)N * sizeof(double)));
    CK(gmalloc(&ctx->st_sc, 8 * sizeof(double)));
  }
  const int hcap = max_iters + CG_POLL;
  if (ctx->st_hcap < hcap) {
    cudaStreamSynchronize(st);
    if (ctx->st_hist) gfree(ctx->st_hist);
    if (ctx->st_hhist) cudaFreeHost(ctx->st_hhist);
    CK(gmalloc(&ctx->st_hist, hcap * sizeof(double)));
    CK(cudaMallocHost(&ctx->st_hhist, hcap * sizeof(double)));
    ctx->st_hcap = hcap;
  }
  if (!ctx->d_gbad) CK(gmalloc(&ctx->d_gbad, sizeof(unsigned long long)));
  double *dg = ctx->st_buf, *r = dg + N, *p = r + N, *Ap = p + N;
  CK(cudaMemsetAsync(ctx->d_gbad, 0xff, sizeof(unsigned long long), st));
  k_state_diag<<<ew_grid(N), 256, 0, st>>>(ctx->P, y, dg, ctx->d_gbad);
  CKL();
  CK(cudaMemsetAsync(x, 0, N * sizeof(double), st));
  CK(cudaMemcpyAsync(r, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(p, b, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  k_dot<<<RED_BLOCKS, RED_THREADS, 0, st>>>(N, b, b, ctx->red_partials, ctx->red_counter,
                                            ctx->st_sc, 0);
  CKL();
  unsigned long long bad = 0;
  double bb = 0.0;
  CK(cudaMemcpyAsync(&bad, ctx->d_gbad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&bb, ctx->st_sc, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad != ~0ull) return fail(ctx, OCP_ERR_NONFINITE, "phi'(y)@%lld", (long long)bad);
  const double thr2 = rel_tol * rel_tol * bb;
  *iters_out = 0; *resid_out = std::sqrt(bb); *conv_out = 1;
  if (bb == 0.0) return OCP_OK;
  CK(cudaMemcpyAsync(ctx->st_sc + 4, &thr2, sizeof(double), cudaMemcpyHostToDevice, st));
  int it = 0;
  while (it < max_iters) {
    const int it0 = it;
    for (int q = 0; q < CG_POLL && it < max_iters; ++q, ++it) {
      k_cg_ap<<<RED_BLOCKS, RED_THREADS, 0, st>>>(ctx->P, dg, p, Ap, ctx->red_partials,
                                                  ctx->red_counter, ctx->st_sc);
      k_cg_xr<<<RED_BLOCKS, RED_THREADS, 0, st>>>(N, p, Ap, x, r, ctx->red_partials,
                                                  ctx->red_counter, ctx->st_sc, ctx->st_hist, it);
      k_cg_p<<<ew_grid(N), 256, 0, st>>>(N, r, p, ctx->st_sc);
      ctx->launches += 3;
    }
    CKL();
    CK(cudaMemcpyAsync(ctx->st_hhist + it0, ctx->st_hist + it0, (it - it0) * sizeof(double),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int k = it0; k < it; ++k) {
      const double rr = ctx->st_hhist[k];
      if (!std::isfinite(rr)) return fail(ctx, OCP_ERR_NONFINITE, "CG residual@%d", k);
      if (rr <= thr2) {   // the kernels froze x at this iterate
        *iters_out = k + 1; *resid_out = std::sqrt(rr);
        return OCP_OK;
      }
    }
  }
  *iters_out = it; *resid_out = std::sqrt(ctx->st_hhist[it - 1]); *conv_out = 0;
  return OCP_OK;
}

// GMRES, the whole solve in native code (krylov.py:44-151 with x0 = None,
// restart = None).  kind 0: the RASPEN Jacobian action from stored factors,
// no preconditioner; kind 1: J(x) from its diagonals, left-preconditioned by
// one-level RAS (w = M J q_j, threshold on ||M b||).
static int gmres_impl(ocp_ctx* ctx, int kind, const double* fac, const double* jd, const double* b,
                      double rel_tol, double abs_tol, int max_iters, double* x, int* iters_out,
                      double* resid_out, int* conv_out, double* history) {
  if (!ctx || !fac || !b || !x || max_iters < 1 || (kind == 1 && !jd))
    return fail(ctx, OCP_ERR_ARG, "bad argument");
  cudaStream_t st = ctx->stream;
  const long long n = 2 * ctx->N;
  if (kind == 1 && !ctx->gm_t && gmalloc(&ctx->gm_t, (size_t)n * sizeof(double)) != cudaSuccess)
    return fail(ctx, OCP_ERR_CUDA, "GMRES work vector allocation failed");
  const double* r0 = b;
  if (kind == 1) {   // mb = M b (krylov.py:55-60)
    if (int rc = ocp_ras_apply(ctx, fac, b, ctx->gm_t)) return rc;
    r0 = ctx->gm_t;
  }
  double bnorm = 0.0;
  if (int rc = ocp_vec_nrm2(ctx, n, r0, &bnorm)) return rc;
  const double threshold = std::max(rel_tol * bnorm, abs_tol);   // krylov.py:58
  const double beta = bnorm;                                       // r = M b
  int hist_len = 0;
  history[hist_len++] = beta;
  if (!std::isfinite(beta)) return fail(ctx, OCP_ERR_GMRES_BREAKDOWN, "nonfinite initial residual");
  CK(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  if (beta <= threshold) {
    *iters_out = 0; *resid_out = beta; *conv_out = 1;
    CK(cudaStreamSynchronize(st));
    return OCP_OK;
  }
  // basis Q: the reference grows an (n, cap+1) array by doubling
  // (krylov.py:89-107); here one grow-only device buffer is kept by the
  // context (doubling too), so repeated solves do not reallocate
  if (ctx->gm_Q && ctx->gm_n != n) {   // a basis for another vector length
    cudaFreeAsync(ctx->gm_Q, st);
    ctx->gm_Q = nullptr;
    ctx->gm_cols = 0;
  }
  if (!ctx->gm_Q) {
    size_t bytes = 0;
    if (double* q = spare_take((size_t)(std::min(32, max_iters) + 2) * n * sizeof(double), &bytes)) {
      ctx->gm_Q = q;
      ctx->gm_cols = (long long)(bytes / ((size_t)n * sizeof(double)));
    }
  }
  ctx->gm_n = n;
  auto ensure = [&](long long cols) -> bool {
    if (cols <= ctx->gm_cols) return true;
    long long ncols = std::max(cols, 2 * ctx->gm_cols);
    double* Q2 = nullptr;
    if (cudaMallocAsync(&Q2, (size_t)ncols * n * sizeof(double), st) != cudaSuccess) return false;
    if (ctx->gm_Q) cudaFreeAsync(ctx->gm_Q, st);
    ctx->gm_Q = Q2;
    ctx->gm_cols = ncols;
    return true;
  };
  if (!ctx->gm_w && gmalloc(&ctx->gm_w, (size_t)n * sizeof(double)) != cudaSuccess)
    return fail(ctx, OCP_ERR_CUDA, "GMRES work vector allocation failed");
  // Arnoldi coefficient slots: step j writes slot j&1 on the device, copies it
  // to pinned host memory and records gm_ev[j&1]
  if (ctx->gm_hcap < max_iters + 2) {
    cudaStreamSynchronize(st);
    if (ctx->gm_dh) gfree(ctx->gm_dh);
    if (ctx->gm_hh) cudaFreeHost(ctx->gm_hh);
    ctx->gm_dh = nullptr; ctx->gm_hh = nullptr; ctx->gm_hcap = 0;
    if (gmalloc(&ctx->gm_dh, 2 * (size_t)(max_iters + 2) * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&ctx->gm_hh, 2 * (size_t)(max_iters + 2) * sizeof(double)) != cudaSuccess)
      return fail(ctx, OCP_ERR_CUDA, "GMRES coefficient buffers");
    ctx->gm_hcap = max_iters + 2;
  }
  for (auto& e : ctx->gm_ev)
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return fail(ctx, OCP_ERR_CUDA, "GMRES events");
  const int hs = ctx->gm_hcap;
  if (!ensure(std::min(32, max_iters) + 2)) return fail(ctx, OCP_ERR_CUDA, "GMRES basis allocation failed");
  double* Q = ctx->gm_Q;
  double* w = ctx->gm_w;
  auto cleanup = [&]() {};
  k_div<<<ew_grid(n), 256, 0, st>>>(n, r0, beta, Q);   // q0 = r0 / beta
  ++ctx->launches;
  // One Arnoldi step (JVP + MGS) is always queued ahead of the host's Givens
  // update: step j+1 is enqueued before step j's coefficients are inspected,
  // so the device never idles on the host round trip.  When step j converges
  // the speculative step j+1 is discarded (it only wrote basis column j+2 and
  // slot (j+1)&1); decisions and results are those of the sequential loop.
  bool pipelined = true;
  auto enqueue = [&](int jj) -> int {
    if (jj + 2 > ctx->gm_cols) {   // grow, keeping the first jj+1 columns (stream-ordered copy)
      double* Q2 = nullptr;
      const long long ncols = std::max<long long>(jj + 2, 2 * ctx->gm_cols);
      if (cudaMallocAsync(&Q2, (size_t)ncols * n * sizeof(double), st) != cudaSuccess)
        return fail(ctx, OCP_ERR_CUDA, "GMRES basis growth failed");
      cudaMemcpyAsync(Q2, Q, (size_t)(jj + 1) * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      cudaFreeAsync(ctx->gm_Q, st);   // stream-ordered: after the copy and every queued step
      ctx->gm_Q = Q = Q2;
      ctx->gm_cols = ncols;
    }
    if (kind == 0) {
      if (int rc = ocp_raspen_jvp(ctx, fac, Q + (long long)jj * n, w)) return rc;
    } else {
      if (int rc = ocp_global_jvp(ctx, jd, Q + (long long)jj * n, ctx->gm_t)) return rc;
      if (int rc = ocp_ras_apply(ctx, fac, ctx->gm_t, w)) return rc;
    }
    double* dh = ctx->gm_dh + (jj & 1) * hs;
    if (pipelined) {
      Timer t(ctx, CLS_MGS);
      cudaError_t e = launch_arnoldi(st, ctx->num_sms, n, Q, n, jj, w, ctx->arn_partials, dh,
                                     ctx->arn_bar, &ctx->arn_epoch);
      if (e == cudaSuccess) {
        ++ctx->launches;
      } else if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        pipelined = false;
      } else {
        return fail(ctx, OCP_ERR_CUDA, "cooperative Arnoldi launch: %s", cudaGetErrorString(e));
      }
    }
    if (!pipelined) {   // per-pass kernels (vectors too large for the cooperative kernel)
      if (int rc = ocp_arnoldi(ctx, n, Q, n, jj, w, ctx->gm_hh + (jj & 1) * hs)) return rc;
    } else {
      CK(cudaMemcpyAsync(ctx->gm_hh + (jj & 1) * hs, dh, (jj + 2) * sizeof(double),
                         cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(ctx->gm_ev[jj & 1], st));
    return OCP_OK;
  };
  std::vector<double> cs, sn, g(max_iters + 1, 0.0), h(max_iters + 2);
  std::vector<std::vector<double>> cols;
  g[0] = beta;
  double residual = beta;
  bool converged = false;
  int j = 0;
  if (int rc = enqueue(0)) return rc;
  for (j = 0; j < max_iters; ++j) {
    if (j + 1 < max_iters && pipelined)
      if (int rc = enqueue(j + 1)) { cleanup(); return rc; }
    CK(cudaEventSynchronize(ctx->gm_ev[j & 1]));
    std::copy(ctx->gm_hh + (j & 1) * hs, ctx->gm_hh + (j & 1) * hs + j + 2, h.begin());
    for (int i = 0; i <= j + 1; ++i)
      if (!std::isfinite(h[i])) {
        cleanup();
        cudaStreamSynchronize(st);
        return fail(ctx, OCP_ERR_GMRES_BREAKDOWN, "nonfinite Arnoldi entries at iteration %d", j + 1);
      }
    double hmax = 0.0;
    for (int i = 0; i <= j; ++i) hmax = std::max(hmax, std::fabs(h[i]));
    const bool happy = h[j + 1] <= 1e-14 * std::max(1.0, hmax);   // krylov.py:120
    for (int i = 0; i < j; ++i) {                                   // krylov.py:124-127
      const double hi = cs[i] * h[i] + sn[i] * h[i + 1];
      h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
      h[i] = hi;
    }
    const double rad = std::hypot(h[j], h[j + 1]);
    double c = 1.0, sv = 0.0;
    if (rad != 0.0) { c = h[j] / rad; sv = h[j + 1] / rad; }
    cs.push_back(c);
    sn.push_back(sv);
    h[j] = rad;
    g[j + 1] = -sv * g[j];
    g[j] = c * g[j];
    cols.emplace_back(h.begin(), h.begin() + j + 1);
    residual = std::fabs(g[j + 1]);
    history[hist_len++] = residual;
    if (residual <= threshold || happy) {
      converged = true;
      break;
    }
    if (!pipelined && j + 1 < max_iters)
      if (int rc = enqueue(j + 1)) { cleanup(); return rc; }
  }
  const int steps = std::min(j + 1, max_iters);
  // back substitution (krylov.py:145-150)
  std::vector<double> y(steps, 0.0);
  for (int i = steps - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int k = i + 1; k < steps; ++k) dot += cols[k][i] * y[k];
    y[i] = (g[i] - dot) / cols[i][i];
  }
  int rc = ocp_gemv_add(ctx, n, Q, n, steps, y.data(), x, x);
  cleanup();
  if (rc) return rc;
  *iters_out = steps;
  *resid_out = residual;
  *conv_out = converged ? 1 : 0;
  return OCP_OK;
}

int ocp_raspen_gmres(ocp_ctx* ctx, const double* fac, const double* b, double rel_tol,
                     double abs_tol, int max_iters, double* x, int* iters_out, double* resid_out,
                     int* conv_out, double* history) {
  return gmres_impl(ctx, 0, fac, nullptr, b, rel_tol, abs_tol, max_iters, x, iters_out, resid_out,
                    conv_out, history);
}

int ocp_ras_gmres(ocp_ctx* ctx, const double* jd, const double* fac, const double* b,
                  double rel_tol, double abs_tol, int max_iters, double* x, int* iters_out,
                  double* resid_out, int* conv_out, double* history) {
  return gmres_impl(ctx, 1, fac, jd, b, rel_tol, abs_tol, max_iters, x, iters_out, resid_out,
                    conv_out, history);
}

int ocp_gemv_add(ocp_ctx* ctx, long long n, const double* Q, long long ldq, int k, const double* y_host,
                 const double* x, double* out) {
  if (k + 2 > ctx->h_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(gfree(ctx->d_h));
    ctx->h_cap = 2 * (k + 2);
    CK(gmalloc(&ctx->d_h, ctx->h_cap * sizeof(double)));
  }
  CK(cudaMemcpyAsync(ctx->d_h, y_host, k * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  k_gemv_add<<<ew_grid(n), 256, 0, ctx->stream>>>(n, Q, ldq, k, ctx->d_h, x, out);
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  return OCP_OK;
}

int ocp_recover_control(ocp_ctx* ctx, long long n, const double* p, double eps, double* u) {
  k_recover_control<<<ew_grid(n), 256, 0, ctx->stream>>>(n, ctx->P, p, eps, u);
  CKL();
  return OCP_OK;
}

int ocp_set_profiling(ocp_ctx* ctx, int on) {
  if (!ctx) return OCP_ERR_ARG;
  ctx->prof = on != 0;
  return OCP_OK;
}

int ocp_stats(ocp_ctx* ctx, double* stats, int len) {
  if (!ctx || !stats) return OCP_ERR_ARG;
  drain_events(ctx);
  double v[15] = {(double)ctx->launches, ctx->stat_ms[CLS_FACTOR], ctx->stat_cnt[CLS_FACTOR],
                  ctx->stat_ms[CLS_SOLVE], ctx->stat_cnt[CLS_SOLVE], ctx->stat_flops,
                  ctx->stat_bytes, ctx->stat_ms[CLS_SWEEP], ctx->stat_dof, ctx->stat_ms[CLS_JVP],
                  ctx->stat_ms[CLS_INNER_SOLVE], ctx->stat_ms[CLS_MGS], ctx->stat_ms[CLS_RESID],
                  ctx->stat_cnt[CLS_RESID], ctx->stat_rbytes};
  for (int i = 0; i < len && i < 15; ++i) stats[i] = v[i];
  return OCP_OK;
}

int ocp_reset_stats(ocp_ctx* ctx) {
  if (!ctx) return OCP_ERR_ARG;
  drain_events(ctx);
  ctx->launches = 0;
  for (int i = 0; i < NCLS; ++i) ctx->stat_ms[i] = ctx->stat_cnt[i] = 0;
  ctx->stat_flops = ctx->stat_bytes = ctx->stat_dof = ctx->stat_rbytes = 0;
  return OCP_OK;
}

#ifdef OCP_PHASE_TIMING
int ocp_debug_subt(long long* out, int n) {
  ocp::read_subt(out, n);
  return 0;
}
int ocp_debug_phase(unsigned long long* out) {
  for (int i = 0; i < 8; ++i) out[i] = 0;   // (slots of the removed band format)
  ocp::read_bphase(out + 8);
  {   // + the narrow-line instance's counters (one of the two instances runs per context)
    unsigned long long nw[8];
    ocp_nw::read_bphase(nw);
    for (int i = 0; i < 8; ++i) out[8 + i] += nw[i];
  }
  ocp::read_aphase(out + 16);
  return 0;
}
#endif

int ocp_check_guards(long long* corrupted, long long* buffers) {
  ocp_ctx* ctx = nullptr;
  if (!corrupted || !buffers) return fail(ctx, OCP_ERR_ARG, "null argument");
  *corrupted = 0;
  *buffers = 0;
  if (!guard_on()) return fail(ctx, OCP_ERR_ARG, "guard zones are off (set OCP_GUARD=1)");
  CK(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_guard_mu);
  *corrupted = g_guard_freed_bad;   // buffers freed so far were checked at free
  for (const auto& kv : g_guards) {
    const long long bad = count_guard(kv.second.first, kv.second.second, &g_guard_first);
    if (bad < 0) return fail(ctx, OCP_ERR_CUDA, "guard readback failed");
    *corrupted += bad;
    ++*buffers;
  }
  if (*corrupted) g_global_err = g_guard_first;
  return OCP_OK;
}

int ocp_event_record(ocp_ctx* ctx, int slot) {
  if (!ctx || slot < 0 || slot >= 16) return OCP_ERR_ARG;
  if (!ctx->marks[slot]) CK(cudaEventCreate(&ctx->marks[slot]));
  CK(cudaEventRecord(ctx->marks[slot], ctx->stream));
  return OCP_OK;
}

int ocp_event_elapsed(ocp_ctx* ctx, int a, int b, double* ms) {
  if (!ctx || a < 0 || a >= 16 || b < 0 || b >= 16 || !ctx->marks[a] || !ctx->marks[b])
    return OCP_ERR_ARG;
  CK(cudaEventSynchronize(ctx->marks[b]));
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, ctx->marks[a], ctx->marks[b]));
  *ms = f;
  return OCP_OK;
}

}  // extern "C"
