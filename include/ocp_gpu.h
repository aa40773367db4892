/*
 * ocp_gpu.h - C ABI of the B200 (sm_100a) RASPEN hot path.
 *
 * The reference (`ocp`, pure Python) has no FFI; its operator protocol for
 * this path is a set of Python callables.  These entry points
 * are what a binding of that protocol needs; each cites the reference
 * function it replaces.  Conventions:
 *
 *   - plain pointers and sizes only; "dev" pointers are CUDA device memory
 *     (from ocp_malloc), "host" pointers are ordinary host memory;
 *   - every call returns an ocp_status; no exception crosses the ABI;
 *     ocp_last_error(ctx) holds the message of the last failing call;
 *   - one context per (problem, decomposition); one CUDA stream per context;
 *     calls on one context are not reentrant (the Python shim serialises);
 *   - global vectors are [y; p] of length 2N, N = n*n, row-major fields
 *     (`pkg/src/ocp/system.py:109-115`, `pkg/src/ocp/grid.py:26-33`);
 *   - "reference local layout" is [y_loc; p_loc] with the overlap rectangle
 *     row-major, concatenated over subdomains in decomposition order
 *     (`pkg/src/ocp/schwarz.py:88-91,116-119`).
 */
#ifndef OCP_GPU_H
#define OCP_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ocp_ctx ocp_ctx;

typedef enum {
  OCP_OK = 0,
  OCP_ERR_ARG = 1,            /* ValueError: bad argument / decomposition */
  OCP_ERR_CUDA = 2,           /* CUDA runtime failure */
  OCP_ERR_LOCAL_SOLVE = 3,    /* LocalSolveError(subdomain, msg), schwarz.py:32-37 */
  OCP_ERR_NONFINITE = 4,      /* NonfiniteFieldError(where, index), grid.py:9-23 */
  OCP_ERR_NONFINITE_INIT = 5, /* ValueError("nonfinite residual at the initial guess"), newton.py:146-147 */
  OCP_ERR_UNSUPPORTED = 6,    /* shape outside the compiled kernel limits */
  OCP_ERR_NO_DEVICE = 7,
  OCP_ERR_GMRES_BREAKDOWN = 8 /* GmresBreakdownError, krylov.py:15 */
} ocp_status;

/* phi selector: kappa*(s^3+e^{kappa s}) (system.py:31-74), y^3, e^y-1 */
enum { OCP_PHI_KAPPA = 0, OCP_PHI_CUBIC = 1, OCP_PHI_EXPM1 = 2 };

/* ---- context ------------------------------------------------------------
 * Replaces decompose + build_local_systems (schwarz.py:94-163): builds the
 * reference tiling (_tile_edges: remainder to the last tile, overlap clipped),
 * uploads f and y_d, sizes the local pools.  Errors mirror decompose's
 * ValueErrors (message in ocp_last_error(NULL) when *out is not created).
 * s1 = s2 = 0 creates a grid-only context (whole-grid operators, no subdomains). */
int ocp_ctx_create(int n, int s1, int s2, int overlap, double nu, double mu,
                   int phi_kind, double kappa, const double* f_host,
                   const double* y_d_host, ocp_ctx** out);
void ocp_ctx_destroy(ocp_ctx* ctx);
const char* ocp_last_error(const ocp_ctx* ctx);
/* info[0]=subdomains, [1]=local pool doubles, [2]=factor-store doubles,
 * [3]=max padded half-bandwidth, [4]=panel width NB, [5]=sum of 2*R_i*C_i,
 * [6]=reference-layout local length */
int ocp_ctx_info(const ocp_ctx* ctx, long long* info);
/* rects[11*i ...]: r0 r1 c0 c1 own_r0 own_r1 own_c0 own_c1 orient nr nc */
int ocp_subdomain_table(const ocp_ctx* ctx, int* rects);

/* ---- device memory (the context's stream) ------------------------------ */
int ocp_malloc(size_t bytes, void** dev);
int ocp_free(void* dev);
int ocp_h2d(ocp_ctx* ctx, void* dev, const void* host, size_t bytes);
int ocp_d2h(ocp_ctx* ctx, void* host, const void* dev, size_t bytes);
int ocp_d2d(ocp_ctx* ctx, void* dst, const void* src, size_t bytes);
int ocp_memset0(ocp_ctx* ctx, void* dev, size_t bytes);
int ocp_sync(ocp_ctx* ctx);

/* ---- the hot path ------------------------------------------------------- */

/* One RAS sweep: every subdomain's frozen-exterior damped Newton with the
 * eps schedule (eps0, gamma, eps_min) [inner newton_continuation,
 * newton.py:133-181, via _solve_local schwarz.py:194-200], then the
 * refactorisation at the converged values into fac_dev (schwarz.py:305-315)
 * and f_val = sum_i P~_i values_i - x (schwarz.py:317).
 * Replaces raspen_residual (schwarz.py:285-324).
 *   x_dev      [2N] frozen global iterate
 *   fac_dev    factor store of ocp_ctx_info()[2] doubles (written)
 *   fval_dev   [2N] output
 *   inner_iters_host [I] per-subdomain inner Newton iterations
 *   failed_sub_host  lowest failing subdomain or -1
 * Returns OCP_ERR_LOCAL_SOLVE with the reference message text in
 * ocp_last_error when a subdomain fails. */
int ocp_raspen_residual(ocp_ctx* ctx, const double* x_dev, double* fac_dev,
                        double eps0, double gamma, double eps_min,
                        double inner_tol, int inner_max_outer, double sigma,
                        int max_halvings, double* fval_dev,
                        int* inner_iters_host, int* failed_sub_host);

/* ocp_raspen_residual with the refactorisation at `eps` instead of the
 * inner schedule's floor: raspen_residual(x, dec, spec, eps, inner_cfg,
 * inner_sched) solves the local problems along inner_sched and factors the
 * local Jacobians at eps (schwarz.py:296-315). */
int ocp_raspen_residual_at(ocp_ctx* ctx, const double* x_dev, double* fac_dev, double eps,
                           double eps0, double gamma, double eps_min,
                           double inner_tol, int inner_max_outer, double sigma,
                           int max_halvings, double* fval_dev,
                           int* inner_iters_host, int* failed_sub_host);

/* Inner Newton of subdomain `sub` alone (local_correction, schwarz.py:211-218):
 * only that subdomain is solved, so another subdomain's failure cannot
 * surface.  Its values are then read with ocp_local_values; fac_dev is the
 * scratch factor store of the inner solves (no refactorisation at the values,
 * no f_val).  inner_iters_host[sub] receives its count. */
int ocp_local_correction(ocp_ctx* ctx, const double* x_dev, double* fac_dev, int sub,
                         double eps0, double gamma, double eps_min,
                         double inner_tol, int inner_max_outer, double sigma,
                         int max_halvings, int* inner_iters_host, int* failed_sub_host);

/* Jacobian action from the stored factors of the last ocp_raspen_residual
 * into fac_dev: out[own_i] = -(d_loc + J_i^{-1} A_ext d)[own_i].
 * Replaces raspen_jacobian_apply (schwarz.py:327-345). */
int ocp_raspen_jvp(ocp_ctx* ctx, const double* fac_dev, const double* d_dev,
                   double* out_dev);

/* Current local values (last sweep) in the reference local layout. */
int ocp_local_values(ocp_ctx* ctx, double* values_dev);

/* Parity hooks for the kernels: local residual of every subdomain at local
 * values v (reference layout) with the exterior frozen at x
 * (_local_problem.local_residual, schwarz.py:181-186), and one Newton
 * direction -J(v)^{-1} F(v) by the batched block-Thomas factor (newton.py:127). */
int ocp_local_residual(ocp_ctx* ctx, const double* x_dev, const double* v_ref_dev,
                       double eps, double* r_ref_dev);
int ocp_local_direction(ocp_ctx* ctx, const double* x_dev, const double* v_ref_dev,
                        double eps, double* d_ref_dev);
/* Squared norms of the line-search trial residual ||F_i(v_i + alpha_i d_i)||^2 of every
 * subdomain (newton.py:96-112: residual(x + alpha * d), product rounded first), the
 * staged-direction instance of the residual kernel; v, d in the reference layout,
 * alpha_host / norm2_host: I doubles on the host.  Parity hook. */
int ocp_local_residual_trial(ocp_ctx* ctx, const double* x_dev, const double* v_ref_dev,
                             const double* d_ref_dev, const double* alpha_host, double eps,
                             double* norm2_host);

/* ---- GMRES vector kernels (krylov.py:44-151), deterministic reductions -- */
int ocp_vec_nrm2(ocp_ctx* ctx, long long n, const double* x, double* out_host);
int ocp_vec_dot(ocp_ctx* ctx, long long n, const double* x, const double* y,
                double* out_host);
/* out = x + alpha*d  (numpy: x + alpha * d, product rounded first) */
int ocp_vec_add_scaled(ocp_ctx* ctx, long long n, const double* x, double alpha,
                       const double* d, double* out);
/* out = a*x  */
int ocp_vec_scale(ocp_ctx* ctx, long long n, double a, const double* x, double* out);
/* out = x / s */
int ocp_vec_div(ocp_ctx* ctx, long long n, const double* x, double s, double* out);
int ocp_vec_equal(ocp_ctx* ctx, long long n, const double* x, const double* y,
                  int* equal_host);
int ocp_vec_all_finite(ocp_ctx* ctx, long long n, const double* x, int* finite_host);
/* Modified Gram-Schmidt of w against Q[:, 0..j] (columns ldq apart):
 * h_i = q_i.w ; w -= h_i q_i (krylov.py:113-115), then h[j+1] = ||w||.
 * h_host receives j+2 values. */
int ocp_mgs(ocp_ctx* ctx, long long n, const double* Q, long long ldq, int j,
            double* w, double* h_host);
/* One whole Arnoldi step (krylov.py:110-122): MGS of w_in = A q_j against
 * Q[:, 0..j] (w_in is not modified), h_host[0..j+1], and
 * Q[:, j+1] = w / h[j+1] (written even on a happy breakdown; unused then).
 * Single cooperative kernel; falls back to per-pass kernels for large n. */
int ocp_arnoldi(ocp_ctx* ctx, long long n, double* Q, long long ldq, int j,
                const double* w_in, double* h_host);
/* Unpreconditioned, unrestarted MGS-GMRES on the RASPEN Jacobian action
 * (the configuration raspen_solve uses: newton.py:115-124 with precond None,
 * krylov.py:44-151 with x0 None).  Everything of one GMRES solve in one
 * call: JVPs and Arnoldi steps on the device, Givens rotations / back
 * substitution on the host in float64 with the reference's operation order.
 *   b_dev  [n] right-hand side;  x_dev [n] solution (written)
 *   history_host [max_iters+1] residual history (len = iters + 1)
 * Returns OCP_ERR_GMRES_BREAKDOWN for nonfinite Arnoldi entries. */
int ocp_raspen_gmres(ocp_ctx* ctx, const double* fac_dev, const double* b_dev, double rel_tol,
                     double abs_tol, int max_iters, double* x_dev, int* iters_host,
                     double* residual_host, int* converged_host, double* history_host);
/* out = x + Q[:, :k] @ y  (krylov.py:151) */
int ocp_gemv_add(ocp_ctx* ctx, long long n, const double* Q, long long ldq, int k,
                 const double* y_host, const double* x, double* out);
/* ---- linear-RAS Newton-Krylov (method newton-ras-eps) -------------------
 * harness/experiments.py:72-84: monolithic newton_continuation on the global
 * residual with GMRES left-preconditioned by one-level RAS. */
/* r = F_eps(x) on the whole grid, check=False  (system.py:147-152) */
int ocp_global_residual(ocp_ctx* ctx, const double* x_dev, double eps, double* r_dev);
/* Jacobian of F_eps at x as its per-point diagonals jd_dev[4N] =
 * (4/h^2 + phi'(y), b12, b21, 0)  (system.py:135-144, 155-160: jacobian()).
 * OCP_ERR_NONFINITE "phi'(y)@k" / "phi''(y)@k" like the reference's checks. */
int ocp_global_jacobian(ocp_ctx* ctx, const double* x_dev, double eps, double* jd_dev);
/* out = J d, the CSR row sums of jacobian(x) @ d  (system.py:155-160) */
int ocp_global_jvp(ocp_ctx* ctx, const double* jd_dev, const double* d_dev, double* out_dev);
/* ras_preconditioner build (schwarz.py:221-232): local pair Jacobians at
 * x[pair_idx] of every subdomain, batched block factor into fac_dev (a factor
 * store as for ocp_raspen_residual).  OCP_ERR_LOCAL_SOLVE ("singular local
 * block") / OCP_ERR_NONFINITE with *failed_sub = subdomain. */
int ocp_ras_factor(ocp_ctx* ctx, const double* x_dev, double eps, double* fac_dev,
                   int* failed_sub);
/* out = sum_i P~_i J_i^-1 R_i v  (the apply closure, schwarz.py:234-239) */
int ocp_ras_apply(ocp_ctx* ctx, const double* fac_dev, const double* v_dev, double* out_dev);
/* GMRES on J(x) (jd_dev) left-preconditioned by the RAS factors: the
 * direction solve of newton.py:115-124 with precond = ras_preconditioner
 * (krylov.py:44-151: threshold on ||M b||, w = M J q_j).  Same outputs and
 * status codes as ocp_raspen_gmres. */
int ocp_ras_gmres(ocp_ctx* ctx, const double* jd_dev, const double* fac_dev, const double* b_dev,
                  double rel_tol, double abs_tol, int max_iters, double* x_dev, int* iters_host,
                  double* residual_host, int* converged_host, double* history_host);

/* ---- manufactured-problem setup on the device (system.py:181-265) -------
 * A context created with s1 = s2 = 0 is grid-only (no subdomains): the
 * whole-grid and state-equation entry points work, the subdomain ones
 * return OCP_ERR_ARG. */
/* out = A y + phi(y) - rhs  (solve_state's residual, check=False, system.py:188-189) */
int ocp_state_residual(ocp_ctx* ctx, const double* y_dev, const double* rhs_dev, double* out_dev);
/* (A + diag(phi'(y))) x = b by CG from x = 0 to ||r|| <= rel_tol ||b||: the
 * device replacement of the direction solve splu(state_jacobian(y)).solve
 * (system.py:191-196); OCP_ERR_NONFINITE "phi'(y)@k" like the reference's
 * derivative check.  *converged_host = 0 when max_iters is reached. */
int ocp_state_cg(ocp_ctx* ctx, const double* y_dev, const double* b_dev, double rel_tol,
                 int max_iters, double* x_dev, int* iters_host, double* residual_host,
                 int* converged_host);
/* y_d = y_bar - A p_bar - phi'(y_bar) p_bar  (_manufacture, system.py:263) */
int ocp_manufacture_yd(ocp_ctx* ctx, const double* ybar_dev, const double* pbar_dev,
                       double* yd_dev);

/* u = -(p + mu P_eps(-p/mu))/nu  (system.py:173-174) */
int ocp_recover_control(ocp_ctx* ctx, long long n, const double* p, double eps,
                        double* u);

/* ---- instrumentation (bench.py) ----------------------------------------
 * stats[0]=kernel launches, [1]=factor ms, [2]=factor launches,
 * [3]=solve ms (stored-factor JVP solves), [4]=solve launches,
 * [5]=factor flops, [6]=JVP-solve factor bytes, [7]=residual-sweep ms,
 * [8]=DOF-updates, [9]=jvp ms, [10]=inner-solve ms, [11]=mgs ms,
 * [12]=full-set local-residual ms, [13]=its launches, [14]=its algorithmic bytes
 * Times need ocp_set_profiling(ctx, 1) (CUDA events on the context stream). */
int ocp_set_profiling(ocp_ctx* ctx, int on);
int ocp_stats(ocp_ctx* ctx, double* stats, int len);
int ocp_reset_stats(ocp_ctx* ctx);
/* CUDA events on the context stream (slot 0..15) for device-side timing of
 * whole solves; elapsed milliseconds between two recorded slots. */
int ocp_event_record(ocp_ctx* ctx, int slot);
int ocp_event_elapsed(ocp_ctx* ctx, int slot_a, int slot_b, double* ms_host);

/* Verification aid (not on the hot path): with OCP_GUARD=1 in the
 * environment every device buffer the library allocates carries 64 KB guard
 * zones of a fill pattern on both sides; this counts guard bytes that kernels
 * overwrote (out-of-bounds writes) across all live buffers.  OCP_ERR_ARG
 * when guard zones are off. */
int ocp_check_guards(long long* corrupted_bytes, long long* buffers);

#ifdef __cplusplus
}
#endif
#endif /* OCP_GPU_H */
