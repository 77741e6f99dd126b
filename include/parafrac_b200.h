/*
 * parafrac_b200 — C-ABI of the B200-native parareal fine-propagator path.
 *
 * Drop-in boundary for the reference package `parafrac` 0.1.0 (pure Python,
 * /root/reference/pkg/src/parafrac).  The reference has no FFI layer: its
 * boundary is Python function signatures.  Each entry point below replaces
 * one of those functions; INTEGRATION.md shows the ctypes binding a
 * maintainer adds to the reference.
 *
 *   pf_fine_sweep      <- stepping.fine_sweep_intervals   (stepping.py:189-243)
 *   pf_coarse_step     <- stepping.coarse_step            (stepping.py:87-112)
 *   pf_run_coarse      <- stepping.run_coarse             (stepping.py:115-121)
 *   pf_fine_propagate  <- stepping.fine_propagate         (stepping.py:142-186)
 *   pf_chain_fine      <- stepping.chain_fine             (stepping.py:246-257)
 *   pf_fine_sequential <- stepping.run_fine_sequential    (stepping.py:260-288)
 *   pf_parareal        <- parareal._solve                 (parareal.py:91-155)
 *   pf_last_error      <- errors.SolverFailure / CoefficientError /
 *                         DivergenceError / ValueError    (errors.py:8-34)
 *
 * Conventions: host arrays are row-major float64 and
 * caller-owned; the library copies in and out.  Entry points return PF_OK (0)
 * or an error code; pf_last_error() returns the details the reference's
 * exception carries (step, node, iteration).  There is no CPU fallback:
 * every compute entry point runs sm_100a kernels and fails with
 * PF_ERR_CUDA when no B200 is present.
 *
 * The pf_dev_* entry points take DEVICE pointers on the context's stream and
 * are the building blocks of the multi-GPU driver (one process per GPU,
 * slices sharded by parareal._block_bounds, parareal.py:62-72).
 */
#ifndef PARAFRAC_B200_H
#define PARAFRAC_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------- */
#define PF_OK 0
#define PF_ERR_ARGUMENT 1    /* ValueError (argument checks, stepping.py:98-99,158-163,199-200) */
#define PF_ERR_SOLVER 2      /* SolverFailure(step)            errors.py:8-17  */
#define PF_ERR_COEFFICIENT 3 /* CoefficientError(node_index)   errors.py:20-25 */
#define PF_ERR_DIVERGENCE 4  /* DivergenceError(iteration, n)  errors.py:28-34 */
#define PF_ERR_CUDA 5        /* CUDA runtime failure (no device, launch error)  */
#define PF_ERR_UNSUPPORTED 6 /* ValueError: unknown functor / size outside the built kernels */

/* ---- spatial discretisations ------------------------------------------- */
#define PF_SPACE_CHEB1D 1 /* the reference's Chebyshev-Lobatto collocation (spectral.py:74-136) */
#define PF_SPACE_SINE1D 2 /* sine spectral Galerkin, M modes, Q=2M midpoints */
#define PF_SPACE_SINE2D 3 /* tensor sine Galerkin, M x M modes */

/* ---- device coefficient functors (problems.py registry, BASELINE configs) */
/* D(x,t,u) and f(x,t,u) cannot be Python callbacks on the device; problems
 * are named functors with parameters p[0..5].                              */
#define PF_FN_POLY 1   /* D = p0 + p1*u ; f = p2*u + p3*sin(pi x)*exp(-t)
                          (paper42, linear-heat, constant-D, zero, problems.py:107-133) */
#define PF_FN_CFG12 2  /* D = 1 + u^2/(1+u^2) ; f = sin(pi x) cos(u)        (configs 1-2) */
#define PF_FN_CFG3 3   /* D = 1.5 + 0.5 tanh(u) ; f = -u + 0.1 sin(2 pi x)  (config 3)   */
#define PF_FN_CFG45 4  /* D = (1+0.5 x1)(1+0.5 sin(u)^2) ; f = u(1-u^2)/(1+u^2) (configs 4-5) */
#define PF_FN_NAN_AT 5 /* D = NaN where |x - p0| < 1e-12, else p1 ; f = 0  (failure injection) */

typedef struct pf_ctx pf_ctx;

typedef struct {
  int functor;      /* PF_FN_* */
  double p[6];      /* functor parameters */
  double alpha;     /* fractional order in (0, 1]          (problems.py:36) */
  double t_final;   /* horizon T                            (problems.py:35) */
  double a, b;      /* spatial interval (Chebyshev only; sine spaces use (0,1)) */
} pf_problem;

typedef struct {
  int nt; /* coarse intervals = parareal slices P  (l1.py:71) */
  int m;  /* fine steps per slice                  (l1.py:72) */
} pf_grid;

typedef struct {
  int kind;  /* PF_SPACE_* */
  int modes; /* sine: M per axis; Chebyshev: polynomial degree (npts = degree+1) */
  /* Chebyshev only: the caller's operator arrays (spectral.build_operator),
   * passed in so the device sees the caller's exact nodes / D1 / weights. */
  const double* nodes;        /* npts */
  const double* d1;           /* npts*npts row-major */
  const double* quad_weights; /* npts */
  /* sine spaces: PCG relative-residual tolerance and iteration cap */
  double pcg_tol;
  int pcg_maxit;
} pf_space;

/* L1 weight tables exactly as the caller computes them (l1.py:127-144), so
 * device results follow the caller's rounding of (x+1)^e - x^e.  NULL
 * pointers make the library evaluate the same formula with libm pow.    */
typedef struct {
  const double* b_fine; /* b_q,     q = 0..len_fine-1  (on_grid(1, .))  */
  long len_fine;        /* >= max(m, nt) + 2; nt*m + 1 for pf_fine_sequential */
  const double* b_frac; /* b_{q/m}, q = 0..len_frac-1  (on_grid(m, .))  */
  long len_frac;        /* >= (nt-1)*m + 1 */
  double gamma_2_minus; /* Gamma(2-alpha) (l1.py:40-42); <= 0: library computes exp(lgamma) */
} pf_weights;

typedef struct {
  int code;       /* PF_* */
  int step_n;     /* SolverFailure.step: coarse step index, or interval of (n, r) */
  int step_r;     /* substep r of (n, r); -1 for a coarse step                    */
  int node;       /* CoefficientError.node_index                                  */
  int iteration;  /* DivergenceError.iteration                                    */
  int interval;   /* DivergenceError.interval                                     */
  int cuda_error; /* cudaError_t when code == PF_ERR_CUDA                          */
  char message[256];
} pf_error;

typedef struct {
  long long fine_launches;      /* fine-sweep kernel launches since create      */
  long long coarse_launches;    /* coarse / correction kernel launches          */
  long long pcg_iterations;     /* PCG iterations summed over every solve (sine) */
  long long solves;             /* linear solves (substeps + coarse steps)      */
  double last_fine_ms;          /* device time of the last fine-sweep launch    */
  double last_coarse_ms;        /* device time of the last coarse-kernel launch */
  long long helper_launches;    /* fine sweeps that ran with far-history helper CTAs */
  long long kernel_launches;    /* every kernel this context launched */
} pf_stats;

/* ---- lifecycle ---------------------------------------------------------- */
int pf_create(const pf_problem* problem, const pf_grid* grid, const pf_space* space,
              const pf_weights* weights, int device, pf_ctx** out);
void pf_destroy(pf_ctx* ctx);
int pf_last_error(const pf_ctx* ctx, pf_error* out);
int pf_state_size(const pf_ctx* ctx);
int pf_get_stats(const pf_ctx* ctx, pf_stats* out);
int pf_reset_stats(pf_ctx* ctx);
/* cudaStream_t used by every launch (NULL = the context's own stream). */
int pf_set_stream(pf_ctx* ctx, void* stream);
const char* pf_version(void);
/* development aid: per-phase cycle counters of slice 0 (zeros unless built with -DPF_PHASE_TIMING) */
int pf_debug_phases(long long* out16, int reset);
/* development aid: per-warp clock64 timeline of 8 substeps of one slice CTA, out[8 warps][8 substeps][64
   points] (zeros unless built with -DPF_TRACE; tools/r02/trace.py) */
int pf_debug_trace(long long* out4096);
/* development aid: clock64 at the loop top of substeps 0..n-1 (n <= 4096) of the traced slice (-DPF_TRACE) */
int pf_debug_looptop(long long* out, int n);
/* development aid: entry/exit times (GPU globaltimer, ns) of each slice of the last 1-D fine
   sweep, out[2i] = entry, out[2i+1] = exit (load-balance diagnostic, tools/slice_finish.py) */
int pf_debug_slice_times_ns(const pf_ctx* ctx, long long* out, int n);

/* ---- host-buffer entry points (reference-facing) ------------------------ */
/* stepping.coarse_step: history = states at coarse nodes 0..n_states-1 */
int pf_coarse_step(pf_ctx* ctx, const double* history, int n_states, int step_index, double* out);
/* stepping.run_coarse: traj has (nt+1) rows, traj[0] = u0 */
int pf_run_coarse(pf_ctx* ctx, const double* u0, double* traj);
/* stepping.fine_sweep_intervals: u_nodes has (n_states) rows, out (n_hi-n_lo) rows */
int pf_fine_sweep(pf_ctx* ctx, const double* u_nodes, int n_states, int n_lo, int n_hi, double* out);
/* stepping.fine_propagate: start (size; NULL = coarse_history[n]) seeds path[0]
 * (stepping.py:170-171), coarse_history rows 0..n feed the bracket; endpoint
 * (size) and path (m, size) */
int pf_fine_propagate(pf_ctx* ctx, const double* start, const double* coarse_history, int n_states,
                      double* endpoint, double* path);
/* stepping.chain_fine: traj (nt+1) rows */
int pf_chain_fine(pf_ctx* ctx, const double* u0, double* traj);
/* stepping.run_fine_sequential: states (nt+1) rows (every m-th fine state) */
int pf_fine_sequential(pf_ctx* ctx, const double* u0, double* states);
/* parareal._solve.  tol <= 0 disables the stop rule (tol=None).  reference
 * (nullable, (nt+1) rows) enables errors_vs_reference (k_max+1 entries).
 * Outputs: states (nt+1 rows), coarse_new/coarse_old/fine_endpoints (nt rows),
 * diffs/iteration_times (k_max entries), *iterations, *stop_reason (0 k_max,
 * 1 tol).  Any output pointer may be NULL. */
int pf_parareal(pf_ctx* ctx, const double* u0, double tol, int k_max, const double* reference,
                double* states, double* coarse_new, double* coarse_old, double* fine_endpoints,
                double* diffs, double* iteration_times, double* errors, int* iterations,
                int* stop_reason);

/* ---- device-buffer building blocks (multi-GPU driver, bench) ------------ */
/* Fine sweep of slices [n_lo, n_hi) from device states d_u (>= n_hi+1 rows)
 * into d_out ((n_hi-n_lo) rows).  Synchronises the stream and checks status. */
int pf_dev_fine_sweep(pf_ctx* ctx, const double* d_u, int n_lo, int n_hi, double* d_out);
/* Same, without the trailing synchronisation / status check (bench timing). */
int pf_dev_fine_sweep_async(pf_ctx* ctx, const double* d_u, int n_lo, int n_hi, double* d_out);
int pf_dev_check(pf_ctx* ctx); /* synchronise and translate device status */
/* Parareal state machine on device: init runs run_coarse from host u0 and
 * sets coarse_old = traj[1:]; correct runs the sequential sweep
 * (parareal.py:114-128) with fine endpoints d_fold (nt rows, device), the
 * guards, and writes the iterate's diff; iteration k names errors. */
int pf_dev_parareal_init(pf_ctx* ctx, const double* u0);
const double* pf_dev_parareal_states(pf_ctx* ctx); /* device pointer, (nt+1) rows */
int pf_dev_parareal_correct(pf_ctx* ctx, const double* d_fold, int k, double* diff);
int pf_dev_parareal_read(pf_ctx* ctx, double* states, double* coarse_new, double* coarse_old);
/* Leading nodes the last correction left bitwise unchanged (0 before the
 * first).  Slices below it have exactly the inputs of their previous fine
 * sweep, so their F_old rows stand and the next sweep may start there --
 * parareal's finite termination (parareal.py:114-118, 175-189) made exact. */
int pf_dev_parareal_frozen(pf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PARAFRAC_B200_H */
