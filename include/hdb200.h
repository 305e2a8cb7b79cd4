/*
 * hdb200 — C ABI of the B200-native MADP-FGMRES library (libhdb200.so).
 *
 * Drop-in boundary for the reference package `helmdef` (arXiv 2412.04980
 * reference implementation, /root/reference/pkg/src/helmdef).  The reference
 * has no FFI of its own: its "plugin surface" is the Python API re-exported in
 * __init__.py:9-62.  Each entry point below replaces the compute behind one
 * reference call (file:line relative to pkg/src/helmdef/); the Python package
 * paper_2412_04980_b200 binds them with ctypes and keeps the reference names
 * and signatures.
 *
 * Conventions
 *   - complex128 fields are interleaved (re, im) doubles, row-major (x fastest),
 *     exactly numpy's complex128 layout; k^2 fields are float64.
 *   - pointers are DEVICE pointers unless the argument name ends in _host.
 *   - every function returns a status: 0 ok, 1 bad argument (ShapeError /
 *     LevelError / ConfigError), 2 CUDA failure (HelmdefError), 3 non-finite
 *     value (NumericalError), 4 multigrid divergence (MgDivergence), 5 Bi-CGSTAB
 *     breakdown (BreakdownError; x holds the best iterate);
 *     hdb_last_error() returns the message of the last failure (thread-local).
 *   - all work is ordered on one library stream per process (hdb_stream);
 *     functions that return host scalars synchronise it.
 *   - boundary kinds per side (west, east, south, north): 0 Sommerfeld, 1 Dirichlet.
 */
#ifndef HDB200_H
#define HDB200_H
#ifdef __cplusplus
extern "C" {
#endif

#define HDB_OK 0
#define HDB_E_ARG 1
#define HDB_E_CUDA 2
#define HDB_E_NONFINITE 3
#define HDB_E_MGDIV 4
#define HDB_E_BREAKDOWN 5

typedef struct hdb_op hdb_op;        /* one level operator  -Lap - shift*I(k^2)   */
typedef struct hdb_mg hdb_mg;        /* CSLP multigrid (mg.py:51)                  */
typedef struct hdb_solver hdb_solver;/* MADP solver (madp.py:220)                  */

/* out = Op(in) on device buffers of the operator's level; return nonzero on failure */
typedef int (*hdb_linop_fn)(void* user, const void* in, void* out);
/* on_iteration(iteration, relres) hook (krylov.py:153-154); return nonzero to abort */
typedef int (*hdb_iter_fn)(void* user, int iteration, double relres);

/* ---- library ------------------------------------------------------------ */
int hdb_version(void);
const char* hdb_last_error(void);
/* select the device and create the library stream (idempotent per device) */
int hdb_init(int device);
int hdb_stream(void** stream_out);
/* order all library work on an external stream (e.g. torch's current stream) */
int hdb_set_stream(void* stream);
int hdb_sync(void);
/* kernels launched through the library so far, device bytes allocated */
int hdb_stats(long long* launches, long long* bytes_alloc);
/* ranks: one process per GPU over NCCL (id from hdb_comm_unique_id on rank 0,
 * broadcast by the caller), or host threads of one process, each with its own
 * engine (hdb_thread_engine_begin) — used to test the slab path on one GPU    */
int hdb_comm_unique_id(char* out128);
int hdb_comm_init_nccl(const char* id128, int nranks, int rank);
/* one-rank NCCL round trip on this engine's device (library resolution, communicator,
   all-reduce / grouped send-recv / all-gather of the slab path, results checked): what a
   single GPU can verify of the NCCL transport */
int hdb_comm_selftest_nccl(void);
int hdb_comm_init_threads(long long group, int nranks, int rank);
/* host-only rule of the sharded -> replicated level transition: the coarse rows
 * [*row0, *row0 + *ny) this rank restricts before the all-gather, given every
 * rank's fine slab start (no device needed)                                   */
int hdb_plan_gather_rows(const int* fine_slab_row0, int nranks, int rank, int ncy_g, int* row0, int* ny);
int hdb_thread_engine_begin(int device);
int hdb_thread_engine_end(void);

/* ---- level operators: replaces LevelOperator (operators.py:96-208) -------- */
/* lap: (2r+1)^2 float coefficients = lap_coef (operators.py:111);
 * mass_re/mass_im: mass_coef (operators.py:112-113); ksq_host: ny*nx k^2   */
int hdb_op_create(hdb_op** out, int nx, int ny, int radius, double h, const int* bc4,
                  const double* lap, const double* mass_re, const double* mass_im,
                  const double* ksq_host);
int hdb_op_destroy(hdb_op* op);
/* row slab [row0, row0+ny_local) of a level with ny_global rows (row-slab
 * decomposition); `halo` rows (>= radius, >= 2) are carried by
 * this level's vectors; slab_row0/slab_ny: every rank's slab                  */
int hdb_op_create_slab(hdb_op** out, int nx, int ny_global, int radius, double h, const int* bc4,
                       const double* lap, const double* mass_re, const double* mass_im,
                       const double* ksq_full_host, int row0, int ny_local, int halo, int nranks,
                       const int* slab_row0, const int* slab_ny);
/* the same operator from a k^2 field already on the device (GPU-side setup, below): the
   field is range-checked (finite, nonnegative: grid.py:266-267) and copied device to
   device; whole grid, one rank */
int hdb_op_create_dev(hdb_op** out, int nx, int ny, int radius, double h, const int* bc4, const double* lap,
                      const double* mass_re, const double* mass_im, const double* ksq_dev);

/* ---- problem setup on the device; every field bit-identical to grid.py ----
   k^2 = (w / c)^2 with w = 2 pi f at the vertices (ox + hx i, oy + hy j), row-major (ny, nx):
   _fine_ksq grid.py:261-268; constant: the value itself; wedge: `nlayers` (y at first x, y at
   last x, velocity) triples top to bottom, the last one the catch-all (grid.py:120-135);
   raster: bilinear sampling of a device float64 raster (rny, rnx), origin (rx0, ry0), steps
   (rdx, rdy), clamped (grid.py:138-160) */
int hdb_setup_ksq_constant(double* out_dev, long long n, double ksq);
int hdb_setup_ksq_wedge(double* out_dev, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                        int nlayers, const double* layers3);
int hdb_setup_ksq_raster(double* out_dev, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                         const double* raster_dev, int rnx, int rny, double rx0, double ry0, double rdx, double rdy);
/* coarse k^2 by injection at coincident vertices, ksq[::2, ::2] (grid.py:285) */
int hdb_setup_inject(const double* fine_dev, int nfx, int nfy, double* coarse_dev);
/* out3 = { min, max, number of non-finite values } of a device float64 array (finite values only) */
int hdb_setup_stats(const double* a_dev, long long n, double* out3);
/* point_source_rhs (grid.py:309-320): rhs = 0 except rhs[index] = value (= 1 / (hx hy)) */
int hdb_setup_point_source(void* rhs_dev, long long n, long long index, double value);

/* LevelOperator.apply (operators.py:130-147): out = A u, Dirichlet rows pinned */
int hdb_op_apply(hdb_op* op, const void* u, void* out);
/* out = b - A u  (MG residual mg.py:116, A-DEF1 v - A t madp.py:325-326) */
int hdb_op_residual(hdb_op* op, const void* b, const void* u, void* out);
/* fused matvec + residual + norms (MG divergence guard, mg.py:131-138):
   out2 = { ||b - A u||^2, ||b||^2 }; the residual is not stored (radius 1: one
   pass over u, b, k^2 — 40 B/pt); synchronises to return the values
   (out2 == NULL: enqueue only, no sync — microbenchmarks) */
int hdb_op_resnorm(hdb_op* op, const void* b, const void* u, double* out2);
/* one damped-Jacobi sweep (_kernels.py:53-68 + mg.py:88-102); x == NULL: from zero */
int hdb_op_jacobi(hdb_op* op, const void* x, const void* b, void* out, double omega);
/* fused MG coarse right-hand side (mg.py:116-117): coarse = Z^T (b - A u), coarse Dirichlet
   rows zeroed per zero_mask (bit 0 west, 1 east, 2 south, 3 north); one pass, the residual is
   not stored (44 B per fine point instead of 56 + 20); unsharded radius-1 operators;
   bit-identical to hdb_op_residual followed by hdb_restrict */
int hdb_op_residual_restrict(hdb_op* op, const void* b, const void* u, void* coarse, int zero_mask);
/* the last post-smoothing sweep with the A-DEF1 sum folded in (mg.py:122 + madp.py:327):
   out = Jacobi(x), out2 = out + addt; bit-identical to hdb_op_jacobi followed by the add */
int hdb_op_jacobi_add(hdb_op* op, const void* x, const void* b, void* out, double omega, const void* addt,
                      void* out2);

/* ---- transfers: replaces restrict_array / prolong_array (transfers.py:59-88) */
/* zero_mask bits 1 W, 2 E, 4 S, 8 N: coarse rows set to 0 (mg.py:118-119)  */
int hdb_restrict(const void* fine, int nfy, int nfx, void* coarse, int zero_mask);
/* fine = Z coarse  (base != NULL: fine = base + Z coarse, mg.py:121)          */
int hdb_prolong(const void* coarse, int nfy, int nfx, const void* base, void* fine);

/* ---- reductions: replaces reduce_dot (parallel.py:168-195) ---------------- */
/* out2_host == NULL: enqueue only (result stays on the device; microbenchmarks) */
int hdb_dot(const void* u, const void* v, long long n, double* out2_host);

/* ---- CSLP multigrid: replaces CslpMultigrid (mg.py:59-139) ---------------- */
/* ops: sub-level operators finest first (radius 1); inv_host: dense inverse of
 * the coarsest operator (ninv x ninv complex, row-major) or NULL for the GMRES
 * fallback with (coarse_tol, coarse_max)                                      */
int hdb_mg_create(hdb_mg** out, hdb_op* const* ops, int nlev, const double* inv_host, int ninv,
                  double omega, int pre, int post, double guard, double coarse_tol, int coarse_max);
int hdb_mg_destroy(hdb_mg* mg);
/* one V-cycle (mg.py:125-139) from x0 (NULL: zero); HDB_E_MGDIV on the guard  */
int hdb_mg_vcycle(hdb_mg* mg, const void* b, const void* x0, void* x);

/* ---- Krylov: replaces fgmres / gmres (krylov.py:61-182) ------------------- */
/* x0 may be NULL (zero initial guess); M may be NULL (GMRES); hook may be NULL */
int hdb_fgmres(long long n, hdb_linop_fn A, void* A_user, hdb_linop_fn M, void* M_user,
               const void* b, const void* x0, void* x, double rel_tol, int max_iters,
               hdb_iter_fn hook, void* hook_user,
               int* iterations, double* final_relres, int* converged,
               double* history_host, int history_cap);

/* Bi-CGSTAB (krylov.py:185-276); HDB_E_BREAKDOWN leaves the best iterate in x
 * and its counts in the outputs                                              */
int hdb_bicgstab(long long n, hdb_linop_fn A, void* A_user, hdb_linop_fn M, void* M_user,
                 const void* b, const void* x0, void* x, double rel_tol, int max_iters,
                 int* iterations, double* final_relres, int* converged,
                 double* history_host, int history_cap, int* history_len);

/* GMRES on one level operator, no preconditioner (the CSLP solve of
 * madp.py:290-291): mode -1 launch-driven engine, 0 device-resident on one
 * thread-block cluster, 1 device-resident cooperative grid, 2 automatic      */
int hdb_op_gmres(hdb_op* op, const void* b, void* x, double rel_tol, int max_iters, int mode,
                 int* iterations, double* final_relres);

/* telemetry: enable=1 zeroes and arms per-phase cycle counters of the
 * device-resident solver; enable=0 disarms and copies the 12 counters out    */
int hdb_resident_profile(int enable, long long* host_out12);

/* ---- MADP solver: replaces MadpSolver (madp.py:220-371) ------------------- */
int hdb_solver_create(hdb_solver** out, int ml, double outer_tol, int outer_max);
/* cslp: 0 none, 1 mg, 2 gmres, 3 bicgstab (madp.py:55-58); level 1 ignores the cycle rule */
int hdb_solver_set_level(hdb_solver* s, int level, hdb_op* A, hdb_op* M, hdb_mg* mg, int cslp,
                         double cslp_tol, int cslp_max, double cycle_tol, int cycle_max);
/* MadpSolver.solve (madp.py:329-371); host_buffers != 0: b, x are host pointers
 * (copies included in the call)                                              */
int hdb_solver_solve(hdb_solver* s, const void* b, void* x, int host_buffers);
int hdb_solver_report(hdb_solver* s, int* outer_iterations, int* converged, double* final_relres,
                      double* wall_ms, int* history_len);
int hdb_solver_history(hdb_solver* s, double* history_host, double* iteration_wall_ms_host, int cap);
/* kind 0: deflation-cycle iterations, 1: CSLP iterations, per application    */
int hdb_solver_counts(hdb_solver* s, int level, int kind, int* buf_host, int cap, int* count);
int hdb_solver_matvecs(hdb_solver* s, long long* buf_host, int cap);
/* MadpSolver.apply_preconditioner (madp.py:301-327) on device vectors */
int hdb_solver_precond(hdb_solver* s, int level, const void* v, void* out);
/* telemetry of the last solve: inclusive host ms and call counts per
 * (level, role) at index level*3 + role (0 deflation FGMRES, 1 CSLP, 2 A-DEF1),
 * host synchronisations and kernel launches                                   */
int hdb_solver_profile(hdb_solver* s, double* ms_host, long long* calls_host, int cap,
                       long long* syncs, long long* launches);
/* algorithmic HBM bytes of the last solve's launches (SURVEY §8(d) per-point
 * figures x points, counted by the host driver; device-resident solves from
 * their iteration counts) -> solve-level achieved bandwidth = bytes / time      */
int hdb_solver_bytes(hdb_solver* s, double* alg_bytes);
int hdb_solver_destroy(hdb_solver* s);

/* separable form of a radius-2/3 Galerkin operator (host-verified factors,
 * 2r+1 entries each): lap = lsc (sa (x) sm + sm (x) sa), mass = msc (sm (x) sm);
 * the level then applies as 1D passes (K2) unless "rg_exact" is set          */
int hdb_op_set_separable(hdb_op* op, const double* sa, const double* sm, double lsc, double msc_re,
                         double msc_im);

/* ---- engine options (not on the reference API) ----------------------------- */
/* "mgs_ls": 1 (default) one-launch MGS steps of large levels use the
 * low-synchronisation form (two grid reductions per Arnoldi step), 0 the
 * reference's coefficient-by-coefficient MGS order (HDB_MGS_LS=0 likewise).
 * "rg_exact": 1 radius-2/3 operators use the reference's row-major tap order
 * (bit-identical to contract_general; HDB_RG_EXACT=1), 0 (default) the
 * separable 1D passes where the operator has them.
 * "pinv": 1 every reduction of a level sums per-row partials in global row order
 * and every level keeps the launch-driven Krylov path, so a solve is bit-identical
 * on any number of ranks (reduce_dot's worker-count invariance, parallel.py:168-195;
 * HDB_PINV=1); 0 (default) the fast per-rank reduction trees.
 * "lsh_prefer": 1 levels beyond the one-launch low-synchronisation step (> 7168
 * points per CTA) use its HBM-streaming form instead of the MGS-order one-launch
 * kernels (HDB_LSH_PREFER=1); 0 (default: measured equal or slower)             */
int hdb_option(const char* name, int value);

/* ---- launch accounting / timing (measurement, not on the reference API) ---- */
/* enable = 1: zero the per-family counters and record a CUDA-event pair on the
 * library stream around every launch; 0: counters only (always on)           */
int hdb_kprof(int enable);
/* family fam (0..count-1; fam < 0 returns the count in *launches): name,
 * launches, algorithmic bytes and summed event time (ms) since hdb_kprof      */
int hdb_kprof_read(int fam, char* name_out32, long long* launches, double* alg_bytes, double* device_ms);

#ifdef __cplusplus
}
#endif
#endif
