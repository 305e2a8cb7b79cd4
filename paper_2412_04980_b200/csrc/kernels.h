// Kernel launchers (internal C++ interface between the engine and the .cu files).
#pragma once
#include <functional>
#include "hdb_common.cuh"

namespace hdb {

struct RedWS {  // per-stream reduction workspace
  cd* partials = nullptr;   // kMaxReduceBlocks
  unsigned* ticket = nullptr;
  cd* big = nullptr;        // per-tile partials of the fused stencil norms (grown on demand)
  long long big_cap = 0;
};

int reduce_blocks(long long n);

// mode 0: out = A u ; mode 1: out = b - A u
void launch_apply(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* out, int mode,
                  cudaStream_t st);
// radius 1 only: dst = (||b - A u||^2, ||b||^2) in one pass (residual not stored)
long long resnorm_partials(const Geom& g);  // partial slots launch_resnorm needs
void launch_resnorm(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* partials,
                    cd* dst, cudaStream_t st);
// radius 1, unsharded: coarse = Z^T (b - A u) with coarse Dirichlet rows zeroed, one pass (mg.py:116-117)
bool resrestrict_fits(const OpCoef& c, const Geom& g);
void launch_resrestrict(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* coarse,
                        int zero_mask, cudaStream_t st);
void launch_jacobi(const OpCoef& c, const Geom& g, const cd* x, const cd* b, const double* k, cd* out, double omega,
                   bool from_zero, cudaStream_t st);
// Jacobi sweep with a second output out2 = out + addt (A-DEF1 r + t folded into the last post-smooth)
bool jacobi_add_fits(const Geom& g);
void launch_jacobi_add(const OpCoef& c, const Geom& g, const cd* x, const cd* b, const double* k, cd* out,
                       double omega, const cd* addt, cd* out2, cudaStream_t st);
// transfer geometry: fine rows [f_row0, f_row0+f_ny) of nfy_g, coarse rows [c_row0, c_row0+c_ny) of ncy_g
struct TGeom {
  int nfx, f_row0, f_ny, nfy_g;
  int ncx, c_row0, c_ny, ncy_g;
};
TGeom full_tgeom(int nfx, int nfy);
void launch_restrict(const cd* fine, cd* coarse, const TGeom& t, int zero_mask, cudaStream_t st);
void launch_prolong(const cd* coarse, const cd* base, cd* fine, const TGeom& t, int accumulate, cudaStream_t st);

// device-side problem setup (kernels_setup.cu; grid.py:120-160, 261-287, 309-320)
struct SetupLayers {
  int n;
  double y0[8], y1[8], v[8];
};
void launch_setup_fill(double* out, long long n, double v, cudaStream_t st);
void launch_setup_wedge(double* out, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                        const SetupLayers& L, cudaStream_t st);
void launch_setup_raster(double* out, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                         const double* g, int rnx, int rny, double rx0, double ry0, double rdx, double rdy,
                         cudaStream_t st);
void launch_setup_inject(const double* fine, int nfx, double* coarse, int ncx, int ncy, cudaStream_t st);
int setup_stats_blocks(long long n);
void launch_setup_stats(const double* a, long long n, double* part, unsigned* ticket, double* out3, cudaStream_t st);
void launch_setup_point(cd* rhs, long long n, long long idx, double v, cudaStream_t st);

// rank-count-invariant reductions: per-row partials (one block per row), then an ordered
// sum over the global rows (parallel.py:168-195)
void launch_rowdot(const cd* u, const cd* v, int nx, int ny, cd* rowpart, cudaStream_t st);
void launch_rowmgs(cd* w, const cd* vi, const cd* hsrc, const cd* vn, int nx, int ny, cd* rowpart, cudaStream_t st);
void launch_rowsubnorm(const cd* b, const cd* t, int nx, int ny, cd* rowpart, cudaStream_t st);
void launch_rowsum(const cd* rows, int nyg, cd* dst, cudaStream_t st);
void launch_dot(const cd* u, const cd* v, long long n, RedWS& ws, cd* dst, cudaStream_t st);
// epilogue of a fused MGS launch: the one-iteration FGMRES scalar update (launch_step1) run by the
// block that finishes the reduction, on (b2, h0, the launch's own result)
struct Step1Epi {
  const cd* b2;
  const cd* h0;
  cd* y;
  int* its;
  cd* flag;
};
void launch_mgs(cd* w, const cd* vi, const cd* hsrc, const cd* vn, long long n, RedWS& ws, cd* dst, cudaStream_t st,
                const Step1Epi* epi = nullptr);
// guard != null: a non-finite ||b - t||^2 raises the flag (launch_finite_guard folded in)
void launch_subnorm(const cd* b, const cd* t, long long n, RedWS& ws, cd* dst, cudaStream_t st, cd* guard = nullptr);
void launch_scale(const cd* x, cd* out, double inv, long long n, cudaStream_t st);
void launch_lincomb(const cd* const* basis, const cd* y, int m, const cd* x0, cd* x, long long n, cudaStream_t st);
void launch_add(const cd* a, const cd* b, cd* out, long long n, int sub, cudaStream_t st);
void launch_gemv(const cd* A, const cd* b, cd* x, int n, cudaStream_t st);
void launch_scale_dev(const cd* x, cd* out, const cd* nrm2, long long n, cudaStream_t st,
                      const int* skip = nullptr);  // out = x / sqrt(nrm2) (0 when the norm is 0)
void launch_step1(const cd* b2, const cd* h0, const cd* hn2, cd* y, int* its, cd* flag, cudaStream_t st);
void launch_finite_guard(const cd* v, cd* flag, cudaStream_t st);
void launch_axpy(const cd* y, cd a, const cd* x, cd* out, long long n, int sub, cudaStream_t st);
void launch_bicg_p(const cd* r, cd* p, const cd* v, cd beta, cd omega, long long n, cudaStream_t st);
void launch_pack_im(cd* dst, const cd* src, cudaStream_t st);  // dst->y = src->x
void launch_guard(const cd* post2, const cd* bn2, const cd* r02, double guard, cd* flag, cudaStream_t st);

// device-resident GMRES (kernels_resident.cu).  mode 0: one cluster, 1: whole grid
// (cooperative).  Returns nonzero when the problem does not fit that mode.
int resident_max_cap();
long long resident_cluster_points();
long long resident_grid_points();
int resident_grid_ctas();
int resident_vec_cap();
long long resident_gpart_elems();  // SmallSolve::gpart size (grid-reduction partials and sums)
void resident_set_profile(long long* dev_counters);
// one Arnoldi step's MGS chain in a cooperative launch (large levels); 1 = does not fit
// tg != null: the low-synchronisation form (two grid reductions per step) where the
// level fits it; tg holds the T = (I + L)^{-1} rows of the Arnoldi process so far
// (mgs_ls_tg_elems() elements; every step j of the process must go through it)
// fuse != null (device-driven GMRES, low-synchronisation form only: mgs_ls_fits(n, j)): the
// step also runs the Givens / stopping update of k_gm_givens on the solve's device state
struct GmFuseArgs {
  cd* st;        // gm_state_elems(cap) state of the solve
  int cap, maxit;
  double tol;
  cd* flag;
};
int launch_mgs_grid(cd* w, const cd* const* Vtab, int j, long long n, cd* gpart, cd* hout, cudaStream_t st,
                    const int* skip = nullptr, cd* tg = nullptr, const GmFuseArgs* fuse = nullptr);
bool mgs_ls_fits(long long n, int j);
// the same low-synchronisation step as streaming passes over HBM (w too large for
// the one-launch form): Vtab device pointer table, Vhost the same pointers on the
// host; part >= lsh_part_elems(n, j) elements; Tg (cap+1)(cap+2)/2; 1 = j too large
long long lsh_part_elems(long long n, int maxj);
// allreduce (may be empty): sums a device vector over the ranks of a sharded level, in place
int launch_mgs_lsh(cd* w, const cd* const* Vtab, const cd* const* Vhost, int j, long long n, cd* part, cd* Tg,
                   cd* hout, cudaStream_t st, const std::function<void(cd*, int)>& allreduce,
                   const int* skip = nullptr);  // skip: device flag of a device-driven loop (nonzero: do nothing)
// levels whose w slice does not fit the one-launch low-synchronisation step take the streaming
// form instead of the MGS-order one-launch kernels when asked to (off by default: measured equal
// or slower, engine.cu)
bool mgs_prefers_lsh(long long n, int cap);
void set_lsh_prefer(int on);
bool mgs_ls_on();
void set_mgs_ls(int on);
void set_rg_exact(int on);
bool rg_exact_on();    // separable K2 kernel: 0 tile form, 1 column-marching form (default)  // 1: radius-2/3 levels use the reference's exact tap order (HDB_RG_EXACT=1)  // runtime switch (HDB_MGS_LS=0 at start-up does the same)
long long mgs_ls_tg_elems();
bool mgs_grid_fits(long long n);
// device-driven GMRES control (launch path; kernels_resident.cu)
long long gm_state_elems(int cap);
void launch_gm_init(const cd* nn, cd* st, int cap, cd* flag, cudaStream_t s);
void launch_gm_scale(const cd* b, cd* v0, const cd* st, long long n, cudaStream_t s);
void launch_gm_givens(int j, const cd* hcol, cd* st, int cap, int maxit, double tol, cd* flag, cudaStream_t s);
void launch_gm_solve(cd* st, int cap, cudaStream_t s);
void launch_gm_final(const cd* nn, const cd* st, int cap, int* its_out, double* rel_out, cd* flag, cudaStream_t s);
const int* gm_flags(const cd* st);
cd* gm_y(cd* st, int cap);  // 8 per-phase cycle counters or null
// ortho 0: modified Gram-Schmidt (reference order), 1: CGS2 (caps <= resident_vec_cap()),
// 2: CGS + DGKS, 3: low-synchronisation MGS, 4: 3 on levels >= 131072 points, else 2
int launch_resident_gmres(int mode, int ortho, const OpCoef& c, const Geom& g, const double* ksq, const cd* b, cd* x,
                          cd* basis, cd* Rg, cd* gpart, long long n, double tol, int cap, int* its_out,
                          double* relres_out, cd* flag, cudaStream_t st);

}  // namespace hdb
