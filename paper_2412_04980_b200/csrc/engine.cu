// Engine implementation: Krylov driver, multigrid, A-DEF1 recursion.
//
// References (paths relative to /root/reference/pkg/src/helmdef/):
//   fgmres            krylov.py:61-177
//   CslpMultigrid     mg.py:51-139
//   MadpSolver        madp.py:220-371 (apply_preconditioner 301-327, _solve_cslp 277-299)
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>

#include "engine.h"

namespace hdb {

// ------------------------------------------------------------- launch accounting
const char* kfam_name(int f) {
  static const char* names[KF_COUNT] = {"apply5", "residual5", "jacobi5", "resnorm5", "galerkin", "restrict",
                                        "prolong", "mgs_coop", "mgs_chain", "blas1", "resident_gmres", "control",
                                        "gemv", "resrestrict"};
  return f >= 0 && f < KF_COUNT ? names[f] : "?";
}

double gmres_alg_bytes(long long n, int m) {
  double per = 48.0 + 16.0 * (m + 1) + 72.0;
  for (int j = 0; j < m; ++j) per += 72.0 + 16.0 * (j + 1);
  return per * (double)n;
}

cudaEvent_t KProf::get() {
  if (used == pool.size()) {
    cudaEvent_t e;
    HDB_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

void KProf::resolve() {
  if (recs.empty()) return;
  HDB_CUDA(cudaEventSynchronize(recs.back().b));
  for (const Rec& r : recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) ms[r.fam] += t;
  }
  recs.clear();
  used = 0;
}

void KProf::reset() {
  if (!recs.empty()) resolve();
  for (int f = 0; f < KF_COUNT; ++f) { bytes[f] = 0; n[f] = 0; ms[f] = 0; }
}

// ------------------------------------------------------------------ engine
static std::unique_ptr<Engine> g_engine;

void Engine::check_after(int fam) {
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess)
    throw Error(E_CUDA, std::string("after a ") + kfam_name(fam) + " launch: " + cudaGetErrorString(e));
}

Engine::Engine(int dev) : device(dev) {
  HDB_CUDA(cudaSetDevice(dev));
  const char* dbg = getenv("HDB_DEBUG_SYNC");
  debug_sync = dbg && *dbg && *dbg != '0';
  HDB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  own_st = st;
  HDB_CUDA(cudaMalloc(&red.partials, sizeof(cd) * kMaxReduceBlocks));
  HDB_CUDA(cudaMalloc(&red.ticket, sizeof(unsigned)));
  HDB_CUDA(cudaMemset(red.ticket, 0, sizeof(unsigned)));
  HDB_CUDA(cudaMalloc(&dscal, sizeof(cd) * kScal));
  HDB_CUDA(cudaMemset(dscal, 0, sizeof(cd) * kScal));
  HDB_CUDA(cudaMallocHost(&hscal, sizeof(cd) * kScal));
  std::memset(hscal, 0, sizeof(cd) * kScal);
}

Engine::~Engine() {
  cudaStreamSynchronize(st);
  for (cudaEvent_t e : kp.pool) cudaEventDestroy(e);
  if (own_st) st = own_st;
  delete comm;
  cudaFree(rowpart);
  cudaFree(rowfull);
  cudaFree(red.partials);
  cudaFree(red.big);
  cudaFree(red.ticket);
  cudaFree(dscal);
  cudaFreeHost(hscal);
  cudaStreamDestroy(st);
}

cd* Engine::alloc(long long n) { return (cd*)alloc_bytes(sizeof(cd) * (size_t)(n > 0 ? n : 1)); }

void* Engine::alloc_bytes(size_t b) {
  void* p = nullptr;
  HDB_CUDA(cudaMalloc(&p, b));
  bytes_alloc += b;
  return p;
}

void Engine::free(void* p) {
  if (p) cudaFree(p);
}

void Engine::fetch(int count) {
  syncs++;
  HDB_CUDA(cudaMemcpyAsync(hscal, dscal, sizeof(cd) * count, cudaMemcpyDeviceToHost, st));
  HDB_CUDA(cudaStreamSynchronize(st));
  // leave the flag set for inspection; solver entry points clear it
  if (hscal[kSlotFlag].x == 1.0)
    throw Error(E_MGDIV, "multigrid V-cycle residual exceeded the divergence guard (mg.py:135-138)");
  if (hscal[kSlotFlag].x == 2.0) throw Error(E_NONFINITE, "non-finite value in a device-resident Krylov solve");
}

double Engine::fetch_norm(int slot) {
  const double v = hscal[slot].x;
  return std::sqrt(v > 0.0 ? v : 0.0);
}

static thread_local Engine* t_engine = nullptr;

Engine& engine() {
  if (t_engine) return *t_engine;
  if (!g_engine) throw Error(E_ARG, "hdb_init() has not been called");
  return *g_engine;
}

void thread_engine_begin(int device) {
  if (t_engine) return;
  t_engine = new Engine(device);
}

void thread_engine_end() {
  delete t_engine;
  t_engine = nullptr;
}

void engine_init(int device) {
  if (g_engine && g_engine->device == device) return;
  g_engine.reset();
  g_engine.reset(new Engine(device));
}

bool engine_ready() { return t_engine || (bool)g_engine; }

// --------------------------------------------------------------- level op
void LevelOp::exchange(const cd* u, int rows) const {
  if (!sharded) return;
  Engine& E = engine();
  if (!E.comm) throw Error(E_ARG, "sharded level without a communicator");
  if (rows > H) throw Error(E_ARG, "halo exchange wider than the allocated halo");
  cd* v = const_cast<cd*>(u);
  const long long nx = g.nx;
  const size_t bytes = sizeof(cd) * (size_t)rows * nx;
  E.comm->exchange(v, v - rows * nx, bytes, v + (long long)(g.ny - rows) * nx, v + (long long)g.ny * nx, bytes, E.st);
}

void LevelOp::reduce(cd* slot) const {
  if (!sharded) return;
  Engine& E = engine();
  E.comm->allreduce((double*)slot, 2, E.st);
}

// ---- rank-count-invariant reductions (HDB_PINV=1 / hdb_option("pinv", 1)) ----------------
// Every reduction of a level goes through per-row partials gathered in global row order
// (kernels_blas.cu k_rowred / k_rowsum), so a solve gives the same bits on 1, 2, 4, ...
// ranks (the reference's reduce_dot contract, parallel.py:168-195).  The mode also keeps
// every level on the launch-driven Krylov path: the one-launch MGS steps and the
// device-resident solvers reduce over CTA slices that depend on the local extent.
static int g_pinv = -1;
bool pinv_mode() {
  if (g_pinv < 0) {
    const char* e = getenv("HDB_PINV");
    g_pinv = (e && atoi(e) != 0) ? 1 : 0;
  }
  return g_pinv != 0;
}
void set_pinv(int on) { g_pinv = on ? 1 : 0; }

cd* Engine::rows(int nyg) {
  if (nyg > row_cap) {
    free(rowpart);
    free(rowfull);
    row_cap = nyg;
    rowpart = alloc(row_cap);
    rowfull = alloc(row_cap);
  }
  return rowpart;
}

void LevelOp::finish_rows(cd* slot) const {
  Engine& E = engine();
  const cd* src = E.rowpart;
  if (sharded) {
    const int P = E.comm->size;
    std::vector<size_t> off(P), bytes(P);
    for (int r = 0; r < P; ++r) {
      off[r] = sizeof(cd) * (size_t)slab_row0[r];
      bytes[r] = sizeof(cd) * (size_t)slab_ny[r];
    }
    E.comm->allgatherv(E.rowpart, E.rowfull, off, bytes, E.st);
    src = E.rowfull;
  }
  E.kl(KF_BLAS, 16.0 * g.nyg, [&] { launch_rowsum(src, g.nyg, slot, E.st); });
}

void red_dot(const LevelOp* L, const cd* u, const cd* v, long long n, cd* slot) {
  Engine& E = engine();
  const double bytes = (u == v ? 16.0 : 32.0) * n;
  if (L && pinv_mode()) {
    cd* rp = E.rows(L->g.nyg);
    E.kl(KF_BLAS, bytes, [&] { launch_rowdot(u, v, L->g.nx, L->g.ny, rp, E.st); });
    L->finish_rows(slot);
    return;
  }
  E.kl(KF_BLAS, bytes, [&] { launch_dot(u, v, n, E.red, slot, E.st); });
  if (L && L->sharded) L->reduce(slot);
}

void red_mgs(const LevelOp* L, cd* w, const cd* vi, const cd* hsrc, const cd* vn, long long n, cd* slot, double bytes) {
  Engine& E = engine();
  if (L && pinv_mode()) {
    cd* rp = E.rows(L->g.nyg);
    E.kl(KF_MGS_CHAIN, bytes, [&] { launch_rowmgs(w, vi, hsrc, vn, L->g.nx, L->g.ny, rp, E.st); });
    L->finish_rows(slot);
    return;
  }
  E.kl(KF_MGS_CHAIN, bytes, [&] { launch_mgs(w, vi, hsrc, vn, n, E.red, slot, E.st); });
  if (L && L->sharded) L->reduce(slot);
}

void red_subnorm(const LevelOp* L, const cd* b, const cd* t, long long n, cd* slot) {
  Engine& E = engine();
  if (L && pinv_mode()) {
    cd* rp = E.rows(L->g.nyg);
    E.kl(KF_BLAS, 32.0 * n, [&] { launch_rowsubnorm(b, t, L->g.nx, L->g.ny, rp, E.st); });
    L->finish_rows(slot);
    return;
  }
  E.kl(KF_BLAS, 32.0 * n, [&] { launch_subnorm(b, t, n, E.red, slot, E.st); });
  if (L && L->sharded) L->reduce(slot);
}

void LevelOp::apply(const cd* u, cd* out) const {
  Engine& E = engine();
  exchange(u, c.radius);
  E.kl(c.radius == 1 ? KF_APPLY5 : KF_GALERKIN, 40.0 * n, [&] { launch_apply(c, g, u, nullptr, ksq, out, 0, E.st); });
}
void LevelOp::residual(const cd* b, const cd* u, cd* out) const {
  Engine& E = engine();
  exchange(u, c.radius);
  E.kl(c.radius == 1 ? KF_RESID5 : KF_GALERKIN, 56.0 * n, [&] { launch_apply(c, g, u, b, ksq, out, 1, E.st); });
}
void LevelOp::resnorm(const cd* b, const cd* u, cd* slot, cd* scratch) const {
  Engine& E = engine();
  exchange(u, c.radius);
  if (pinv_mode()) {  // tile partials depend on the slab: residual, then two row-ordered norms
    E.kl(c.radius == 1 ? KF_RESID5 : KF_GALERKIN, 56.0 * n, [&] { launch_apply(c, g, u, b, ksq, scratch, 1, E.st); });
    red_dot(this, scratch, scratch, n, slot);
    red_dot(this, b, b, n, E.dscal + kSlotMgB);
    E.kl(KF_BLAS, 0.0, [&] { launch_pack_im(slot, E.dscal + kSlotMgB, E.st); });
    return;
  }
  if (c.radius == 1) {
    const long long G = resnorm_partials(g);
    if (G > E.red.big_cap) {  // grows once per new largest level
      E.free(E.red.big);
      E.red.big = (cd*)E.alloc_bytes(sizeof(cd) * (size_t)G);
      E.red.big_cap = G;
    }
    E.kl(KF_RESNORM, 40.0 * n, [&] { launch_resnorm(c, g, u, b, ksq, E.red.big, slot, E.st); }, 2);
  } else {
    E.kl(KF_GALERKIN, 56.0 * n, [&] { launch_apply(c, g, u, b, ksq, scratch, 1, E.st); });
    E.kl(KF_BLAS, 32.0 * n, [&] {
      launch_dot(scratch, scratch, n, E.red, slot, E.st);
      launch_dot(b, b, n, E.red, E.dscal + kSlotMgB, E.st);
      launch_pack_im(slot, E.dscal + kSlotMgB, E.st);
    }, 3);
  }
  reduce(slot);
}
void LevelOp::jacobi(const cd* x, const cd* b, cd* out, double omega, bool from_zero) const {
  Engine& E = engine();
  if (!from_zero) exchange(x, 1);
  E.kl(KF_JACOBI, (from_zero ? 40.0 : 56.0) * n, [&] { launch_jacobi(c, g, x, b, ksq, out, omega, from_zero, E.st); });
}
bool LevelOp::jacobi_add_ok() const { return c.radius == 1 && jacobi_add_fits(g); }
void LevelOp::jacobi_add(const cd* x, const cd* b, cd* out, double omega, const cd* addt, cd* out2) const {
  Engine& E = engine();
  exchange(x, 1);
  E.kl(KF_JACOBI, 88.0 * n, [&] { launch_jacobi_add(c, g, x, b, ksq, out, omega, addt, out2, E.st); });
}

// ----------------------------------------------------------- level transfers
TGeom level_tgeom(const LevelOp& f, const LevelOp& c) {
  TGeom t;
  t.nfx = f.g.nx; t.f_row0 = f.g.row0; t.f_ny = f.g.ny; t.nfy_g = f.g.nyg;
  t.ncx = c.g.nx; t.c_row0 = c.g.row0; t.c_ny = c.g.ny; t.ncy_g = c.g.nyg;
  return t;
}

// coarse rows this rank restricts when a sharded level feeds a replicated one:
// coarse row c is centred on fine row 2c, so the rank owning fine rows [f0, f1)
// takes coarse rows [ceil(f0/2), ceil(f1/2)) -- every centre lies inside its own
// slab and the 5-tap restriction reads at most 2 rows beyond it (the exchanged
// halo).  Cut rows of the last sharded depth can be odd (P not a power of two).
void gather_rows(const std::vector<int>& fine_slab_row0, int rank, int ncy_g, int& row0, int& ny) {
  const int P = (int)fine_slab_row0.size();
  row0 = (fine_slab_row0[rank] + 1) / 2;
  const int end = rank == P - 1 ? ncy_g : (fine_slab_row0[rank + 1] + 1) / 2;
  ny = end - row0;
}
static void coarse_slab_of(const LevelOp& f, int rank, int ncy_g, int& row0, int& ny) {
  gather_rows(f.slab_row0, rank, ncy_g, row0, ny);
}

void restrict_levels(const LevelOp& f, const LevelOp& c, const cd* fine, cd* out, cd* slab, int zero_mask) {
  Engine& E = engine();
  f.exchange(fine, 2);
  if (f.sharded && !c.sharded) {
    // restrict this rank's part of the coarse grid, then gather the replicated vector
    TGeom t = level_tgeom(f, c);
    const int P = E.comm->size;
    int r0, rn;
    coarse_slab_of(f, E.comm->rank, c.g.nyg, r0, rn);
    t.c_row0 = r0;
    t.c_ny = rn;
    E.kl(KF_RESTRICT, 20.0 * f.n, [&] { launch_restrict(fine, slab, t, zero_mask, E.st); });
    std::vector<size_t> off(P), bytes(P);
    for (int r = 0; r < P; ++r) {
      int a, n;
      coarse_slab_of(f, r, c.g.nyg, a, n);
      off[r] = sizeof(cd) * (size_t)a * c.g.nx;
      bytes[r] = sizeof(cd) * (size_t)n * c.g.nx;
    }
    E.comm->allgatherv(slab, out, off, bytes, E.st);
    return;
  }
  E.kl(KF_RESTRICT, 20.0 * f.n, [&] { launch_restrict(fine, out, level_tgeom(f, c), zero_mask, E.st); });
}

void prolong_levels(const LevelOp& c, const LevelOp& f, const cd* coarse, const cd* base, cd* fine) {
  Engine& E = engine();
  c.exchange(coarse, 1);
  E.kl(KF_PROLONG, (base ? 36.0 : 20.0) * f.n,
       [&] { launch_prolong(coarse, base, fine, level_tgeom(f, c), base != nullptr, E.st); });
}

// ------------------------------------------------------------------- KWS
void KWS::ensure(long long n_, int cap_, bool flexible) {
  Engine& E = engine();
  if (n_ != n && n != 0) throw Error(E_ARG, "Krylov workspace reused with a different vector length");
  n = n_;
  if (!tmp) tmp = E.alloc_h(n, halo);
  if (cap_ + 1 > cap) {
    if (dbasis) { E.free(dbasis); E.free(dy); cudaFreeHost(hbasis); cudaFreeHost(hy); }
    cap = cap_ + 1;
    dbasis0 = nullptr;
    dbasis = (cd**)E.alloc_bytes(sizeof(cd*) * cap);
    dy = (cd*)E.alloc_bytes(sizeof(cd) * cap);
    HDB_CUDA(cudaMallocHost(&hbasis, sizeof(cd*) * cap));
    HDB_CUDA(cudaMallocHost(&hy, sizeof(cd) * cap));
  }
  (void)flexible;
}

cd* KWS::v(int i) {
  while ((int)V.size() <= i) V.push_back(engine().alloc_h(n, halo));
  return V[i];
}
cd* KWS::z(int i) {
  while ((int)Z.size() <= i) Z.push_back(engine().alloc_h(n, halo));
  return Z[i];
}

KWS::~KWS() {
  if (!engine_ready()) return;
  Engine& E = engine();
  E.free(gst);
  if (hflags) cudaFreeHost(hflags);
  if (hvtab) cudaFreeHost(hvtab);
  E.free(dV);
  E.free(gpart);
  E.free(tg);
  E.free(tgh);
  E.free(lpart);
  for (auto p : V) E.free_h(p, halo);
  for (auto p : Z) E.free_h(p, halo);
  E.free_h(tmp, halo);
  if (dbasis) { E.free(dbasis); E.free(dy); cudaFreeHost(hbasis); cudaFreeHost(hy); }
}

// ------------------------------------------------- device-resident solves
static long long env_ll(const char* name, long long dflt) {
  const char* e = getenv(name);
  return e ? atoll(e) : dflt;
}

int resident_ortho() {
  static int o = -1;
  if (o < 0) {
    // auto (default): the low-synchronisation MGS on levels >= 131072 points, CGS + DGKS
    // below (measured per level, profiles/r02m_modes.log: 513^2 54.2 vs 60.5 us/it; 257^2 ..
    // 65^2 DGKS 21-24 vs 25-29); dgks / ls force one; cgs2: always two passes; mgs: the
    // reference's order
    const char* e = getenv("HDB_ORTHO");
    const std::string v = e ? e : "auto";
    o = v == "mgs" ? 0 : v == "cgs2" ? 1 : v == "dgks" ? 2 : v == "ls" ? 3 : 4;
  }
  return o;
}

bool step1_enabled() {
  static int v = -1;
  if (v < 0) v = (int)env_ll("HDB_STEP1", 1);
  return v != 0;
}

// levels from this many points (and not sharded) take the HBM-streaming low-sync
// MGS step when the one-launch forms do not fit (HDB_LSH_N; 0 disables)
static long long lsh_min() {
  static long long v = -1;
  if (v < 0) v = env_ll("HDB_LSH_N", 1LL << 20);
  return v > 0 ? v : (1LL << 62);
}

// sharded levels with at least this many local points take the HBM-streaming low-sync
// step: two all-reduces per Arnoldi step (the 2j + 1 coefficient sums and ||w||^2) instead of
// one per MGS coefficient (HDB_LSH_SHARD_N; default 0 = every sharded level, -1 = off).
// (Round 2 kept it off for an intermittent illegal address in the one-GPU thread-rank
// emulation; the cause was not this step but the radius-2/3 tile loaders, which sampled
// rows beyond a slab's halo when the slab height is not a multiple of the tile height --
// fixed in stencil.cuh tile_row_needed, 14 / 14 stress runs clean, profiles/r03r_*.)
static long long lsh_shard_min() {
  static long long v = -2;
  if (v == -2) v = env_ll("HDB_LSH_SHARD_N", 0);
  return v < 0 ? (1LL << 62) : v;
}

// Levels whose w slice does not fit the one-launch low-synchronisation step (> 7168 points per
// CTA) CAN take the HBM-streaming form of the same algorithm instead of the MGS-order one-launch
// kernels (hdb_option("lsh_prefer", 1) / HDB_LSH_PREFER=1; host-driven and device-driven loops).
// Off by default: measured equal on config 5's 2049^2 level (2.59 vs 2.58 s of MGS time per
// solve) and slower on config 4's 3065 x 1001 level (9.9 vs 9.1 s) -- two passes over the basis
// at ~0.9 of the copy peak move as many bytes per unit time as one pass with j + 2 grid
// barriers (profiles/r03f_bench_*.json vs r03d_bench_*.json).
static int g_lsh_prefer = -1;
void set_lsh_prefer(int on) { g_lsh_prefer = on ? 1 : 0; }
bool mgs_prefers_lsh(long long n, int cap) {
  if (g_lsh_prefer < 0) {
    const char* e = getenv("HDB_LSH_PREFER");
    g_lsh_prefer = (e && atoi(e) != 0) ? 1 : 0;
  }
  return g_lsh_prefer && mgs_ls_on() && n >= lsh_min() && cap <= 511 && !mgs_ls_fits(n, 0);
}

long long coop_mgs_min() {
  static long long v = -1;
  if (v < 0) v = env_ll("HDB_COOP_MGS_N", 2000);  // (config 3 @40 Hz: 1018 -> 997 ms vs 150000)
  return v > 0 ? v : (1LL << 62);
}

int resident_mode(long long n, int cap) {
  if (pinv_mode()) return -1;
  static long long small = -1, grid = -1;
  if (small < 0) {
    // cluster mode only when asked: the grid mode is faster at every config-2 level since
    // r02i (65^2: 20.8 vs 22.7 us/it; 129^2: 21.9 vs 37.9 -- profiles/r02i_modes.log)
    small = std::min(env_ll("HDB_SMALL_N", 0), resident_cluster_points());
    grid = std::min(env_ll("HDB_GRID_N", 2000000), resident_grid_points());
  }
  if (cap > resident_max_cap()) return -1;
  if (n <= small) return 0;
  if (n <= grid) return 1;
  return -1;
}

void SmallSolve::ensure(const LevelOp* o, int cap_) {
  if (op == o && cap >= cap_) return;
  Engine& E = engine();
  E.free(basis);
  E.free(Rg);
  E.free(gpart);
  op = o;
  cap = cap_;
  basis = E.alloc((long long)(cap + 1) * o->n);
  Rg = E.alloc((long long)cap * (cap + 1) / 2 + cap + (long long)(cap + 1) * (cap + 2) / 2);
  gpart = E.alloc(resident_gpart_elems());
  HDB_CUDA(cudaMemsetAsync(gpart, 0, sizeof(cd) * (size_t)resident_gpart_elems(), E.st));
}

bool SmallSolve::try_run(const cd* b, cd* x, Stop stop, int* its_dev, double* rel_dev) {
  Engine& E = engine();
  const int mode = resident_mode(op->n, stop.max_iters);
  if (mode < 0) return false;
  int rc = 0;
  E.kl(KF_RESIDENT, 0.0, [&] {
    rc = launch_resident_gmres(mode, resident_ortho(), op->c, op->g, op->ksq, b, x, basis, Rg, gpart, op->n,
                               stop.rel_tol, stop.max_iters, its_dev, rel_dev, E.dscal + kSlotFlag, E.st);
  });
  if (rc != 0) {
    E.launches--;
    E.kp.n[KF_RESIDENT]--;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw Error(E_CUDA, std::string("device-resident GMRES launch: ") + cudaGetErrorString(err));
    return false;  // does not fit the resident working set: caller uses the launch path
  }
  return true;
}

SmallSolve::~SmallSolve() {
  if (!engine_ready()) return;
  Engine& E = engine();
  E.free(basis);
  E.free(Rg);
  E.free(gpart);
}



// ----------------------------------------------------------------- FGMRES
static const double kHappy = 1e-30;  // krylov.py:28

KReport fgmres(long long n, const LinOp& A, const LinOp* M, const cd* b, cd* x, Stop stop, KWS& ws,
               const std::function<void(int, double)>* hook, const cd* x0, const LevelOp* dist) {
  const bool shard = dist && dist->sharded;
  const bool pinv = dist && pinv_mode();
  Engine& E = engine();
  if (stop.max_iters < 1) throw Error(E_ARG, "max_iters must be >= 1");
  if (stop.max_iters + kSlotH + 2 >= 900) throw Error(E_ARG, "Krylov iteration cap too large (max 896)");
  ws.ensure(n, stop.max_iters, M != nullptr);
  KReport rep;

  red_dot(dist, b, b, n, E.dscal + kSlotH);
  E.fetch(kSlotH + 1);
  const double bnorm = E.fetch_norm(kSlotH);
  auto copy_x0 = [&] {
    if (x0) HDB_CUDA(cudaMemcpyAsync(x, x0, sizeof(cd) * n, cudaMemcpyDeviceToDevice, E.st));
    else HDB_CUDA(cudaMemsetAsync(x, 0, sizeof(cd) * n, E.st));
  };
  // r0 = b - A x0 (krylov.py:92-95); zero guess: r0 = b
  const cd* r0 = b;
  double beta = bnorm;
  if (x0) {
    A(x0, ws.tmp);
    E.kl(KF_BLAS, 48.0 * n, [&] { launch_add(b, ws.tmp, ws.tmp, n, 1, E.st); });
    red_dot(dist, ws.tmp, ws.tmp, n, E.dscal + kSlotH);
    r0 = ws.tmp;
  }
  if (bnorm == 0.0) {  // krylov.py:96-97
    copy_x0();
    rep.history = {0.0};
    rep.converged = true;
    return rep;
  }
  if (x0) {
    E.fetch(kSlotH + 1);
    beta = E.fetch_norm(kSlotH);
  }
  double rel = beta / bnorm;
  rep.history.push_back(rel);
  if (rel <= stop.rel_tol && stop.rel_tol < 1.0) {
    copy_x0();
    rep.final_relres = rel;
    rep.converged = true;
    return rep;
  }
  if (!std::isfinite(beta)) throw Error(E_NONFINITE, "initial residual is not finite");

  E.kl(KF_BLAS, 32.0 * n, [&] { launch_scale(r0, ws.v(0), 1.0 / beta, n, E.st); });  // V0 = r0 / beta

  std::vector<std::vector<cplx>> R;
  std::vector<double> cs;
  std::vector<cplx> sn, g;
  g.push_back(cplx(beta, 0.0));
  int its = 0;
  bool conv = false;
  bool ls_ok = true, lsh_ok = true;
  for (int j = 0; j < stop.max_iters; ++j) {
    const cd* z = ws.v(j);
    if (M) {
      (*M)(ws.v(j), ws.z(j));
      z = ws.z(j);
    }
    cd* w = ws.v(j + 1);
    A(z, w);
    // MGS chain (krylov.py:121-124): one cooperative launch on large levels,
    // else one fused launch per coefficient
    bool coop = false;
    auto ensure_dv = [&] {
      if (ws.dV_cap < j + 1) {
        E.sync();  // copies from the old pinned mirror may still be pending
        E.free(ws.dV);
        if (ws.hvtab) cudaFreeHost(ws.hvtab);
        ws.dV_cap = std::max(2 * (j + 1), 64);
        ws.dV = (cd**)E.alloc_bytes(sizeof(cd*) * ws.dV_cap);
        HDB_CUDA(cudaMallocHost(&ws.hvtab, sizeof(cd*) * ws.dV_cap));
        ws.dV_n = 0;
      }
      // append V pointers (their addresses never change) through a pinned mirror: an
      // asynchronous copy from ws.V itself could read storage a later push_back frees
      while (ws.dV_n < j + 1) {
        ws.hvtab[ws.dV_n] = ws.v(ws.dV_n);  // (allocates the vector if it does not exist yet)
        HDB_CUDA(cudaMemcpyAsync(ws.dV + ws.dV_n, ws.hvtab + ws.dV_n, sizeof(cd*), cudaMemcpyHostToDevice, E.st));
        ws.dV_n++;
      }
    };
    if (!shard && !pinv && n >= coop_mgs_min() && !mgs_prefers_lsh(n, stop.max_iters)) {
      if (!ws.gpart) ws.gpart = E.alloc(2LL * resident_grid_ctas() * (resident_vec_cap() + 1) + 2LL * (resident_vec_cap() + 1));
      if (!ws.tg) ws.tg = E.alloc(mgs_ls_tg_elems());
      ensure_dv();
      // the low-synchronisation step needs every earlier step of this Arnoldi process in it
      if (j == 0) ls_ok = true;
      const bool use_ls = ls_ok && mgs_ls_fits(n, j);
      ls_ok = use_ls;
      E.kl(KF_MGS_COOP, (16.0 * (j + 1) + 32.0) * n, [&] {
        coop = launch_mgs_grid(w, (const cd* const*)ws.dV, j, n, ws.gpart, E.dscal + kSlotH, E.st, nullptr,
                               use_ls ? ws.tg : nullptr) == 0;
      });
      if (!coop) {  // did not fit or could not be co-scheduled: clear the error, use the chain
        cudaGetLastError();
        ls_ok = false;
        E.launches--;
        E.kp.n[KF_MGS_COOP]--;
        E.kp.bytes[KF_MGS_COOP] -= (16.0 * (j + 1) + 32.0) * n;
      }
    }
    // large unsharded levels: the low-synchronisation step as HBM streaming passes (every
    // step of this Arnoldi process must use it: the T rows accumulate)
    // sharded levels take it at any size: two all-reduces per Arnoldi step (the (2j+1)
    // coefficient sums and ||w||^2) instead of one per MGS coefficient
    bool lsh = false;
    if (!coop && !pinv && ((shard && n >= lsh_shard_min()) || (!shard && n >= lsh_min())) && mgs_ls_on() &&
        (j == 0 || lsh_ok) &&
        stop.max_iters <= 511) {
      if (ws.tgh_cap < stop.max_iters) {
        E.free(ws.tgh);
        E.free(ws.lpart);
        ws.tgh = E.alloc((long long)(stop.max_iters + 1) * (stop.max_iters + 2) / 2);
        ws.lpart = E.alloc(lsh_part_elems(n, stop.max_iters));
        ws.tgh_cap = stop.max_iters;
      }
      ensure_dv();
      const int nl = (j == 0 ? 1 : (j + 7) / 8) + (j + 8) / 8 + 2;
      int rc = 0;
      std::function<void(cd*, int)> allred;
      if (shard) allred = [&](cd* v, int m) { E.comm->allreduce((double*)v, 2 * m, E.st); };
      E.kl(KF_MGS_CHAIN, (16.0 * (j + 1) + 32.0) * n, [&] {
        rc = launch_mgs_lsh(w, (const cd* const*)ws.dV, ws.V.data(), j, n, ws.lpart, ws.tgh, E.dscal + kSlotH, E.st,
                            allred);
      }, nl);
      lsh = rc == 0;
    }
    lsh_ok = lsh;
    if (!coop && !lsh) {  // the fused MGS chain (algorithmic bytes booked: w + V_0, then each V_i, w out)
      red_mgs(dist, w, nullptr, nullptr, ws.v(0), n, E.dscal + kSlotH, 32.0 * n);
      for (int i = 0; i < j; ++i)
        red_mgs(dist, w, ws.v(i), E.dscal + kSlotH + i, ws.v(i + 1), n, E.dscal + kSlotH + i + 1, 16.0 * n);
      red_mgs(dist, w, ws.v(j), E.dscal + kSlotH + j, nullptr, n, E.dscal + kSlotH + j + 1, 16.0 * n);
    }
    E.fetch(kSlotH + j + 2);
    std::vector<cplx> col(j + 2);
    for (int i = 0; i <= j; ++i) col[i] = cplx(E.hscal[kSlotH + i].x, E.hscal[kSlotH + i].y);
    const double hn = E.fetch_norm(kSlotH + j + 1);
    col[j + 1] = cplx(hn, 0.0);
    for (int i = 0; i < j + 2; ++i)
      if (!std::isfinite(col[i].real()) || !std::isfinite(col[i].imag()))
        throw Error(E_NONFINITE, "non-finite Hessenberg entries");
    // apply previous rotations, form the new one (krylov.py:130-148)
    for (int i = 0; i < j; ++i) {
      const cplx t = cs[i] * col[i] + sn[i] * col[i + 1];
      col[i + 1] = -std::conj(sn[i]) * col[i] + cs[i] * col[i + 1];
      col[i] = t;
    }
    const cplx h1 = col[j], h2 = col[j + 1];
    double c;
    cplx s;
    if (std::abs(h2) == 0.0) {
      c = 1.0; s = cplx(0.0, 0.0);
    } else if (std::abs(h1) == 0.0) {
      c = 0.0; s = cplx(1.0, 0.0);
    } else {
      const double t = std::hypot(std::abs(h1), std::abs(h2));
      c = std::abs(h1) / t;
      s = (h1 / std::abs(h1)) * std::conj(h2) / t;
    }
    cs.push_back(c);
    sn.push_back(s);
    col[j] = c * h1 + s * h2;
    R.emplace_back(col.begin(), col.begin() + j + 1);
    g.push_back(-std::conj(s) * g[j]);
    g[j] = c * g[j];
    its = j + 1;
    rel = std::abs(g[j + 1]) / bnorm;
    rep.history.push_back(rel);
    if (hook) (*hook)(its, rel);
    if (hn < kHappy || rel <= stop.rel_tol) {
      conv = true;
      break;
    }
    if (!coop)  // the cooperative MGS already wrote V_{j+1} = w / hnext
      E.kl(KF_BLAS, 32.0 * n, [&] { launch_scale(w, w, 1.0 / hn, n, E.st); });
  }
  // least squares R y = g (krylov.py:161-168), solution update (169-172)
  const int m = its;
  std::vector<cplx> y(m);
  for (int i = m - 1; i >= 0; --i) {
    cplx acc = g[i];
    for (int k = i + 1; k < m; ++k) acc -= R[k][i] * y[k];
    y[i] = acc / R[i][i];
  }
  for (int i = 0; i < m; ++i) {
    ws.hbasis[i] = M ? ws.z(i) : ws.v(i);
    ws.hy[i] = mkc(y[i].real(), y[i].imag());
  }
  ws.dbasis0 = nullptr;  // (the one-step path's cached table entry is overwritten)
  HDB_CUDA(cudaMemcpyAsync(ws.dbasis, ws.hbasis, sizeof(cd*) * m, cudaMemcpyHostToDevice, E.st));
  HDB_CUDA(cudaMemcpyAsync(ws.dy, ws.hy, sizeof(cd) * m, cudaMemcpyHostToDevice, E.st));
  E.kl(KF_BLAS, 16.0 * (m + 1 + (x0 ? 1 : 0)) * n, [&] { launch_lincomb(ws.dbasis, ws.dy, m, x0, x, n, E.st); });
  // explicit true residual (krylov.py:174)
  A(x, ws.tmp);
  red_subnorm(dist, b, ws.tmp, n, E.dscal + kSlotH);
  E.fetch(kSlotH + 1);
  const double fin = E.fetch_norm(kSlotH) / bnorm;
  if (!std::isfinite(fin)) throw Error(E_NONFINITE, "non-finite solution");
  rep.iterations = m;
  rep.final_relres = fin;
  rep.converged = conv;
  return rep;
}

// --------------------------------------------- device-driven GMRES (launch path)
static bool gmres_device_enabled() {
  static int v = -1;
  if (v < 0) v = (int)env_ll("HDB_GMRES_DEV", 1);
  return v != 0;
}

// make V_0..V_upto exist and their pointers visible in the device table ws.dV
static void ensure_vtab(KWS& ws, int upto) {
  Engine& E = engine();
  ws.v(upto);
  if (ws.dV_cap < upto + 1) {
    E.sync();  // copies from the old pinned mirror may still be pending
    E.free(ws.dV);
    if (ws.hvtab) cudaFreeHost(ws.hvtab);
    ws.dV_cap = std::max(2 * (upto + 1), 64);
    ws.dV = (cd**)E.alloc_bytes(sizeof(cd*) * ws.dV_cap);
    HDB_CUDA(cudaMallocHost(&ws.hvtab, sizeof(cd*) * ws.dV_cap));
    ws.dV_n = 0;
  }
  if (ws.dV_n < upto + 1) {  // pinned mirror: the copy stays asynchronous, its source stays valid
    for (int i = ws.dV_n; i <= upto; ++i) ws.hvtab[i] = ws.V[i];
    HDB_CUDA(cudaMemcpyAsync(ws.dV + ws.dV_n, ws.hvtab + ws.dV_n, sizeof(cd*) * (upto + 1 - ws.dV_n),
                             cudaMemcpyHostToDevice, E.st));
    ws.dV_n = upto + 1;
  }
}

bool gmres_device(const LevelOp* op, const cd* b, cd* x, Stop stop, KWS& ws, int* its_dev, double* rel_dev) {
  const long long n = op->n;
  const int cap = stop.max_iters;
  // Sharded levels qualify through the streaming low-synchronisation step: its two reductions are
  // all-reduced in-stream (NCCL), the halo exchange precedes every stencil, the Givens / stopping
  // kernels run redundantly on every rank (identical all-reduced inputs -> identical flags), so a
  // sharded CSLP-GMRES also runs without a host round trip per Arnoldi step (HDB_GMRES_DEV_SHARD=0:
  // host-driven loop).  A finished solve skips its kernels; the collectives of the surplus steps
  // of a batch still run on every rank (same sequence everywhere).
  const bool shard = op->sharded;
  static const bool shard_ok = env_ll("HDB_GMRES_DEV_SHARD", 1) != 0;
  const bool lsh = shard ? (shard_ok && mgs_ls_on() && n >= lsh_shard_min() && cap <= 511)
                         : mgs_prefers_lsh(n, cap);  // streaming step instead of the one-launch kernels
  if (!gmres_device_enabled() || pinv_mode() || (shard && !lsh) || (!shard && n < coop_mgs_min()) || cap < 1 ||
      cap + kSlotH + 2 >= 900 || !(stop.rel_tol < 1.0) || !(lsh || mgs_grid_fits(n)))
    return false;
  Engine& E = engine();
  std::function<void(cd*, int)> allred;
  if (shard) allred = [&E](cd* v, int m) { E.comm->allreduce((double*)v, 2 * m, E.st); };
  ws.ensure(n, cap, false);
  if (lsh && ws.tgh_cap < cap) {
    E.free(ws.tgh);
    E.free(ws.lpart);
    ws.tgh = E.alloc((long long)(cap + 1) * (cap + 2) / 2);
    ws.lpart = E.alloc(lsh_part_elems(n, cap));
    ws.tgh_cap = cap;
  }
  if (!ws.gpart) ws.gpart = E.alloc(2LL * resident_grid_ctas() * (resident_vec_cap() + 1) + 2LL * (resident_vec_cap() + 1));
  if (!ws.tg) ws.tg = E.alloc(mgs_ls_tg_elems());
  if (ws.gst_cap < cap) {
    E.free(ws.gst);
    ws.gst = E.alloc(gm_state_elems(cap));
    ws.gst_cap = cap;
  }
  if (!ws.hflags) HDB_CUDA(cudaMallocHost(&ws.hflags, 4 * sizeof(int)));
  cd* st = ws.gst;
  const int lay = ws.gst_cap;
  const int* skip = gm_flags(st);
  cd* hcol = E.dscal + kSlotH;
  cd* flag = E.dscal + kSlotFlag;
  ensure_vtab(ws, 0);
  E.kl(KF_BLAS, 16.0 * n, [&] { launch_dot(b, b, n, E.red, hcol, E.st); });
  op->reduce(hcol);
  E.kl(KF_CONTROL, 0.0, [&] { launch_gm_init(hcol, st, lay, flag, E.st); });
  E.kl(KF_BLAS, 32.0 * n, [&] { launch_gm_scale(b, ws.v(0), st, n, E.st); });  // krylov.py:92-115 with x0 = 0
  OpCoef cs = op->c;
  cs.skip = skip;
  // first batch: one short of the previous solve's count (the counts of one
  // level's CSLP solves are close), then small batches until the flag is up
  int batch = ws.last_its > 1 ? ws.last_its - 1 : 4;
  int j = 0;
  for (;;) {
    const int jend = std::min(cap, j + batch);
    ensure_vtab(ws, jend);
    for (; j < jend; ++j) {
      // bytes are booked after the loop for the steps that ran (later ones return at once)
      op->exchange(ws.v(j), op->c.radius);
      E.kl(op->c.radius == 1 ? KF_APPLY5 : KF_GALERKIN, 0.0,
           [&] { launch_apply(cs, op->g, ws.v(j), nullptr, op->ksq, ws.v(j + 1), 0, E.st); });  // krylov.py:119
      int rc = 0;
      bool givens_fused = false;
      if (lsh) {
        const int nl = (j == 0 ? 1 : (j + 7) / 8) + (j + 8) / 8 + 3;
        E.kl(KF_MGS_CHAIN, 0.0, [&] {
          rc = launch_mgs_lsh(ws.v(j + 1), (const cd* const*)ws.dV, ws.V.data(), j, n, ws.lpart, ws.tgh, hcol, E.st,
                              allred, skip);
          launch_scale_dev(ws.v(j + 1), ws.v(j + 1), hcol + j + 1, n, E.st, skip);  // V_{j+1} = w / ||w||
        }, nl);
      } else {
        // low-synchronisation one-launch step: the Givens / stopping update rides in its tail
        // (HDB_LS_GIVENS=0: separate one-warp kernel)
        static const bool fuse_on = env_ll("HDB_LS_GIVENS", 1) != 0;
        givens_fused = fuse_on && mgs_ls_fits(n, j);
        GmFuseArgs fa{st, lay, cap, stop.rel_tol, flag};
        E.kl(KF_MGS_COOP, 0.0, [&] {
          rc = launch_mgs_grid(ws.v(j + 1), (const cd* const*)ws.dV, j, n, ws.gpart, hcol, E.st, skip, ws.tg,
                               givens_fused ? &fa : nullptr);
        });
      }
      if (rc != 0) {
        const cudaError_t err = cudaGetLastError();
        throw Error(E_CUDA, std::string("cooperative MGS launch: ") + cudaGetErrorString(err));
      }
      if (!givens_fused)
        E.kl(KF_CONTROL, 0.0, [&] { launch_gm_givens(j, hcol, st, lay, cap, stop.rel_tol, flag, E.st); });
    }
    HDB_CUDA(cudaMemcpyAsync(ws.hflags, skip, 2 * sizeof(int), cudaMemcpyDeviceToHost, E.st));
    HDB_CUDA(cudaStreamSynchronize(E.st));
    E.syncs++;
    if (ws.hflags[0] || j >= cap) break;
    batch = 3;
  }
  const int its = ws.hflags[1];
  for (int q = 0; q < its; ++q) {
    E.kp.bytes[op->c.radius == 1 ? KF_APPLY5 : KF_GALERKIN] += 40.0 * n;
    E.kp.bytes[lsh ? KF_MGS_CHAIN : KF_MGS_COOP] += (16.0 * (q + 1) + 32.0) * n + (lsh ? 32.0 * n : 0.0);
  }
  if (its == 0) {
    HDB_CUDA(cudaMemsetAsync(x, 0, sizeof(cd) * n, E.st));  // b = 0 (or non-finite ||b||: flag raised)
  } else {
    E.kl(KF_CONTROL, 0.0, [&] { launch_gm_solve(st, lay, E.st); });  // krylov.py:161-168
    E.kl(KF_BLAS, 16.0 * (its + 1) * n,
         [&] { launch_lincomb((const cd* const*)ws.dV, gm_y(st, lay), its, nullptr, x, n, E.st); });  // 169-172
    op->apply(x, ws.tmp);                                                                           // 174
    E.kl(KF_BLAS, 32.0 * n, [&] { launch_subnorm(b, ws.tmp, n, E.red, hcol, E.st); });
    op->reduce(hcol);
  }
  E.kl(KF_CONTROL, 0.0, [&] { launch_gm_final(hcol, st, lay, its_dev, rel_dev, flag, E.st); });
  ws.last_its = its;
  return true;
}

// ------------------------------------------------------ one-step FGMRES
// device scalar slots of the step: 5 per level (nested steps at deeper levels run
// inside M and must not overwrite this level's scalars), above any Hessenberg column
constexpr int kS1Base = 900;

void fgmres_step1(long long n, const LinOp& A, const LinOp& M, const cd* b, cd* x, KWS& ws, int* its_dev,
                  const LevelOp* dist, int level) {
  Engine& E = engine();
  if (level < 1 || kS1Base + 5 * level + 4 >= kSlotMgR0) throw Error(E_ARG, "one-step FGMRES level out of range");
  const int kS1B = kS1Base + 5 * level, kS1H0 = kS1B + 1, kS1HN = kS1B + 2, kS1Y = kS1B + 3, kS1F = kS1B + 4;
  ws.ensure(n, 1, true);
  cd* S = E.dscal;
  red_dot(dist, b, b, n, S + kS1B);  // ||b||^2 (krylov.py:92)
  E.kl(KF_BLAS, 32.0 * n, [&] { launch_scale_dev(b, ws.v(0), S + kS1B, n, E.st); });  // V0 = r0 / beta
  M(ws.v(0), ws.z(0));
  cd* w = ws.v(1);
  A(ws.z(0), w);
  red_mgs(dist, w, nullptr, nullptr, ws.v(0), n, S + kS1H0, 32.0 * n);
  // where the reductions finish on this rank (no all-reduce, no row-ordered mode) the scalar
  // update and the finiteness guard ride in the launch that produces their input: the block
  // that finishes the reduction runs them (same operations; HDB_STEP1_FUSE=0: separate kernels)
  static const bool fuse_on = env_ll("HDB_STEP1_FUSE", 1) != 0;
  const bool local = fuse_on && !(dist && dist->sharded) && !(dist && pinv_mode());
  if (local) {
    const Step1Epi epi{S + kS1B, S + kS1H0, S + kS1Y, its_dev, S + kSlotFlag};
    E.kl(KF_MGS_CHAIN, 16.0 * n,
         [&] { launch_mgs(w, ws.v(0), S + kS1H0, nullptr, n, E.red, S + kS1HN, E.st, &epi); });
  } else {
    red_mgs(dist, w, ws.v(0), S + kS1H0, nullptr, n, S + kS1HN, 16.0 * n);
    E.kl(KF_CONTROL, 0.0, [&] { launch_step1(S + kS1B, S + kS1H0, S + kS1HN, S + kS1Y, its_dev, S + kSlotFlag, E.st); });
  }
  if (ws.dbasis0 != ws.z(0)) {  // the one-entry pointer table of x = y0 Z0 is constant across calls
    ws.hbasis[0] = ws.z(0);
    HDB_CUDA(cudaMemcpyAsync(ws.dbasis, ws.hbasis, sizeof(cd*), cudaMemcpyHostToDevice, E.st));
    ws.dbasis0 = ws.z(0);
  }
  E.kl(KF_BLAS, 32.0 * n, [&] { launch_lincomb(ws.dbasis, S + kS1Y, 1, nullptr, x, n, E.st); });  // x = y0 Z0
  // explicit true residual: only its finiteness matters to the caller (krylov.py:174-176)
  A(x, ws.tmp);
  if (local) {
    E.kl(KF_BLAS, 32.0 * n, [&] { launch_subnorm(b, ws.tmp, n, E.red, S + kS1F, E.st, S + kSlotFlag); });
  } else {
    red_subnorm(dist, b, ws.tmp, n, S + kS1F);
    E.kl(KF_CONTROL, 0.0, [&] { launch_finite_guard(S + kS1F, S + kSlotFlag, E.st); });
  }
}

// --------------------------------------------------------------- Bi-CGSTAB
void BWS::ensure(long long n_) {
  if (n == n_ && r) return;
  Engine& E = engine();
  if (r) throw Error(E_ARG, "Bi-CGSTAB workspace reused with a different vector length");
  n = n_;
  for (cd** q : {&r, &rhat, &p, &v, &s, &t, &ph, &sh, &tmp}) *q = E.alloc_h(n, halo);
}
BWS::~BWS() {
  if (!engine_ready() || !r) return;
  Engine& E = engine();
  for (cd* q : {r, rhat, p, v, s, t, ph, sh, tmp}) E.free_h(q, halo);
}

KReport bicgstab(long long n, const LinOp& A, const LinOp* M, const cd* b, cd* x, Stop stop, BWS& ws,
                 const cd* x0, const LevelOp* dist, bool* breakdown, std::string* why) {
  Engine& E = engine();
  ws.ensure(n);
  *breakdown = false;
  auto dotv = [&](const cd* u, const cd* w) {  // conj-dot to the host (one sync)
    red_dot(dist, u, w, n, E.dscal + kSlotH);
    E.fetch(kSlotH + 1);
    return cplx(E.hscal[kSlotH].x, E.hscal[kSlotH].y);
  };
  auto nrm = [&](const cd* u) { return std::sqrt(std::max(dotv(u, u).real(), 0.0)); };
  const size_t bytes = sizeof(cd) * n;
  KReport rep;
  const double bnorm = nrm(b);
  if (x0) {
    HDB_CUDA(cudaMemcpyAsync(x, x0, bytes, cudaMemcpyDeviceToDevice, E.st));
    A(x0, ws.tmp);
    E.kl(KF_BLAS, 48.0 * n, [&] { launch_add(b, ws.tmp, ws.r, n, 1, E.st); });
  } else {
    HDB_CUDA(cudaMemsetAsync(x, 0, bytes, E.st));
    HDB_CUDA(cudaMemcpyAsync(ws.r, b, bytes, cudaMemcpyDeviceToDevice, E.st));
  }
  if (bnorm == 0.0) {  // krylov.py:203-204
    rep.history = {0.0};
    rep.converged = true;
    return rep;
  }
  double rel = nrm(ws.r) / bnorm;
  rep.history.push_back(rel);
  if (rel <= stop.rel_tol && stop.rel_tol < 1.0) {
    rep.final_relres = rel;
    rep.converged = true;
    return rep;
  }
  HDB_CUDA(cudaMemcpyAsync(ws.rhat, ws.r, bytes, cudaMemcpyDeviceToDevice, E.st));
  HDB_CUDA(cudaMemsetAsync(ws.v, 0, bytes, E.st));
  HDB_CUDA(cudaMemsetAsync(ws.p, 0, bytes, E.st));
  cplx rho(1.0, 0.0), alpha(1.0, 0.0), omega(1.0, 0.0);
  const double eps = 1e-30;  // krylov.py:28
  int its = 0;
  bool conv = false;
  auto brk = [&](const char* m) {
    *breakdown = true;
    *why = m;
    rep.iterations = its;
    rep.final_relres = rep.history.back();
    rep.converged = false;
  };
  for (int it = 1; it <= stop.max_iters; ++it) {
    const cplx rho_new = dotv(ws.rhat, ws.r);
    if (std::abs(rho_new) < eps * bnorm * bnorm) { brk("rho vanished in Bi-CGSTAB"); return rep; }
    const cplx beta = (rho_new / rho) * (alpha / omega);
    E.kl(KF_BLAS, 64.0 * n, [&] {
      launch_bicg_p(ws.r, ws.p, ws.v, mkc(beta.real(), beta.imag()), mkc(omega.real(), omega.imag()), n, E.st);
    });
    const cd* phat = ws.p;
    if (M) { (*M)(ws.p, ws.ph); phat = ws.ph; }
    A(phat, ws.v);
    const cplx denom = dotv(ws.rhat, ws.v);
    if (std::abs(denom) < eps * bnorm * bnorm) { brk("alpha denominator vanished in Bi-CGSTAB"); return rep; }
    alpha = rho_new / denom;
    E.kl(KF_BLAS, 96.0 * n, [&] {
      launch_axpy(ws.r, mkc(alpha.real(), alpha.imag()), ws.v, ws.s, n, 1, E.st);  // s = r - alpha v
      launch_axpy(x, mkc(alpha.real(), alpha.imag()), phat, x, n, 0, E.st);        // x = x + alpha phat
    }, 2);
    its = it;
    const double srel = nrm(ws.s) / bnorm;
    if (srel <= stop.rel_tol) {
      rep.history.push_back(srel);
      conv = true;
      break;
    }
    const cd* shat = ws.s;
    if (M) { (*M)(ws.s, ws.sh); shat = ws.sh; }
    A(shat, ws.t);
    const cplx tt = dotv(ws.t, ws.t);
    if (std::abs(tt) < eps) { brk("omega denominator vanished in Bi-CGSTAB"); return rep; }
    omega = dotv(ws.t, ws.s) / tt;
    if (std::abs(omega) < eps) { brk("omega vanished in Bi-CGSTAB"); return rep; }
    E.kl(KF_BLAS, 96.0 * n, [&] {
      launch_axpy(x, mkc(omega.real(), omega.imag()), shat, x, n, 0, E.st);     // x = x + omega shat
      launch_axpy(ws.s, mkc(omega.real(), omega.imag()), ws.t, ws.r, n, 1, E.st);  // r = s - omega t
    }, 2);
    rel = nrm(ws.r) / bnorm;
    rep.history.push_back(rel);
    if (!std::isfinite(rel)) throw Error(E_NONFINITE, "non-finite residual in Bi-CGSTAB");
    if (rel <= stop.rel_tol) {
      conv = true;
      break;
    }
    rho = rho_new;
  }
  A(x, ws.tmp);  // final true residual (krylov.py:275)
  red_subnorm(dist, b, ws.tmp, n, E.dscal + kSlotH);
  E.fetch(kSlotH + 1);
  rep.iterations = its;
  rep.final_relres = E.fetch_norm(kSlotH) / bnorm;
  rep.converged = conv;
  return rep;
}

// -------------------------------------------------------------- multigrid
static int dirichlet_mask(const OpCoef& c) {
  int m = 0;
  for (int s = 0; s < 4; ++s)
    if (c.bc[s] == HDB_BC_DIRICHLET) m |= 1 << s;
  return m;
}

void Multigrid::setup() {
  Engine& E = engine();
  const int L = (int)ops.size();
  for (auto v : {&X, &Y, &R, &B, &O, &S}) v->assign(L, nullptr);
  for (int i = 0; i < L; ++i) {
    const long long n = ops[i]->n, h = ops[i]->halo_elems();
    if (i < L - 1) { X[i] = E.alloc_h(n, h); Y[i] = E.alloc_h(n, h); R[i] = E.alloc_h(n, h); }
    if (i > 0) {
      B[i] = E.alloc_h(n, h);
      O[i] = E.alloc_h(n, h);
      if (ops[i - 1]->sharded && !ops[i]->sharded) S[i] = E.alloc(n);  // local part before the gather
    }
  }
  if (!R[0]) R[0] = E.alloc_h(ops[0]->n, ops[0]->halo_elems());
}

Multigrid::~Multigrid() {
  if (!engine_ready()) return;
  Engine& E = engine();
  for (size_t i = 0; i < ops.size() && i < X.size(); ++i) {
    const long long h = ops[i]->halo_elems();
    for (auto v : {&X, &Y, &R, &B, &O}) E.free_h((*v)[i], h);
    E.free(S[i]);
  }
  E.free(Ainv);
}

// mg.py:111-123.  Input x is the zero vector at every level (vcycle starts
// from x0 = 0 and the recursion passes zeros), so the first pre-smoothing
// sweep is the closed form (w D^-1) b.  The result is written to x.
void Multigrid::cycle(int i, const cd* b, cd* x, const cd* x_init, const cd* addt, cd* xsum) {
  Engine& E = engine();
  const int L = (int)ops.size();
  if (i == L - 1) {  // mg.py:104-109
    if (Ainv) {
      E.kl(KF_GEMV, 16.0 * ninv * (double)ninv + 32.0 * ninv, [&] { launch_gemv(Ainv, b, x, ninv, E.st); });
    } else {
      const LevelOp* op = ops[i];
      Engine& E2 = engine();
      bool done = false;
      if (resident_mode(op->n, coarse_stop.max_iters) >= 0) {
        small_coarse.ensure(op, coarse_stop.max_iters);
        done = !op->sharded && small_coarse.try_run(b, x, coarse_stop, (int*)(E2.dscal + kSlotMisc), (double*)(E2.dscal + kSlotMisc) + 1);
      }
      if (!done) {
        LinOp A = [op](const cd* in, cd* out) { op->apply(in, out); };
        coarse_ws.halo = op->halo_elems();
        fgmres(op->n, A, nullptr, b, x, coarse_stop, coarse_ws, nullptr, nullptr, op);
      }
    }
    return;
  }
  const LevelOp* op = ops[i];
  const long long n = op->n;
  cd* cur = X[i];
  cd* oth = Y[i];
  // pre-smoothing (first sweep from zero in closed form unless an initial guess is given)
  if (pre > 0) {
    op->jacobi(x_init, b, cur, omega, x_init == nullptr);
    for (int s = 1; s < pre; ++s) { op->jacobi(cur, b, oth, omega, false); std::swap(cur, oth); }
  } else if (x_init) {
    HDB_CUDA(cudaMemcpyAsync(cur, x_init, sizeof(cd) * n, cudaMemcpyDeviceToDevice, E.st));
  } else {
    HDB_CUDA(cudaMemsetAsync(cur, 0, sizeof(cd) * n, E.st));
  }
  // coarse-grid correction: residual and restriction in one pass where the fused kernel
  // applies (mg.py:116-117; bit-identical to the pair), else the two launches
  const LevelOp* co = ops[i + 1];
  if (!op->sharded && !co->sharded && resrestrict_fits(op->c, op->g)) {
    E.kl(KF_RESRESTRICT, 44.0 * n, [&] {
      launch_resrestrict(op->c, op->g, cur, b, op->ksq, B[i + 1], dirichlet_mask(co->c), E.st);
    });
  } else {
    op->residual(b, cur, R[i]);
    restrict_levels(*op, *co, R[i], B[i + 1], S[i + 1], dirichlet_mask(co->c));
  }
  cycle(i + 1, B[i + 1], O[i + 1], nullptr);
  cd* dst = (post == 0) ? x : oth;
  prolong_levels(*co, *op, O[i + 1], cur, dst);
  if (post == 0) return;
  std::swap(cur, dst);  // cur = corrected iterate, dst = free buffer
  for (int s = 0; s < post; ++s) {
    cd* out = (s == post - 1) ? x : dst;
    if (s == post - 1 && xsum) op->jacobi_add(cur, b, out, omega, addt, xsum);  // x and x + addt in one sweep
    else op->jacobi(cur, b, out, omega, false);
    dst = cur;
    cur = out;
  }
}

// the top level's last post-smoothing sweep can also write x + addt (madp.py:327)
bool Multigrid::can_fold_sum() const { return post > 0 && ops.size() > 1 && ops[0]->jacobi_add_ok(); }

void Multigrid::vcycle(const cd* b, cd* x, const cd* x0, const cd* addt, cd* xsum) {
  Engine& E = engine();
  if (X.empty()) setup();
  const LevelOp* op = ops[0];
  // r0 (mg.py:131): ||b|| from zero, ||b - M x0|| otherwise
  if (x0) {
    op->residual(b, x0, R[0]);
    red_dot(op, R[0], R[0], op->n, E.dscal + kSlotMgR0);
  }
  cycle(0, b, x, x0, addt, xsum);
  // divergence guard (mg.py:133-138), evaluated on device; raised at the next host sync.
  // One fused pass: (||b - M x||^2, ||b||^2) without storing the residual.
  op->resnorm(b, x, E.dscal + kSlotMgPost, R[0]);
  E.kl(KF_CONTROL, 0.0, [&] {
    launch_guard(E.dscal + kSlotMgPost, nullptr, x0 ? E.dscal + kSlotMgR0 : nullptr, guard, E.dscal + kSlotFlag, E.st);
  });
}

}  // namespace hdb

namespace hdb {

// ----------------------------------------------------------- MADP solver
void MadpSolver::set_levels(int ml_) {
  ml = ml_;
  lv.clear();
  lv.resize(ml + 1);
}

void MadpSolver::setup() {
  Engine& E = engine();
  if (!dcounts) {
    dcap = 1 << 20;  // never flushed mid-solve: a reserved slot may still be awaiting its kernel
    dcounts = (int*)E.alloc_bytes(sizeof(int) * dcap);
    drel = (double*)E.alloc_bytes(sizeof(double) * dcap);
  }
  for (int l = 1; l <= ml; ++l) {
    MadpLevel& L = lv[l];
    if (!L.A) throw Error(E_ARG, "level operator missing");
    const long long n = L.A->n, h = L.A->halo_elems();
    L.ws_defl.halo = h;
    L.ws_cslp.halo = h;
    if (l >= 2 && !L.vhat) {
      L.vhat = E.alloc_h(n, h);
      L.vtil = E.alloc_h(n, h);
      if (lv[l - 1].A->sharded && !L.A->sharded) L.slab = E.alloc(n);
    }
    if (l < ml && !L.t) { L.t = E.alloc_h(n, h); L.rhs = E.alloc_h(n, h); L.r = E.alloc_h(n, h); }
    if (l == 1 && L.A->sharded && !L.xh) { L.bh = E.alloc_h(n, h); L.xh = E.alloc_h(n, h); }
  }
}

MadpSolver::~MadpSolver() {
  for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  if (!engine_ready()) return;
  Engine& E = engine();
  for (auto& L : lv) {
    const long long h = L.A ? L.A->halo_elems() : 0;
    for (cd* p : {L.vhat, L.vtil, L.t, L.rhs, L.r, L.bh, L.xh}) E.free_h(p, h);
    E.free(L.slab);
  }
  E.free(dcounts);
  E.free(drel);
}

void MadpSolver::reset_report() {
  rep = SolveReport();
  dused = 0;
  pending.clear();
  rep.cycle_iters.assign(ml + 1, {});
  rep.cslp_iters.assign(ml + 1, {});
  rep.matvecs.assign(ml + 1, 0);
  rep.prof_ms.assign((ml + 1) * PROF_KINDS, 0.0);
  rep.dev_ms.assign((ml + 1) * PROF_KINDS, 0.0);
  evs.clear();
  ev_used = 0;
  rep.prof_calls.assign((ml + 1) * PROF_KINDS, 0);
}

static bool dev_profiling() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HDB_PROFILE");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

cudaEvent_t MadpSolver::ev_get() {
  if (ev_used == ev_pool.size()) {
    cudaEvent_t e;
    HDB_CUDA(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_used++];
}

void MadpSolver::ev_resolve() {
  if (evs.empty()) return;
  HDB_CUDA(cudaEventSynchronize(evs.back().b));
  for (const EvRec& r : evs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) rep.dev_ms[r.slot] += ms;
  }
  evs.clear();
  ev_used = 0;
}

namespace {
struct ProfScope {
  MadpSolver& s;
  int slot;
  std::chrono::steady_clock::time_point t0;
  cudaEvent_t ea = nullptr;
  ProfScope(MadpSolver& s_, int level, int kind)
      : s(s_), slot(level * PROF_KINDS + kind), t0(std::chrono::steady_clock::now()) {
    if (dev_profiling()) {
      ea = s.ev_get();
      cudaEventRecord(ea, engine().st);
    }
  }
  ~ProfScope() {
    s.rep.prof_ms[slot] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    s.rep.prof_calls[slot] += 1;
    if (ea) {
      cudaEvent_t eb = s.ev_get();
      cudaEventRecord(eb, engine().st);
      s.evs.push_back({slot, ea, eb});
      if (s.evs.size() > 20000) s.ev_resolve();
    }
  }
};
}  // namespace

void MadpSolver::A(int l, const cd* u, cd* out) {
  rep.matvecs[l] += 1;  // madp.py:271-273
  lv[l].A->apply(u, out);
}

// madp.py:277-299
void MadpSolver::cslp_apply(int l, const cd* rhs, cd* out, const cd* addt, cd* sum) {
  ProfScope ps(*this, l, PROF_CSLP);
  MadpLevel& L = lv[l];
  Engine& E = engine();
  auto add_sum = [&] {  // sum = out + addt (madp.py:327) when the solve could not fold it in
    if (sum) E.kl(KF_BLAS, 48.0 * L.A->n, [&] { launch_add(out, addt, sum, L.A->n, 0, E.st); });
  };
  if (L.cslp == CSLP_NONE) {
    HDB_CUDA(cudaMemcpyAsync(out, rhs, sizeof(cd) * L.A->n, cudaMemcpyDeviceToDevice, E.st));
    add_sum();
    return;
  }
  if (L.cslp == CSLP_MG) {
    rep.cslp_iters[l].push_back(1);
    if (sum && L.mg->can_fold_sum()) {
      L.mg->vcycle(rhs, out, nullptr, addt, sum);
    } else {
      L.mg->vcycle(rhs, out);
      add_sum();
    }
    return;
  }
  cslp_krylov(l, rhs, out);
  add_sum();
}

// the Krylov forms of the CSLP solve (madp.py:288-297)
void MadpSolver::cslp_krylov(int l, const cd* rhs, cd* out) {
  MadpLevel& L = lv[l];
  const LevelOp* M = L.M;
  if (L.cslp == CSLP_BICGSTAB) {  // madp.py:292-297: a breakdown still yields a usable iterate
    LinOp Mop = [M](const cd* in, cd* o) { M->apply(in, o); };
    L.ws_bicg.halo = M->halo_elems();
    bool brk = false;
    std::string why;
    KReport r = bicgstab(M->n, Mop, nullptr, rhs, out, L.cslp_stop, L.ws_bicg, nullptr, M, &brk, &why);
    rep.cslp_iters[l].push_back(r.iterations);
    return;
  }
  if (!M->sharded && resident_mode(M->n, L.cslp_stop.max_iters) >= 0) {
    L.small_cslp.ensure(M, L.cslp_stop.max_iters);
    const int slot = reserve_count(l);
    slot_npts[slot] = M->n;
    if (L.small_cslp.try_run(rhs, out, L.cslp_stop, dcounts + slot, drel + slot)) return;
    unreserve_count(l);  // did not fit: the launch path below reports its own count
  }
  {
    const int slot = reserve_count(l);
    if (gmres_device(M, rhs, out, L.cslp_stop, L.ws_cslp, dcounts + slot, drel + slot)) return;
    unreserve_count(l);
  }
  LinOp Mop = [M](const cd* in, cd* o) { M->apply(in, o); };
  KReport r = fgmres(M->n, Mop, nullptr, rhs, out, L.cslp_stop, L.ws_cslp, nullptr, nullptr, M);
  rep.cslp_iters[l].push_back(r.iterations);
}

// count slot for a device-side solve at `level` (< 0: deflation cycle of -level,
// > 0: CSLP of level); its report entry is filled by flush_counts at the end
int MadpSolver::reserve_count(int level) {
  if (dused >= dcap) throw Error(E_ARG, "too many device-side solves in one call (raise dcap)");
  auto& lst = level < 0 ? rep.cycle_iters[-level] : rep.cslp_iters[level];
  lst.push_back(-1);
  pending.emplace_back(level, (int)lst.size() - 1);
  slot_npts.push_back(0);
  return dused++;
}

void MadpSolver::unreserve_count(int level) {
  auto& lst = level < 0 ? rep.cycle_iters[-level] : rep.cslp_iters[level];
  lst.pop_back();
  pending.pop_back();
  slot_npts.pop_back();
  dused--;
}

// copy device-resident iteration counts into the report
void MadpSolver::flush_counts() {
  Engine& E = engine();
  if (dused > 0) {
    std::vector<int> h(dused);
    HDB_CUDA(cudaMemcpyAsync(h.data(), dcounts, sizeof(int) * dused, cudaMemcpyDeviceToHost, E.st));
    E.fetch(1);  // sync + flag check
    for (int k = 0; k < dused; ++k) {
      const int lvl = pending[k].first;
      if (lvl < 0) rep.cycle_iters[-lvl][pending[k].second] = h[k];
      else rep.cslp_iters[lvl][pending[k].second] = h[k];
      if (slot_npts[k] > 0) E.kp.bytes[KF_RESIDENT] += gmres_alg_bytes(slot_npts[k], h[k]);
    }
  }
  dused = 0;
  pending.clear();
  slot_npts.clear();
}

// madp.py:301-327  (A-DEF1, lambda = 1)
void MadpSolver::precond(int l, const cd* v, cd* out) {
  ProfScope ps(*this, l, PROF_ADEF);
  Engine& E = engine();
  MadpLevel& L = lv[l];
  MadpLevel& N = lv[l + 1];
  restrict_levels(*L.A, *N.A, v, N.vhat, N.slab, 0);
  const int nxt = l + 1;
  LinOp Aop = [this, nxt](const cd* in, cd* o) { A(nxt, in, o); };
  LinOp Mop;
  if (nxt == ml) Mop = [this, nxt](const cd* in, cd* o) { cslp_apply(nxt, in, o); };
  else Mop = [this, nxt](const cd* in, cd* o) { precond(nxt, in, o); };
  {
    ProfScope pd(*this, nxt, PROF_DEFL);
    if (N.cycle_stop.rel_tol >= 1.0 && step1_enabled()) {  // exactly one iteration: no host round trip
      // reserve the count slot BEFORE the call: nested solves inside M reserve their own
      const int slot = reserve_count(-nxt);
      fgmres_step1(N.A->n, Aop, Mop, N.vhat, N.vtil, N.ws_defl, dcounts + slot, N.A, nxt);
    } else {
      KReport r = fgmres(N.A->n, Aop, &Mop, N.vhat, N.vtil, N.cycle_stop, N.ws_defl, nullptr, nullptr, N.A);
      rep.cycle_iters[nxt].push_back(r.iterations);
    }
  }
  prolong_levels(*N.A, *L.A, N.vtil, nullptr, L.t);
  rep.matvecs[l] += 1;
  L.A->residual(v, L.t, L.rhs);  // v - A t
  cslp_apply(l, L.rhs, L.r, L.t, out);  // r = CSLP(rhs); out = r + t
}

void MadpSolver::solve(const cd* b, cd* x) {
  Engine& E = engine();
  setup();
  reset_report();
  const double bytes0 = E.kp.total_bytes();
  HDB_CUDA(cudaMemsetAsync(E.dscal + kSlotFlag, 0, sizeof(cd), E.st));
  cudaEvent_t e0, e1;
  HDB_CUDA(cudaEventCreate(&e0));
  HDB_CUDA(cudaEventCreate(&e1));
  HDB_CUDA(cudaEventRecord(e0, E.st));
  const long long s0 = E.syncs, l0 = E.launches;
  const auto t0 = std::chrono::steady_clock::now();
  std::function<void(int, double)> hook = [this, t0](int, double) {
    rep.iter_wall_ms.push_back(
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  LinOp Aop = [this](const cd* in, cd* o) { A(1, in, o); };
  LinOp Mop = [this](const cd* in, cd* o) { precond(1, in, o); };
  try {
    const LevelOp* A1 = lv[1].A;
    const long long n1 = A1->n;
    if (A1->sharded) {  // stencil inputs need halo rows: solve through halo'd copies
      HDB_CUDA(cudaMemcpyAsync(lv[1].bh, b, sizeof(cd) * n1, cudaMemcpyDeviceToDevice, E.st));
      rep.outer = fgmres(n1, Aop, &Mop, lv[1].bh, lv[1].xh, outer, lv[1].ws_defl, &hook, nullptr, A1);
      HDB_CUDA(cudaMemcpyAsync(x, lv[1].xh, sizeof(cd) * n1, cudaMemcpyDeviceToDevice, E.st));
    } else {
      rep.outer = fgmres(n1, Aop, &Mop, b, x, outer, lv[1].ws_defl, &hook, nullptr, A1);
    }
    flush_counts();
    ev_resolve();
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  HDB_CUDA(cudaEventRecord(e1, E.st));
  HDB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  HDB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  rep.wall_ms = ms;
  rep.syncs = E.syncs - s0;
  rep.launches = E.launches - l0;
  rep.alg_bytes = E.kp.total_bytes() - bytes0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace hdb
