// extern "C" boundary (declared in include/hdb200.h).  Every entry point
// catches engine exceptions and turns them into a status + message.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hdb200.h"
#include "engine.h"

using namespace hdb;

struct hdb_op {
  LevelOp op;
  SmallSolve resident;  // workspaces reused across hdb_op_gmres calls
  KWS ws;
  int* dres = nullptr;  // its (int) + relres (double)
};
struct hdb_mg { Multigrid mg; };
struct hdb_solver {
  MadpSolver s;
  cd *db = nullptr, *dx = nullptr;  // device staging for host-buffer solves (kept across calls)
  ~hdb_solver() {
    if (engine_ready()) { engine().free(db); engine().free(dx); }
  }
};

static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return HDB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HDB_E_CUDA;
  } catch (...) {
    g_err = "unknown error";
    return HDB_E_CUDA;
  }
}

// constant-k^2 levels get the per-tap coefficient table (same rounding as per point)
static void set_uniform(OpCoef& c, const double* ksq, long long n) {
  c.uniform = 0;
  if (n < 1) return;
  const double k0 = ksq[0];
  for (long long i = 1; i < n; ++i)
    if (ksq[i] != k0) return;
  c.uniform = 1;
  c.ku = k0;
  const int N = 2 * c.radius + 1;
  for (int t = 0; t < N * N; ++t) {
    volatile double mk_r = c.mass[t].x * k0;  // separate roundings, as __dmul_rn / __dadd_rn on device
    volatile double mk_i = c.mass[t].y * k0;
    volatile double re = c.lap[t] + mk_r;
    c.ucoef[t] = mkc(re, mk_i);
  }
}

static void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

extern "C" {

int hdb_version(void) { return 100; }
const char* hdb_last_error(void) { return g_err.c_str(); }

int hdb_init(int device) {
  return guarded([&] { engine_init(device); });
}
int hdb_stream(void** out) {
  return guarded([&] { *out = (void*)engine().st; });
}
int hdb_set_stream(void* stream) {
  return guarded([&] {
    Engine& E = engine();
    E.sync();
    E.st = (cudaStream_t)stream;
  });
}
int hdb_sync(void) {
  return guarded([&] { engine().sync(); });
}
int hdb_stats(long long* launches, long long* bytes) {
  return guarded([&] {
    if (launches) *launches = engine().launches;
    if (bytes) *bytes = (long long)engine().bytes_alloc;
  });
}

int hdb_op_create(hdb_op** out, int nx, int ny, int radius, double h, const int* bc4, const double* lap,
                  const double* mass_re, const double* mass_im, const double* ksq_host) {
  return guarded([&] {
    if (nx < 2 || ny < 2) throw Error(E_ARG, "grid needs at least 2 points per direction");
    if (radius < 1 || radius > 3) throw Error(E_ARG, "radius must be 1, 2 or 3");
    Engine& E = engine();
    auto* o = new hdb_op();
    LevelOp& L = o->op;
    std::memset(&L.c, 0, sizeof(L.c));
    L.c.radius = radius;
    for (int s = 0; s < 4; ++s) L.c.bc[s] = bc4[s];
    L.c.h = h;
    const int N = 2 * radius + 1;
    for (int i = 0; i < N * N; ++i) {
      L.c.lap[i] = lap[i];
      L.c.mass[i] = mkc(mass_re[i], mass_im[i]);
    }
    if (radius == 1) {
      L.c.s = lap[4] / 4.0;   // lap_coef[1,1] / 4   (operators.py:174, 186)
      L.c.mc = L.c.mass[4];   // mass_coef[1,1]
      L.c.E = (-L.c.s * 2.0) * h;  // -lap_scale*2i*h  (operators.py:198)
    }
    L.g.nx = nx; L.g.ny = ny; L.g.row0 = 0; L.g.nyg = ny;
    L.n = (long long)nx * ny;
    set_uniform(L.c, ksq_host, L.n);
    L.ksq = (double*)E.alloc_bytes(sizeof(double) * L.n);
    HDB_CUDA(cudaMemcpyAsync(L.ksq, ksq_host, sizeof(double) * L.n, cudaMemcpyHostToDevice, E.st));
    HDB_CUDA(cudaStreamSynchronize(E.st));
    *out = o;
  });
}

// (min, max, non-finite count) of a device float64 array -> host
static void device_stats(const double* a, long long n, double out3[3]) {
  Engine& E = engine();
  double* part = (double*)E.alloc_bytes(sizeof(double) * 3 * (size_t)(setup_stats_blocks(n) + 1));
  double* res = part + 3 * (size_t)setup_stats_blocks(n);
  launch_setup_stats(a, n, part, E.red.ticket, res, E.st);
  HDB_CUDA(cudaMemcpyAsync(out3, res, sizeof(double) * 3, cudaMemcpyDeviceToHost, E.st));
  HDB_CUDA(cudaStreamSynchronize(E.st));
  E.free(part);
}

// the same operator from a k^2 field that already lives on the device (GPU-side setup:
// no host copy of the level exists); whole grid, one rank
int hdb_op_create_dev(hdb_op** out, int nx, int ny, int radius, double h, const int* bc4, const double* lap,
                      const double* mass_re, const double* mass_im, const double* ksq_dev) {
  return guarded([&] {
    if (nx < 2 || ny < 2) throw Error(E_ARG, "grid needs at least 2 points per direction");
    std::vector<double> dummy((size_t)nx * 2, 0.0);  // coefficients through the host path on a 2-row dummy field
    hdb_op* o = nullptr;
    const int st = hdb_op_create(&o, nx, 2, radius, h, bc4, lap, mass_re, mass_im, dummy.data());
    if (st != HDB_OK) throw Error(st, g_err);
    Engine& E = engine();
    LevelOp& L = o->op;
    E.free(L.ksq);
    L.g.nx = nx; L.g.ny = ny; L.g.row0 = 0; L.g.nyg = ny;
    L.n = (long long)nx * ny;
    double st3[3];
    device_stats(ksq_dev, L.n, st3);
    if (st3[2] != 0.0 || st3[0] < 0.0) {
      delete o;
      throw Error(E_ARG, "k^2 field must be finite and nonnegative");
    }
    // constant k^2 (min == max): the per-tap coefficient table, as set_uniform builds it
    const double ku[1] = {st3[0]};
    L.c.uniform = 0;
    if (st3[0] == st3[1]) set_uniform(L.c, ku, 1);
    L.ksq = (double*)E.alloc_bytes(sizeof(double) * L.n);
    HDB_CUDA(cudaMemcpyAsync(L.ksq, ksq_dev, sizeof(double) * L.n, cudaMemcpyDeviceToDevice, E.st));
    HDB_CUDA(cudaStreamSynchronize(E.st));
    *out = o;
  });
}

// ---- device-side problem setup (grid.py:120-160, 261-287, 309-320) ----------------------
int hdb_setup_ksq_constant(double* out_dev, long long n, double ksq) {
  return guarded([&] { launch_setup_fill(out_dev, n, ksq, engine().st); check_launch(); });
}
int hdb_setup_ksq_wedge(double* out_dev, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                        int nlayers, const double* layers3) {
  return guarded([&] {
    if (nlayers < 1 || nlayers > 8) throw Error(E_ARG, "wedge model: 1..8 layers");
    SetupLayers Ls;
    Ls.n = nlayers;
    for (int q = 0; q < nlayers; ++q) {
      Ls.y0[q] = layers3[3 * q]; Ls.y1[q] = layers3[3 * q + 1]; Ls.v[q] = layers3[3 * q + 2];
    }
    launch_setup_wedge(out_dev, nx, ny, ox, oy, hx, hy, w, Ls, engine().st);
    check_launch();
  });
}
int hdb_setup_ksq_raster(double* out_dev, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                         const double* raster_dev, int rnx, int rny, double rx0, double ry0, double rdx, double rdy) {
  return guarded([&] {
    if (rnx < 1 || rny < 1) throw Error(E_ARG, "empty velocity raster");
    launch_setup_raster(out_dev, nx, ny, ox, oy, hx, hy, w, raster_dev, rnx, rny, rx0, ry0, rdx, rdy, engine().st);
    check_launch();
  });
}
int hdb_setup_inject(const double* fine_dev, int nfx, int nfy, double* coarse_dev) {
  return guarded([&] {
    if ((nfx - 1) % 2 || (nfy - 1) % 2) throw Error(E_ARG, "cannot coarsen: n-1 must be even");
    launch_setup_inject(fine_dev, nfx, coarse_dev, (nfx - 1) / 2 + 1, (nfy - 1) / 2 + 1, engine().st);
    check_launch();
  });
}
int hdb_setup_stats(const double* a_dev, long long n, double* out3) {
  return guarded([&] { device_stats(a_dev, n, out3); check_launch(); });
}
int hdb_setup_point_source(void* rhs_dev, long long n, long long index, double value) {
  return guarded([&] {
    if (index < 0 || index >= n) throw Error(E_ARG, "source index outside the grid");
    launch_setup_point((cd*)rhs_dev, n, index, value, engine().st);
    check_launch();
  });
}

// a row slab [row0, row0+ny_local) of a level with ny_global rows; `halo` rows of
// k^2 are copied around it (from the full host array), vectors of this level
// carry `halo` halo rows; slab_row0/slab_ny list every rank's slab.
int hdb_op_create_slab(hdb_op** out, int nx, int ny_global, int radius, double h, const int* bc4, const double* lap,
                       const double* mass_re, const double* mass_im, const double* ksq_full_host, int row0,
                       int ny_local, int halo, int nranks, const int* slab_row0, const int* slab_ny) {
  return guarded([&] {
    if (halo < radius || halo < 2) throw Error(E_ARG, "halo must cover the stencil radius and the transfer (2)");
    if (ny_local < halo) throw Error(E_ARG, "slab thinner than its halo");
    hdb_op* o = nullptr;
    // build the coefficients through the full-grid path on a dummy k^2, then replace geometry
    const int st = hdb_op_create(&o, nx, std::max(ny_local, 2), radius, h, bc4, lap, mass_re, mass_im, ksq_full_host);
    if (st != HDB_OK) throw Error(st, g_err);
    Engine& E = engine();
    LevelOp& L = o->op;
    E.free(L.ksq);
    L.g.nx = nx; L.g.ny = ny_local; L.g.row0 = row0; L.g.nyg = ny_global;
    L.n = (long long)nx * ny_local;
    L.H = halo;
    L.sharded = nranks > 1;
    L.slab_row0.assign(slab_row0, slab_row0 + nranks);
    L.slab_ny.assign(slab_ny, slab_ny + nranks);
    const long long hel = (long long)halo * nx;
    double* base = (double*)E.alloc_bytes(sizeof(double) * (L.n + 2 * hel));
    HDB_CUDA(cudaMemsetAsync(base, 0, sizeof(double) * (L.n + 2 * hel), E.st));
    L.ksq = base + hel;
    set_uniform(L.c, ksq_full_host, (long long)nx * ny_global);
    const int r_lo = std::max(0, row0 - halo), r_hi = std::min(ny_global, row0 + ny_local + halo);
    HDB_CUDA(cudaMemcpyAsync(L.ksq + (long long)(r_lo - row0) * nx, ksq_full_host + (long long)r_lo * nx,
                             sizeof(double) * (size_t)(r_hi - r_lo) * nx, cudaMemcpyHostToDevice, E.st));
    HDB_CUDA(cudaStreamSynchronize(E.st));
    *out = o;
  });
}

int hdb_comm_unique_id(char* out128) {
  return guarded([&] { nccl_unique_id(out128); });
}
int hdb_comm_init_nccl(const char* id128, int nranks, int rank) {
  return guarded([&] {
    Engine& E = engine();
    delete E.comm;
    E.comm = nullptr;
    if (nranks > 1) E.comm = make_nccl_comm(id128, nranks, rank);
  });
}
int hdb_comm_selftest_nccl(void) {
  return guarded([&] { nccl_selftest(engine().st); });
}
int hdb_comm_init_threads(long long group, int nranks, int rank) {
  return guarded([&] {
    Engine& E = engine();
    delete E.comm;
    E.comm = nullptr;
    if (nranks > 1) E.comm = make_thread_comm(group, nranks, rank);
  });
}
int hdb_thread_engine_begin(int device) {
  return guarded([&] { thread_engine_begin(device); });
}
int hdb_thread_engine_end(void) {
  return guarded([&] { thread_engine_end(); });
}

int hdb_op_destroy(hdb_op* op) {
  return guarded([&] {
    if (!op) return;
    if (engine_ready()) {
      engine().sync();
      engine().free(op->op.ksq - op->op.halo_elems());
      engine().free(op->dres);
    }
    delete op;
  });
}

int hdb_op_apply(hdb_op* op, const void* u, void* out) {
  return guarded([&] { op->op.apply((const cd*)u, (cd*)out); check_launch(); });
}
int hdb_op_residual(hdb_op* op, const void* b, const void* u, void* out) {
  return guarded([&] { op->op.residual((const cd*)b, (const cd*)u, (cd*)out); check_launch(); });
}
int hdb_op_resnorm(hdb_op* op, const void* b, const void* u, double* out2) {
  return guarded([&] {
    Engine& E = engine();
    cd* scratch = (op->op.c.radius == 1 && !pinv_mode()) ? nullptr : E.alloc(op->op.n);
    op->op.resnorm((const cd*)b, (const cd*)u, E.dscal + kSlotMisc, scratch);
    check_launch();
    if (!out2) {  // timing form: result stays in the device slot, no sync
      if (scratch) E.free(scratch);
      return;
    }
    HDB_CUDA(cudaMemcpyAsync(E.hscal + kSlotMisc, E.dscal + kSlotMisc, sizeof(cd), cudaMemcpyDeviceToHost, E.st));
    E.sync();
    if (scratch) E.free(scratch);
    out2[0] = E.hscal[kSlotMisc].x;
    out2[1] = E.hscal[kSlotMisc].y;
  });
}
int hdb_op_jacobi(hdb_op* op, const void* x, const void* b, void* out, double omega) {
  return guarded([&] {
    if (op->op.c.radius != 1) throw Error(E_ARG, "Jacobi is only defined for radius-1 operators");
    op->op.jacobi((const cd*)x, (const cd*)b, (cd*)out, omega, x == nullptr);
    check_launch();
  });
}

int hdb_op_residual_restrict(hdb_op* op, const void* b, const void* u, void* coarse, int zero_mask) {
  return guarded([&] {
    const LevelOp& o = op->op;
    if (o.c.radius != 1 || o.sharded) throw Error(E_ARG, "fused residual + restriction: unsharded radius-1 operators only");
    if ((o.g.nx - 1) % 2 || (o.g.ny - 1) % 2 || o.g.nx < 3 || o.g.ny < 3)
      throw Error(E_ARG, "cannot coarsen: n-1 must be even (transfers.py:53-56)");
    Engine& E = engine();
    E.kl(KF_RESRESTRICT, 44.0 * o.n, [&] {
      launch_resrestrict(o.c, o.g, (const cd*)u, (const cd*)b, o.ksq, (cd*)coarse, zero_mask, E.st);
    });
    check_launch();
  });
}
int hdb_op_jacobi_add(hdb_op* op, const void* x, const void* b, void* out, double omega, const void* addt,
                      void* out2) {
  return guarded([&] {
    const LevelOp& o = op->op;
    if (o.c.radius != 1) throw Error(E_ARG, "Jacobi is only defined for radius-1 operators");
    if (!x || !addt || !out2) throw Error(E_ARG, "jacobi_add needs x, addt and out2");
    if (o.jacobi_add_ok()) {
      o.jacobi_add((const cd*)x, (const cd*)b, (cd*)out, omega, (const cd*)addt, (cd*)out2);
    } else {  // small grids: the sweep, then the sum
      o.jacobi((const cd*)x, (const cd*)b, (cd*)out, omega, false);
      Engine& E = engine();
      E.kl(KF_BLAS, 48.0 * o.n, [&] { launch_add((const cd*)out, (const cd*)addt, (cd*)out2, o.n, 0, E.st); });
    }
    check_launch();
  });
}

int hdb_restrict(const void* fine, int nfy, int nfx, void* coarse, int zero_mask) {
  return guarded([&] {
    if ((nfx - 1) % 2 || (nfy - 1) % 2 || nfx < 3 || nfy < 3)
      throw Error(E_ARG, "cannot coarsen: n-1 must be even (transfers.py:53-56)");
    launch_restrict((const cd*)fine, (cd*)coarse, full_tgeom(nfx, nfy), zero_mask, engine().st);
    check_launch();
  });
}
int hdb_prolong(const void* coarse, int nfy, int nfx, const void* base, void* fine) {
  return guarded([&] {
    if ((nfx - 1) % 2 || (nfy - 1) % 2) throw Error(E_ARG, "fine shape does not refine the coarse grid");
    launch_prolong((const cd*)coarse, (const cd*)base, (cd*)fine, full_tgeom(nfx, nfy), base != nullptr,
                   engine().st);
    check_launch();
  });
}

int hdb_dot(const void* u, const void* v, long long n, double* out2) {
  return guarded([&] {
    Engine& E = engine();
    launch_dot((const cd*)u, (const cd*)v, n, E.red, E.dscal + kSlotMisc, E.st);
    check_launch();
    if (!out2) return;  // timing form: result stays on the device, no sync
    HDB_CUDA(cudaMemcpyAsync(E.hscal + kSlotMisc, E.dscal + kSlotMisc, sizeof(cd), cudaMemcpyDeviceToHost, E.st));
    E.sync();
    out2[0] = E.hscal[kSlotMisc].x;
    out2[1] = E.hscal[kSlotMisc].y;
  });
}

int hdb_mg_create(hdb_mg** out, hdb_op* const* ops, int nlev, const double* inv_host, int ninv, double omega,
                  int pre, int post, double guard, double coarse_tol, int coarse_max) {
  return guarded([&] {
    if (nlev < 1) throw Error(E_ARG, "multigrid needs at least one level");
    if (pre < 0 || post < 0 || pre + post < 1) throw Error(E_ARG, "at least one smoothing step is required");
    Engine& E = engine();
    auto* m = new hdb_mg();
    for (int i = 0; i < nlev; ++i) m->mg.ops.push_back(&ops[i]->op);
    m->mg.omega = omega; m->mg.pre = pre; m->mg.post = post; m->mg.guard = guard;
    m->mg.coarse_stop = Stop{coarse_tol, coarse_max};
    if (inv_host) {
      if ((long long)ninv != ops[nlev - 1]->op.n) { delete m; throw Error(E_ARG, "inverse size mismatch"); }
      m->mg.ninv = ninv;
      m->mg.Ainv = (cd*)E.alloc_bytes(sizeof(cd) * (size_t)ninv * ninv);
      HDB_CUDA(cudaMemcpyAsync(m->mg.Ainv, inv_host, sizeof(cd) * (size_t)ninv * ninv, cudaMemcpyHostToDevice, E.st));
    }
    m->mg.setup();
    E.sync();
    *out = m;
  });
}
int hdb_mg_destroy(hdb_mg* mg) {
  return guarded([&] {
    if (engine_ready()) engine().sync();
    delete mg;
  });
}
int hdb_mg_vcycle(hdb_mg* mg, const void* b, const void* x0, void* x) {
  return guarded([&] {
    Engine& E = engine();
    HDB_CUDA(cudaMemsetAsync(E.dscal + kSlotFlag, 0, sizeof(cd), E.st));
    mg->mg.vcycle((const cd*)b, (cd*)x, (const cd*)x0);
    check_launch();
    E.fetch(1);
  });
}

int hdb_fgmres(long long n, hdb_linop_fn A, void* Au, hdb_linop_fn M, void* Mu, const void* b, const void* x0,
               void* x, double rel_tol, int max_iters, hdb_iter_fn hook, void* hook_user, int* iterations,
               double* final_relres, int* converged, double* hist, int hist_cap) {
  return guarded([&] {
    if (max_iters < 1) throw Error(E_ARG, "max_iters must be >= 1");
    if (rel_tol < 0) throw Error(E_ARG, "rel_tol must be nonnegative");
    LinOp Aop = [A, Au](const cd* in, cd* out) {
      if (A(Au, in, out) != 0) throw Error(E_ARG, "operator callback failed");
    };
    LinOp Mop = [M, Mu](const cd* in, cd* out) {
      if (M(Mu, in, out) != 0) throw Error(E_ARG, "preconditioner callback failed");
    };
    std::function<void(int, double)> H = [hook, hook_user](int it, double rel) {
      if (hook(hook_user, it, rel) != 0) throw Error(E_ARG, "iteration callback failed");
    };
    KWS ws;
    KReport r = fgmres(n, Aop, M ? &Mop : nullptr, (const cd*)b, (cd*)x, Stop{rel_tol, max_iters}, ws,
                       hook ? &H : nullptr, (const cd*)x0);
    engine().sync();
    *iterations = r.iterations;
    *final_relres = r.final_relres;
    *converged = r.converged ? 1 : 0;
    for (int i = 0; i < hist_cap && i < (int)r.history.size(); ++i) hist[i] = r.history[i];
  });
}

int hdb_op_gmres(hdb_op* op, const void* b, void* x, double rel_tol, int max_iters, int mode, int* iterations,
                 double* final_relres) {
  return guarded([&] {
    if (max_iters < 1) throw Error(E_ARG, "max_iters must be >= 1");
    Engine& E = engine();
    HDB_CUDA(cudaMemsetAsync(E.dscal + kSlotFlag, 0, sizeof(cd), E.st));
    const LevelOp* L = &op->op;
    int m = mode == 2 ? resident_mode(L->n, max_iters) : mode;
    if (m >= 0) {
      SmallSolve& ss = op->resident;
      ss.ensure(L, max_iters);
      if (!op->dres) op->dres = (int*)E.alloc_bytes(16);
      int* dits = op->dres;
      double* drel = (double*)(op->dres + 2);
      if (launch_resident_gmres(m, resident_ortho(), L->c, L->g, L->ksq, (const cd*)b, (cd*)x, ss.basis, ss.Rg, ss.gpart, L->n,
                                rel_tol, max_iters, dits, drel, E.dscal + kSlotFlag, E.st) != 0)
        throw Error(E_ARG, "problem does not fit the requested device-resident mode");
      int h_its = 0;
      double h_rel = 0.0;
      HDB_CUDA(cudaMemcpyAsync(&h_its, dits, sizeof(int), cudaMemcpyDeviceToHost, E.st));
      HDB_CUDA(cudaMemcpyAsync(&h_rel, drel, sizeof(double), cudaMemcpyDeviceToHost, E.st));
      E.fetch(1);
      *iterations = h_its;
      *final_relres = h_rel;
      return;
    }
    if (mode == -2) {  // the device-driven loop of large levels (Givens / stopping test on device)
      if (!op->dres) op->dres = (int*)E.alloc_bytes(16);
      int* dits = op->dres;
      double* drel = (double*)(op->dres + 2);
      if (!gmres_device(L, (const cd*)b, (cd*)x, Stop{rel_tol, max_iters}, op->ws, dits, drel))
        throw Error(E_ARG, "level does not qualify for the device-driven GMRES loop");
      int h_its = 0;
      double h_rel = 0.0;
      HDB_CUDA(cudaMemcpyAsync(&h_its, dits, sizeof(int), cudaMemcpyDeviceToHost, E.st));
      HDB_CUDA(cudaMemcpyAsync(&h_rel, drel, sizeof(double), cudaMemcpyDeviceToHost, E.st));
      E.fetch(1);
      *iterations = h_its;
      *final_relres = h_rel;
      return;
    }
    LinOp Aop = [L](const cd* in, cd* o) { L->apply(in, o); };
    KReport r = fgmres(L->n, Aop, nullptr, (const cd*)b, (cd*)x, Stop{rel_tol, max_iters}, op->ws);
    *iterations = r.iterations;
    *final_relres = r.final_relres;
  });
}

// telemetry: per-phase cycle counters of device-resident solves (CTA 0, thread 0)
static long long* g_phase = nullptr;
static constexpr int kPhaseSlots = 12;
int hdb_resident_profile(int enable, long long* host_out12) {
  return guarded([&] {
    Engine& E = engine();
    if (enable) {
      if (!g_phase) g_phase = (long long*)E.alloc_bytes(kPhaseSlots * sizeof(long long));
      HDB_CUDA(cudaMemsetAsync(g_phase, 0, kPhaseSlots * sizeof(long long), E.st));
      resident_set_profile(g_phase);
    } else {
      if (host_out12 && g_phase) {
        HDB_CUDA(cudaMemcpyAsync(host_out12, g_phase, kPhaseSlots * sizeof(long long), cudaMemcpyDeviceToHost, E.st));
        E.sync();
      }
      resident_set_profile(nullptr);
    }
  });
}

int hdb_bicgstab(long long n, hdb_linop_fn A, void* Au, hdb_linop_fn M, void* Mu, const void* b, const void* x0,
                 void* x, double rel_tol, int max_iters, int* iterations, double* final_relres, int* converged,
                 double* hist, int hist_cap, int* hist_len) {
  return guarded([&] {
    if (max_iters < 1) throw Error(E_ARG, "max_iters must be >= 1");
    LinOp Aop = [A, Au](const cd* in, cd* out) {
      if (A(Au, in, out) != 0) throw Error(E_ARG, "operator callback failed");
    };
    LinOp Mop = [M, Mu](const cd* in, cd* out) {
      if (M(Mu, in, out) != 0) throw Error(E_ARG, "preconditioner callback failed");
    };
    BWS ws;
    bool brk = false;
    std::string why;
    KReport r = bicgstab(n, Aop, M ? &Mop : nullptr, (const cd*)b, (cd*)x, Stop{rel_tol, max_iters}, ws,
                         (const cd*)x0, nullptr, &brk, &why);
    engine().sync();
    *iterations = r.iterations;
    *final_relres = r.final_relres;
    *converged = r.converged ? 1 : 0;
    *hist_len = (int)r.history.size();
    for (int i = 0; i < hist_cap && i < (int)r.history.size(); ++i) hist[i] = r.history[i];
    if (brk) throw Error(E_BREAKDOWN, why);
  });
}

int hdb_solver_create(hdb_solver** out, int ml, double outer_tol, int outer_max) {
  return guarded([&] {
    if (ml < 2) throw Error(E_ARG, "hierarchy needs at least two levels");
    auto* s = new hdb_solver();
    s->s.set_levels(ml);
    s->s.outer = Stop{outer_tol, outer_max};
    *out = s;
  });
}
int hdb_solver_set_level(hdb_solver* s, int level, hdb_op* A, hdb_op* M, hdb_mg* mg, int cslp, double cslp_tol,
                         int cslp_max, double cycle_tol, int cycle_max) {
  return guarded([&] {
    if (level < 1 || level > s->s.ml) throw Error(E_ARG, "level outside 1..ml");
    MadpLevel& L = s->s.lv[level];
    L.A = &A->op;
    L.M = M ? &M->op : nullptr;
    L.mg = mg ? &mg->mg : nullptr;
    L.cslp = cslp;
    if (cslp == CSLP_MG && !mg) throw Error(E_ARG, "cslp=mg needs a multigrid");
    if ((cslp == CSLP_GMRES || cslp == CSLP_BICGSTAB) && !M) throw Error(E_ARG, "cslp=gmres/bicgstab needs a CSLP operator");
    L.cslp_stop = Stop{cslp_tol, cslp_max};
    L.cycle_stop = Stop{cycle_tol, cycle_max};
  });
}
int hdb_solver_solve(hdb_solver* s, const void* b, void* x, int host_buffers) {
  return guarded([&] {
    Engine& E = engine();
    const long long n = s->s.lv[1].A->n;
    if (!host_buffers) {
      s->s.solve((const cd*)b, (cd*)x);
      return;
    }
    if (!s->db) {
      s->db = E.alloc(n);
      s->dx = E.alloc(n);
    }
    try {
      HDB_CUDA(cudaMemcpyAsync(s->db, b, sizeof(cd) * n, cudaMemcpyHostToDevice, E.st));
      s->s.solve(s->db, s->dx);
      HDB_CUDA(cudaMemcpyAsync(x, s->dx, sizeof(cd) * n, cudaMemcpyDeviceToHost, E.st));
      E.sync();
    } catch (...) {
      cudaStreamSynchronize(E.st);  // (not E.sync(): a sticky error here must not mask the original one)
      throw;
    }
  });
}
int hdb_solver_report(hdb_solver* s, int* its, int* conv, double* fin, double* wall, int* hl) {
  return guarded([&] {
    const SolveReport& r = s->s.rep;
    *its = r.outer.iterations;
    *conv = r.outer.converged ? 1 : 0;
    *fin = r.outer.final_relres;
    *wall = r.wall_ms;
    *hl = (int)r.outer.history.size();
  });
}
int hdb_solver_history(hdb_solver* s, double* hist, double* iw, int cap) {
  return guarded([&] {
    const SolveReport& r = s->s.rep;
    for (int i = 0; i < cap && i < (int)r.outer.history.size(); ++i) hist[i] = r.outer.history[i];
    if (iw)
      for (int i = 0; i < cap && i < (int)r.iter_wall_ms.size(); ++i) iw[i] = r.iter_wall_ms[i];
  });
}
int hdb_solver_counts(hdb_solver* s, int level, int kind, int* buf, int cap, int* count) {
  return guarded([&] {
    const SolveReport& r = s->s.rep;
    if (level < 1 || level >= (int)r.cycle_iters.size()) throw Error(E_ARG, "level outside 1..ml");
    const std::vector<int>& v = kind == 0 ? r.cycle_iters[level] : r.cslp_iters[level];
    *count = (int)v.size();
    for (int i = 0; i < cap && i < (int)v.size(); ++i) buf[i] = v[i];
  });
}
int hdb_solver_matvecs(hdb_solver* s, long long* buf, int cap) {
  return guarded([&] {
    const SolveReport& r = s->s.rep;
    for (int i = 0; i < cap && i < (int)r.matvecs.size(); ++i) buf[i] = r.matvecs[i];
  });
}
int hdb_solver_precond(hdb_solver* s, int level, const void* v, void* out) {
  return guarded([&] {
    if (level < 1 || level >= s->s.ml) throw Error(E_ARG, "preconditioner level outside 1..ml-1");
    Engine& E = engine();
    s->s.setup();
    s->s.reset_report();
    HDB_CUDA(cudaMemsetAsync(E.dscal + kSlotFlag, 0, sizeof(cd), E.st));
    s->s.precond(level, (const cd*)v, (cd*)out);
    check_launch();
    s->s.flush_counts();
    E.fetch(1);
  });
}
int hdb_solver_profile(hdb_solver* s, double* ms_host, long long* calls_host, int cap, long long* syncs,
                       long long* launches) {
  return guarded([&] {
    const SolveReport& r = s->s.rep;
    for (int i = 0; i < cap && i < (int)r.prof_ms.size(); ++i) {
      // device time when HDB_PROFILE=1 recorded it, else host wall time
      const bool dev = i < (int)r.dev_ms.size() && r.dev_ms[i] > 0.0;
      ms_host[i] = dev ? r.dev_ms[i] : r.prof_ms[i];
      calls_host[i] = r.prof_calls[i];
    }
    *syncs = r.syncs;
    *launches = r.launches;
  });
}
int hdb_solver_bytes(hdb_solver* s, double* alg_bytes) {
  return guarded([&] { *alg_bytes = s->s.rep.alg_bytes; });
}

int hdb_op_set_separable(hdb_op* op, const double* sa, const double* sm, double lsc, double msc_re, double msc_im) {
  return guarded([&] {
    OpCoef& c = op->op.c;
    if (c.radius < 2) throw Error(E_ARG, "the separable form applies to radius-2/3 Galerkin levels");
    const int n = 2 * c.radius + 1;
    for (int q = 0; q < 7; ++q) {
      c.sa[q] = q < n ? sa[q] : 0.0;
      c.sm[q] = q < n ? sm[q] : 0.0;
    }
    c.lsc = lsc;
    c.msc = mkc(msc_re, msc_im);
    c.sep = 1;
  });
}

int hdb_plan_gather_rows(const int* fine_slab_row0, int nranks, int rank, int ncy_g, int* row0, int* ny) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(E_ARG, "rank out of range");
    std::vector<int> r0(fine_slab_row0, fine_slab_row0 + nranks);
    gather_rows(r0, rank, ncy_g, *row0, *ny);
  });
}

int hdb_option(const char* name, int value) {
  return guarded([&] {
    const std::string k = name ? name : "";
    if (k == "mgs_ls") set_mgs_ls(value);
    else if (k == "rg_exact") set_rg_exact(value);
    else if (k == "pinv") set_pinv(value);
    else if (k == "lsh_prefer") set_lsh_prefer(value);
    else throw Error(E_ARG, "unknown option " + k);
  });
}

int hdb_kprof(int enable) {
  return guarded([&] {
    Engine& E = engine();
    E.kp.reset();
    E.kp.on = enable != 0;
  });
}

int hdb_kprof_read(int fam, char* name_out32, long long* launches, double* alg_bytes, double* device_ms) {
  return guarded([&] {
    Engine& E = engine();
    if (fam < 0) {
      *launches = KF_COUNT;
      return;
    }
    if (fam >= KF_COUNT) throw Error(E_ARG, "kernel family out of range");
    E.kp.resolve();
    if (name_out32) {
      std::strncpy(name_out32, kfam_name(fam), 31);
      name_out32[31] = 0;
    }
    *launches = E.kp.n[fam];
    *alg_bytes = E.kp.bytes[fam];
    *device_ms = E.kp.ms[fam];
  });
}

int hdb_solver_destroy(hdb_solver* s) {
  return guarded([&] {
    if (engine_ready()) engine().sync();
    delete s;
  });
}

}  // extern "C"
