// Host-side engine: device buffers, level operators, Krylov driver (FGMRES with
// host Givens), CSLP multigrid V-cycle and the recursive A-DEF1 (MADP) solver,
// single GPU or row slabs over several ranks (Comm).
#pragma once
#include <complex>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.h"
#include "kernels.h"

namespace hdb {

enum Status { OK = 0, E_ARG = 1, E_CUDA = 2, E_NONFINITE = 3, E_MGDIV = 4, E_BREAKDOWN = 5 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline std::string src_tail(const char* path) {  // file name of a source path (error locations)
  const std::string p(path);
  const size_t k = p.find_last_of('/');
  return k == std::string::npos ? p : p.substr(k + 1);
}

#define HDB_CUDA(x)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::hdb::Error(::hdb::E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) +  \
                                            " [" + ::hdb::src_tail(__FILE__) + ":" + std::to_string(__LINE__) + "]"); \
  } while (0)

using cplx = std::complex<double>;

// device scalar block layout (Engine::dscal)
constexpr int kScal = 1024;
constexpr int kSlotFlag = 0;        // .x = 1.0 MG divergence guard fired, 2.0 non-finite (device solve)
constexpr int kSlotH = 1;           // Hessenberg column h_0.. at kSlotH + i
constexpr int kSlotMgR0 = 1019;
constexpr int kSlotMgPost = 1020;
constexpr int kSlotMgB = 1021;
constexpr int kSlotMisc = 1022;

// Kernel families for the launch accounting (algorithmic HBM bytes per launch,
// SURVEY §8(d) per-point figures x the points the launch covers) and, when
// armed, per-launch CUDA-event timing on the engine stream (hdb_kprof).
enum KFam {
  KF_APPLY5 = 0,   // radius-1 apply, 40 B/pt
  KF_RESID5,       // radius-1 residual b - A u, 56 B/pt
  KF_JACOBI,       // damped Jacobi sweep, 56 B/pt (40 from zero)
  KF_RESNORM,      // fused residual + norms, 40 B/pt
  KF_GALERKIN,     // radius-2/3 apply or residual, 40 / 56 B/pt
  KF_RESTRICT,     // Z^T, 20 B per fine pt
  KF_PROLONG,      // Z, 20 (36 with base) B per fine pt
  KF_MGS_COOP,     // one-launch MGS step, 16 (j + 1) + 32 B/pt
  KF_MGS_CHAIN,    // fused MGS launches of the chain, 32-64 B/pt each
  KF_BLAS,         // dot / norm / scale / add / axpy / lincomb
  KF_RESIDENT,     // device-resident GMRES solves (bytes from their iteration counts)
  KF_CONTROL,      // Givens, least squares, guards, flags (no field traffic)
  KF_GEMV,         // dense inverse at the multigrid bottom, 16 n^2 B
  KF_RESRESTRICT,  // fused MG residual + restriction, 44 B per fine pt
  KF_COUNT
};
const char* kfam_name(int f);

struct KProf {
  bool on = false;                 // record an event pair around every launch
  double bytes[KF_COUNT] = {};     // always accumulated
  long long n[KF_COUNT] = {};
  double ms[KF_COUNT] = {};        // resolved event time (armed only)
  struct Rec { int fam; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get();
  void resolve();                  // wait for the recorded pairs, add their times
  void reset();
  double total_bytes() const {
    double t = 0;
    for (double b : bytes) t += b;
    return t;
  }
};

// algorithmic bytes of one GMRES solve of m iterations on n points, counted the
// way the reference's algorithm streams its vectors (krylov.py:92-176): ||b||
// and V0 (48), per iteration a stencil (40) and the MGS chain 16 (j + 1) + 32,
// the solution update 16 (m + 1) and the true residual (40 + 32)
double gmres_alg_bytes(long long n, int m);

struct Engine {
  int device = 0;
  cudaStream_t st = nullptr;      // stream all work is ordered on (may be external)
  cudaStream_t own_st = nullptr;  // the stream created by the engine
  RedWS red;
  cd* dscal = nullptr;   // device scalars
  cd* hscal = nullptr;   // pinned host mirror
  size_t bytes_alloc = 0;
  long long launches = 0;  // kernels launched through the engine (telemetry)
  long long syncs = 0;     // host synchronisations (Hessenberg reads etc.)
  Comm* comm = nullptr;    // row-slab communicator of this rank (owned), null on one rank
  cd *rowpart = nullptr, *rowfull = nullptr;  // per-row partials (local rows / all ranks' rows)
  int row_cap = 0;
  cd* rows(int nyg);       // ensures both hold nyg entries, returns rowpart
  KProf kp;                // launch accounting / optional per-launch timing
  bool debug_sync = false; // HDB_DEBUG_SYNC=1: synchronise and check after every launch (fault location)
  void check_after(int fam);
  // run `f` (which enqueues `nl` kernels of family `fam` moving `bytes`
  // algorithmic bytes) with optional event timing around it
  template <class F>
  void kl(int fam, double bytes, F&& f, int nl = 1) {
    cudaEvent_t a = nullptr;
    if (kp.on) {
      a = kp.get();
      cudaEventRecord(a, st);
    }
    f();
    if (debug_sync) check_after(fam);
    launches += nl;
    kp.bytes[fam] += bytes;
    kp.n[fam] += nl;
    if (a) {
      cudaEvent_t b = kp.get();
      cudaEventRecord(b, st);
      kp.recs.push_back({fam, a, b});
      if (kp.recs.size() > 40000) kp.resolve();
    }
  }

  explicit Engine(int dev);
  ~Engine();
  cd* alloc(long long n);              // complex vector
  void* alloc_bytes(size_t b);
  void free(void* p);
  // vector with `halo` elements before and after (slab halo rows); returns the interior pointer
  cd* alloc_h(long long n, long long halo) { return alloc(n + 2 * halo) + halo; }
  void free_h(cd* p, long long halo) {
    if (p) free(p - halo);
  }
  void sync() { HDB_CUDA(cudaStreamSynchronize(st)); }
  // read slots [0, count) to host (one copy + sync) and raise on a fired device flag
  void fetch(int count);
  double fetch_norm(int slot);  // sqrt(max(re,0)) of a slot, after fetch
};

Engine& engine();            // the calling thread's engine, else the process-wide one
void engine_init(int device);
bool engine_ready();
void thread_engine_begin(int device);  // give the calling thread its own engine (rank threads)
void thread_engine_end();

struct Stop {
  double rel_tol;
  int max_iters;
};

struct KReport {
  int iterations = 0;
  double final_relres = 0.0;
  std::vector<double> history;
  bool converged = false;
};

// one level operator (A or CSLP M) on device; a slab of rows when sharded
struct LevelOp {
  OpCoef c;
  Geom g;
  double* ksq = nullptr;  // device, (ny + 2H) * nx, interior pointer
  long long n = 0;        // local points
  int H = 0;              // halo rows allocated around this level's vectors
  bool sharded = false;
  std::vector<int> slab_row0, slab_ny;  // every rank's slab (sharded levels)
  long long halo_elems() const { return (long long)H * g.nx; }
  void exchange(const cd* u, int rows) const;  // fill `rows` halo rows of u from the neighbours
  void apply(const cd* u, cd* out) const;                 // out = A u
  void residual(const cd* b, const cd* u, cd* out) const;  // out = b - A u
  void jacobi(const cd* x, const cd* b, cd* out, double omega, bool from_zero) const;
  // one sweep writing out = Jacobi(x) and out2 = out + addt (large radius-1 levels)
  bool jacobi_add_ok() const;
  void jacobi_add(const cd* x, const cd* b, cd* out, double omega, const cd* addt, cd* out2) const;
  // slot = (||b - A u||^2, ||b||^2), reduced over the distribution; `scratch`
  // (a level vector) is used only by the unfused radius-2/3 form
  void resnorm(const cd* b, const cd* u, cd* slot, cd* scratch) const;
  // reductions over this level's distribution (all-reduce when sharded)
  void reduce(cd* dev_slot) const;
  // rank-count-invariant mode: the engine's row partials of this level (all ranks' rows
  // gathered in global row order when sharded) summed in a fixed order into the slot
  void finish_rows(cd* dev_slot) const;
};

// rank-count-invariant reductions (HDB_PINV=1 / hdb_option("pinv", 1)); see engine.cu
bool pinv_mode();
void set_pinv(int on);
// <u, v>, the fused MGS step and ||b - t||^2 of a level, reduced over its distribution:
// flat kernels + all-reduce, or the row-ordered form in the invariant mode (L may be null:
// a vector without grid geometry)
void red_dot(const LevelOp* L, const cd* u, const cd* v, long long n, cd* slot);
void red_mgs(const LevelOp* L, cd* w, const cd* vi, const cd* hsrc, const cd* vn, long long n, cd* slot, double bytes);
void red_subnorm(const LevelOp* L, const cd* b, const cd* t, long long n, cd* slot);

using LinOp = std::function<void(const cd* in, cd* out)>;

// Krylov workspace: basis vectors grow on demand and are kept across calls
struct KWS {
  long long n = 0;
  long long halo = 0;      // halo elements around every basis vector (sharded levels)
  std::vector<cd*> V, Z;
  cd** dV = nullptr;       // device table of V pointers (cooperative MGS)
  cd** hvtab = nullptr;    // its pinned host mirror (the copy source)
  int dV_cap = 0, dV_n = 0;
  cd* gpart = nullptr;     // grid-reduction partials
  cd* tg = nullptr;        // T = (I + L)^{-1} rows of the low-synchronisation MGS (mgs_ls_tg_elems())
  cd* tgh = nullptr;       // the same for the HBM-streaming form (cap + 1)(cap + 2) / 2
  cd* lpart = nullptr;     // its block partials (lsh_part_elems)
  int tgh_cap = 0;
  cd* tmp = nullptr;
  cd** dbasis = nullptr;   // device pointer table for the solution update
  cd* dbasis0 = nullptr;   // the vector dbasis[0] currently points to on the device (one-step path cache)
  cd* dy = nullptr;
  cd** hbasis = nullptr;   // pinned staging
  cd* hy = nullptr;
  int cap = 0;
  cd* gst = nullptr;       // device-driven GMRES state (gmres_device)
  int gst_cap = 0;
  int* hflags = nullptr;   // pinned copy of its {done, its} flags
  int last_its = 0;        // previous solve's count: sizes the first launch batch
  void ensure(long long n_, int cap_, bool flexible);
  cd* v(int i);
  cd* z(int i);
  ~KWS();
};

// right-preconditioned unrestarted FGMRES (krylov.py:61-177); M == nullptr -> GMRES.
// `dist` (may be null) distributes the vectors: its reductions all-reduce.
KReport fgmres(long long n, const LinOp& A, const LinOp* M, const cd* b, cd* x, Stop stop, KWS& ws,
               const std::function<void(int, double)>* hook = nullptr, const cd* x0 = nullptr,
               const LevelOp* dist = nullptr);

// Unpreconditioned GMRES with zero guess driven from the device (large,
// unsharded levels whose MGS step runs as one cooperative launch): Arnoldi
// steps are enqueued in batches, Givens/stopping/least squares run on device
// and the host reads one flag per batch instead of a column per step.  The
// count and true relative residual land in *its_dev / *rel_dev.  Returns false
// (nothing launched) when the level does not qualify.
bool gmres_device(const LevelOp* op, const cd* b, cd* x, Stop stop, KWS& ws, int* its_dev, double* rel_dev);

// One-iteration FGMRES (StopRule tol >= 1, zero guess) entirely on device: no host
// synchronisation; the iteration count lands in *its_dev, failures raise the
// device flag (checked at the next host read).  Same arithmetic as fgmres().
void fgmres_step1(long long n, const LinOp& A, const LinOp& M, const cd* b, cd* x, KWS& ws, int* its_dev,
                  const LevelOp* dist, int level);

// Bi-CGSTAB workspace and solver (krylov.py:185-276); on breakdown *breakdown is
// set and x holds the best iterate (the caller decides, as madp.py:293-297 does)
struct BWS {
  long long n = 0, halo = 0;
  cd *r = nullptr, *rhat = nullptr, *p = nullptr, *v = nullptr, *s = nullptr, *t = nullptr, *ph = nullptr,
     *sh = nullptr, *tmp = nullptr;
  void ensure(long long n_);
  ~BWS();
};
KReport bicgstab(long long n, const LinOp& A, const LinOp* M, const cd* b, cd* x, Stop stop, BWS& ws,
                 const cd* x0, const LevelOp* dist, bool* breakdown, std::string* why);

// Krylov solves on levels that fit the resident working set run as ONE
// device-resident launch (kernels_resident.cu): cluster mode up to
// HDB_SMALL_N points (default 12k), whole-grid cooperative mode up to
// HDB_GRID_N points (default 2M) when the stencil windows fit shared memory.
// 0 disables a mode.
int resident_mode(long long n, int cap);  // -1: launch-driven path
int resident_ortho();  // HDB_ORTHO=auto|dgks|ls|cgs2|mgs for device-resident solves (launch_resident_gmres codes)
long long coop_mgs_min();  // levels >= this many points use the one-launch MGS step (HDB_COOP_MGS_N)
bool step1_enabled();  // HDB_STEP1=0 forces the host-driven path for one-iteration FGMRES

struct SmallSolve {  // device-resident GMRES on one level operator
  const LevelOp* op = nullptr;
  cd* basis = nullptr;
  cd* Rg = nullptr;
  cd* gpart = nullptr;
  int cap = 0;
  void ensure(const LevelOp* o, int cap_);
  // launches if the problem fits a resident mode (false: use the launch path);
  // iteration count lands in *its_dev, final relres in *rel_dev
  bool try_run(const cd* b, cd* x, Stop stop, int* its_dev, double* rel_dev);
  ~SmallSolve();
};

// coarse rows [row0, row0 + ny) a rank restricts (then all-gathers) when a sharded
// level feeds a replicated one (host rule; exported as hdb_plan_gather_rows)
void gather_rows(const std::vector<int>& fine_slab_row0, int rank, int ncy_g, int& row0, int& ny);
// slab-to-slab / slab-to-replicated transfer between two levels
TGeom level_tgeom(const LevelOp& fine, const LevelOp& coarse);
// restrict fine (level op f) into coarse buffer `out` of level op c; gathers into
// the full vector when c is replicated and f sharded (`slab` = local scratch)
void restrict_levels(const LevelOp& f, const LevelOp& c, const cd* fine, cd* out, cd* slab, int zero_mask);
// prolong coarse (level op c) into fine (level op f), base != null: fine = base + Z coarse
void prolong_levels(const LevelOp& c, const LevelOp& f, const cd* coarse, const cd* base, cd* fine);

struct Multigrid {
  std::vector<const LevelOp*> ops;  // sub-levels, finest first
  std::vector<cd*> X, Y, R, B, O, S;  // per-level scratch (X,Y,R), rhs (B), output (O), gather slab (S)
  cd* Ainv = nullptr;               // coarsest dense inverse (n <= direct limit)
  int ninv = 0;
  KWS coarse_ws;
  SmallSolve small_coarse;
  Stop coarse_stop{1e-8, 50};
  double omega = 0.8, guard = 10.0;
  int pre = 1, post = 1;
  void setup();
  // mg.py:125-139 (guard -> device flag); xsum != null: also xsum = x + addt (folded into
  // the last post-smoothing sweep; needs can_fold_sum())
  void vcycle(const cd* b, cd* x, const cd* x0 = nullptr, const cd* addt = nullptr, cd* xsum = nullptr);
  void cycle(int i, const cd* b, cd* x, const cd* x_init, const cd* addt = nullptr, cd* xsum = nullptr);
  bool can_fold_sum() const;
  ~Multigrid();
};

enum { CSLP_NONE = 0, CSLP_MG = 1, CSLP_GMRES = 2, CSLP_BICGSTAB = 3 };

struct MadpLevel {
  const LevelOp* A = nullptr;
  const LevelOp* M = nullptr;
  Multigrid* mg = nullptr;
  int cslp = CSLP_NONE;
  Stop cslp_stop{0.1, 1}, cycle_stop{1.0, 1};
  KWS ws_defl, ws_cslp;
  BWS ws_bicg;
  SmallSolve small_cslp;
  cd *vhat = nullptr, *vtil = nullptr;            // this level's input / output as a deflation system
  cd *t = nullptr, *rhs = nullptr, *r = nullptr;  // A-DEF1 temporaries of P_l
  cd* slab = nullptr;                             // restriction slab before a gather (replicated level)
  cd *bh = nullptr, *xh = nullptr;                // level-1 halo'd copies of b and x (sharded solves)
};

// inclusive host wall time per level and role (telemetry for DESIGN.md / profiles/)
enum { PROF_DEFL = 0, PROF_CSLP = 1, PROF_ADEF = 2, PROF_KINDS = 3 };

struct SolveReport {
  KReport outer;
  std::vector<double> prof_ms;        // (ml+1) * PROF_KINDS
  std::vector<double> dev_ms;         // same layout, device time from CUDA events (HDB_PROFILE=1)
  std::vector<long long> prof_calls;  // same layout
  long long syncs = 0, launches = 0;
  std::vector<std::vector<int>> cycle_iters, cslp_iters;  // index = level
  std::vector<long long> matvecs;
  std::vector<double> iter_wall_ms;
  double wall_ms = 0.0;
  double alg_bytes = 0.0;  // algorithmic HBM bytes of the solve's launches (KProf counters)
};

struct MadpSolver {
  int ml = 0;
  int* dcounts = nullptr;      // device iteration counts of device-resident solves
  double* drel = nullptr;
  int dcap = 0, dused = 0;
  std::vector<std::pair<int, int>> pending;  // (level, index into cslp_iters[level]) per slot
  std::vector<long long> slot_npts;          // points of a device-resident solve's level (bytes at flush), else 0
  void flush_counts();
  // device timing (HDB_PROFILE=1): event pairs per (level, kind), resolved at the end of a solve
  struct EvRec { int slot; cudaEvent_t a, b; };
  std::vector<EvRec> evs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t ev_get();
  void ev_resolve();
  int reserve_count(int level);
  void unreserve_count(int level);
  std::vector<MadpLevel> lv;  // index 1..ml
  Stop outer{1e-6, 150};
  SolveReport rep;
  void set_levels(int ml_);
  void reset_report();
  void setup();
  // out = CSLP_l(rhs); sum != null: also sum = out + addt (the A-DEF1 r + t)
  void cslp_apply(int l, const cd* rhs, cd* out, const cd* addt = nullptr, cd* sum = nullptr);
  void cslp_krylov(int l, const cd* rhs, cd* out);
  void precond(int l, const cd* v, cd* out);
  void A(int l, const cd* u, cd* out);
  void solve(const cd* b, cd* x);
  ~MadpSolver();
};

}  // namespace hdb
