// Device-resident GMRES for small levels: one thread-block cluster runs a whole
// unrestarted GMRES solve (krylov.py:61-177 with apply_M = None) — operator
// applies, modified Gram-Schmidt, Givens rotations, stopping test, least
// squares, solution update and the explicit final residual — in ONE launch.
//
// Why: on levels of <= ~70k points every Krylov step of the launch-driven
// engine costs a kernel launch per MGS coefficient plus one host round trip
// for the Hessenberg column (measured 168 us per GMRES iteration on the 65^2
// level of BASELINE config 2, profiles/).  Here a step costs one cluster
// barrier + a DSMEM reduction.
//
// Layout: CTA r of the cluster owns the flat point range [r*N/C, (r+1)*N/C);
// every thread keeps the same points for all element-wise work, so only the
// stencil (which reads other CTAs' points through L2) and the reductions
// need cluster barriers.  Reductions are deterministic: fixed warp/block tree,
// then the C CTA partials are combined in rank order by every CTA.
// Arithmetic of stencils and vector updates is the same as the launch path.
#include <cooperative_groups.h>

#include "kernels.h"
#include "stencil.cuh"

namespace cg = cooperative_groups;

namespace hdb {

constexpr int kCT = 512;        // threads per CTA
constexpr int kMaxCap = 128;    // iteration cap supported by the device solver

struct SmallKrylovArgs {
  OpCoef c;
  Geom g;
  const double* ksq;
  const cd* b;
  cd* x;
  cd* basis;          // (cap + 1) vectors of n points
  long long n;
  double tol;
  int cap;
  int* its_out;       // iteration count
  double* relres_out; // final true relative residual
  cd* flag;           // .x = 2.0 on a non-finite value (NumericalError)
};

template <int R>
__device__ __forceinline__ cd op_point(const OpCoef& c, const Geom& g, const cd* u, const double* k, int gj, int i) {
  const long long p = (long long)(gj - g.row0) * g.nx + i;
  if (pinned(g, c, gj, i)) return u[p];
  if (R == 1) {
    return five_point(c.s, c.mc, k[p], u[p], upad(u, k, g, c, gj, i - 1), upad(u, k, g, c, gj, i + 1),
                      upad(u, k, g, c, gj - 1, i), upad(u, k, g, c, gj + 1, i));
  }
  constexpr int N = 2 * R + 1;
  cd acc = mkc(0.0, 0.0);
#pragma unroll 1
  for (int a = 0; a < N; ++a) {
#pragma unroll
    for (int bb = 0; bb < N; ++bb) {
      const int jj = gj + a - R, ii = i + bb - R;
      const double kp = kpad(k, g, c, jj, ii);
      const cd m = c.mass[a * N + bb];
      const cd coef = mkc(__dadd_rn(c.lap[a * N + bb], __dmul_rn(m.x, kp)), __dmul_rn(m.y, kp));
      acc = c_add(acc, c_mul(coef, upad(u, k, g, c, jj, ii)));
    }
  }
  return acc;
}

struct CSmem {
  cd warp[kCT / 32];
  cd part[2];        // this CTA's partial (double-buffered across reductions)
  cd bcast[2];
  cd hcol[kMaxCap + 2];
  cd sn[kMaxCap];
  double cs[kMaxCap];
  cd g[kMaxCap + 2];
  cd y[kMaxCap];
  cd R[kMaxCap * (kMaxCap + 1) / 2];  // packed upper triangle, column-major
  int decision;
  double rel;
};

__device__ __forceinline__ cd warp_sum_c(cd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// deterministic cluster-wide sum; every thread of every CTA returns the same value
__device__ cd cluster_sum(cd v, CSmem& s, int& buf, cg::cluster_group& cl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum_c(v);
  if (lane == 0) s.warp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    cd t = lane < kCT / 32 ? s.warp[lane] : mkc(0.0, 0.0);
    t = warp_sum_c(t);
    if (lane == 0) s.part[buf] = t;
  }
  cl.sync();
  if (wid == 0) {
    const int C = (int)cl.num_blocks();
    cd t = mkc(0.0, 0.0);
    if (lane < C) t = *cl.map_shared_rank(&s.part[buf], lane);
    t = warp_sum_c(t);
    if (lane == 0) s.bcast[buf] = t;
  }
  __syncthreads();
  const cd r = s.bcast[buf];
  buf ^= 1;
  return r;
}

__device__ __forceinline__ double cabs_(cd z) { return hypot(z.x, z.y); }
__device__ __forceinline__ cd cmul_(cd a, cd b) { return mkc(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cd cdiv_(cd a, cd b) {
  const double d = b.x * b.x + b.y * b.y;
  if (fabs(b.y) == 0.0) return mkc(a.x / b.x, a.y / b.x);
  return mkc((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ cd conj_(cd a) { return mkc(a.x, -a.y); }

template <int R>
__global__ void __launch_bounds__(kCT) k_small_gmres(SmallKrylovArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CSmem& s = *reinterpret_cast<CSmem*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const long long n = A.n;
  const long long p0 = n * rank / C, p1 = n * (rank + 1) / C;
  const int t = threadIdx.x;
  const int nx = A.g.nx;
  int buf = 0;
  auto V = [&](int i) { return A.basis + (long long)i * n; };

  // ||b||
  cd acc = mkc(0.0, 0.0);
  for (long long p = p0 + t; p < p1; p += kCT) acc = c_conjmul_acc(acc, A.b[p], A.b[p]);
  const double bnorm = sqrt(fmax(cluster_sum(acc, s, buf, cl).x, 0.0));
  if (bnorm == 0.0) {  // krylov.py:96-97
    for (long long p = p0 + t; p < p1; p += kCT) A.x[p] = mkc(0.0, 0.0);
    if (rank == 0 && t == 0) { *A.its_out = 0; *A.relres_out = 0.0; }
    return;
  }
  if (!isfinite(bnorm)) {
    if (rank == 0 && t == 0) { A.flag->x = 2.0; *A.its_out = 0; }
    return;
  }
  const double beta = bnorm;  // r0 = b; rel = 1 never triggers the tol < 1 early exit
  {
    const double inv = 1.0 / beta;
    cd* v0 = V(0);
    for (long long p = p0 + t; p < p1; p += kCT) {
      const cd q = A.b[p];
      v0[p] = mkc(__dmul_rn(q.x, inv), __dmul_rn(q.y, inv));
    }
  }
  if (t == 0) s.g[0] = mkc(beta, 0.0);
  int its = 0;
  for (int j = 0; j < A.cap; ++j) {
    cl.sync();  // V_j complete everywhere
    const cd* vj = V(j);
    cd* w = V(j + 1);
    for (long long p = p0 + t; p < p1; p += kCT) {
      const int gj = (int)(p / nx), i = (int)(p % nx);
      w[p] = op_point<R>(A.c, A.g, vj, A.ksq, gj + A.g.row0, i);
    }
    // modified Gram-Schmidt (krylov.py:121-124): h_i = <V_i, w>; w -= h_i V_i
    for (int i = 0; i <= j; ++i) {
      const cd* vi = V(i);
      cd a = mkc(0.0, 0.0);
      for (long long p = p0 + t; p < p1; p += kCT) a = c_conjmul_acc(a, vi[p], w[p]);
      const cd h = cluster_sum(a, s, buf, cl);
      if (t == 0) s.hcol[i] = h;
      for (long long p = p0 + t; p < p1; p += kCT) w[p] = c_sub(w[p], c_mul_np(h, vi[p]));
    }
    cd a = mkc(0.0, 0.0);
    for (long long p = p0 + t; p < p1; p += kCT) a = c_conjmul_acc(a, w[p], w[p]);
    const double hn = sqrt(fmax(cluster_sum(a, s, buf, cl).x, 0.0));
    if (t == 0) {
      // rotations (krylov.py:126-151), same in every CTA
      cd* col = s.hcol;
      col[j + 1] = mkc(hn, 0.0);
      bool finite = true;
      for (int i = 0; i <= j + 1; ++i) finite &= isfinite(col[i].x) && isfinite(col[i].y);
      for (int i = 0; i < j; ++i) {
        const cd tt = mkc(s.cs[i] * col[i].x + cmul_(s.sn[i], col[i + 1]).x,
                          s.cs[i] * col[i].y + cmul_(s.sn[i], col[i + 1]).y);
        const cd nb = cmul_(mkc(-s.sn[i].x, s.sn[i].y), col[i]);
        col[i + 1] = mkc(nb.x + s.cs[i] * col[i + 1].x, nb.y + s.cs[i] * col[i + 1].y);
        col[i] = tt;
      }
      const cd h1 = col[j], h2 = col[j + 1];
      double c;
      cd sn;
      const double a1 = cabs_(h1), a2 = cabs_(h2);
      if (a2 == 0.0) { c = 1.0; sn = mkc(0.0, 0.0); }
      else if (a1 == 0.0) { c = 0.0; sn = mkc(1.0, 0.0); }
      else {
        const double tt = hypot(a1, a2);
        c = a1 / tt;
        const cd ph = mkc(h1.x / a1, h1.y / a1);
        const cd q = cmul_(ph, conj_(h2));
        sn = mkc(q.x / tt, q.y / tt);
      }
      s.cs[j] = c;
      s.sn[j] = sn;
      const cd top = mkc(c * h1.x + cmul_(sn, h2).x, c * h1.y + cmul_(sn, h2).y);
      col[j] = top;
      cd* Rc = s.R + j * (j + 1) / 2;
      for (int i = 0; i <= j; ++i) Rc[i] = col[i];
      const cd gj = s.g[j];
      s.g[j + 1] = cmul_(mkc(-sn.x, sn.y), gj);
      s.g[j] = mkc(c * gj.x, c * gj.y);
      const double rel = cabs_(s.g[j + 1]) / bnorm;
      s.rel = rel;
      s.decision = !finite ? 2 : ((hn < 1e-30 || rel <= A.tol) ? 1 : 0);
    }
    __syncthreads();
    its = j + 1;
    const int dec = s.decision;
    if (dec == 2) {
      if (rank == 0 && t == 0) { A.flag->x = 2.0; *A.its_out = its; }
      return;
    }
    if (dec == 1) break;
    const double inv = 1.0 / hn;
    for (long long p = p0 + t; p < p1; p += kCT) {
      const cd q = w[p];
      w[p] = mkc(__dmul_rn(q.x, inv), __dmul_rn(q.y, inv));
    }
  }
  // least squares (krylov.py:161-168)
  if (t == 0) {
    for (int i = its - 1; i >= 0; --i) {
      cd accy = s.g[i];
      for (int k = i + 1; k < its; ++k) {
        const cd r = s.R[k * (k + 1) / 2 + i];
        const cd pr = cmul_(r, s.y[k]);
        accy = mkc(accy.x - pr.x, accy.y - pr.y);
      }
      s.y[i] = cdiv_(accy, s.R[i * (i + 1) / 2 + i]);
    }
  }
  __syncthreads();
  for (long long p = p0 + t; p < p1; p += kCT) {
    cd xx = mkc(0.0, 0.0);
    for (int i = 0; i < its; ++i) xx = c_add(xx, c_mul_np(s.y[i], V(i)[p]));
    A.x[p] = xx;
  }
  cl.sync();  // x complete everywhere
  // explicit true residual (krylov.py:174)
  cd f = mkc(0.0, 0.0);
  for (long long p = p0 + t; p < p1; p += kCT) {
    const int gj = (int)(p / nx), i = (int)(p % nx);
    const cd d = c_sub(A.b[p], op_point<R>(A.c, A.g, A.x, A.ksq, gj + A.g.row0, i));
    f = c_conjmul_acc(f, d, d);
  }
  const double fin = sqrt(fmax(cluster_sum(f, s, buf, cl).x, 0.0)) / bnorm;
  if (rank == 0 && t == 0) {
    *A.its_out = its;
    *A.relres_out = fin;
    if (!isfinite(fin)) A.flag->x = 2.0;
  }
}

static int g_cluster = 0;  // chosen cluster size

template <int R>
static void launch_small_r(const SmallKrylovArgs& a, cudaStream_t st) {
  const size_t sm = sizeof(CSmem);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_small_gmres<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_small_gmres<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured = true;
  }
  if (g_cluster == 0) {
    for (int c : {16, 8, 4, 2, 1}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(c); cfg.blockDim = dim3(kCT); cfg.dynamicSmemBytes = sm; cfg.attrs = at; cfg.numAttrs = 1;
      int num = 0;
      if (cudaOccupancyMaxActiveClusters(&num, k_small_gmres<R>, &cfg) == cudaSuccess && num > 0) {
        g_cluster = c;
        break;
      }
      cudaGetLastError();
    }
    if (g_cluster == 0) g_cluster = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g_cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(g_cluster);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_small_gmres<R>, a);
}

int small_gmres_max_cap() { return kMaxCap; }
int small_gmres_cluster() { return g_cluster; }

void launch_small_gmres(const OpCoef& c, const Geom& g, const double* ksq, const cd* b, cd* x, cd* basis,
                        long long n, double tol, int cap, int* its_out, double* relres_out, cd* flag,
                        cudaStream_t st) {
  SmallKrylovArgs a;
  a.c = c; a.g = g; a.ksq = ksq; a.b = b; a.x = x; a.basis = basis; a.n = n; a.tol = tol; a.cap = cap;
  a.its_out = its_out; a.relres_out = relres_out; a.flag = flag;
  if (c.radius == 1) launch_small_r<1>(a, st);
  else if (c.radius == 2) launch_small_r<2>(a, st);
  else launch_small_r<3>(a, st);
}

}  // namespace hdb
