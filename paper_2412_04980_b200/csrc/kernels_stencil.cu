// Level-operator kernels: radius-1 (5-point) and radius-2/3 (Galerkin 5x5 /
// 7x7) matrix-free applies with fused epilogues, and damped Jacobi.
//
// Reference: _kernels.py:14-68, operators.py:130-178, mg.py:88-102.
// Memory-bound: 40 B/pt algorithmic for an apply (u 16 + k^2 8 + out 16),
// 56 B/pt for the residual / A-DEF1 form (+ b 16), 56 B/pt per Jacobi sweep.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "stencil.cuh"
#include "reduce.cuh"

namespace hdb {

// ------------------------------------------------------------------------
// radius 1.  One thread per point; neighbours come through L1 (32x8 tiles).
// mode 0: out = A u            (pinned rows: u)
// mode 1: out = b - A u        (pinned rows: b - u)          [residual / A-DEF1]
// mode 2: out = u + (w dinv)(b - A u)   (pinned: u + w(b - u)) [Jacobi sweep]
// mode 3: out = (w dinv) b     (pinned: w b)                  [Jacobi from x = 0]
// ------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(256) k_r1(const cd* __restrict__ u, const cd* __restrict__ b,
                                            const double* __restrict__ k, cd* __restrict__ out,
                                            Geom g, OpCoef c, double omega) {
  if (c.skip && *c.skip) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;  // local row
  if (i >= g.nx || j >= g.ny) return;
  const int gj = j + g.row0;
  const long long p = (long long)j * g.nx + i;
  if (MODE == 3) {
    const cd bb = b[p];
    if (pinned(g, c, gj, i)) { out[p] = c_scale(omega, bb); return; }
    const cd d = dinv_at(k, g, c, gj, i);
    out[p] = c_mul(c_scale(omega, d), bb);
    return;
  }
  const cd uc = u[p];
  if (pinned(g, c, gj, i)) {
    if (MODE == 0) out[p] = uc;
    else if (MODE == 1) out[p] = c_sub(b[p], uc);
    else out[p] = c_add(uc, c_scale(omega, c_sub(b[p], uc)));
    return;
  }
  const cd w = upad(u, k, g, c, gj, i - 1);
  const cd e = upad(u, k, g, c, gj, i + 1);
  const cd so = upad(u, k, g, c, gj - 1, i);
  const cd no = upad(u, k, g, c, gj + 1, i);
  const cd Au = five_point(c.s, c.mc, k[p], uc, w, e, so, no);
  if (MODE == 0) { out[p] = Au; return; }
  const cd r = c_sub(b[p], Au);
  if (MODE == 1) { out[p] = r; return; }
  const cd d = dinv_at(k, g, c, gj, i);
  out[p] = c_add(uc, c_mul(c_scale(omega, d), r));
}

// ------------------------------------------------------------------------
// radius 1, column-strip form (the hot fine-level kernel).  A warp owns 32
// consecutive columns; each thread walks RB rows keeping rows j-1, j, j+1 of
// its column in registers (one new row load per output row); W/E come from
// lane shuffles (edge lanes load their outer neighbour).  Blocks that touch a
// physical boundary or a slab edge take the per-point closure path.  Same
// arithmetic as k_r1 (bit-identical).
// interior Jacobi reciprocal 1 / (4s + mc k^2) (no Sommerfeld terms), numpy's
// Smith division (same operations as dinv_at)
__device__ __forceinline__ cd interior_dinv(const OpCoef& c, double kc) {
  const double dr = __dadd_rn(4.0 * c.s, __dmul_rn(c.mc.x, kc)), di = __dmul_rn(c.mc.y, kc);
  if (fabs(dr) >= fabs(di)) {
    const double rat = __ddiv_rn(di, dr), scl = __ddiv_rn(1.0, __dadd_rn(dr, __dmul_rn(di, rat)));
    return mkc(scl, __dmul_rn(-rat, scl));
  }
  const double rat = __ddiv_rn(dr, di), scl = __ddiv_rn(1.0, __dadd_rn(di, __dmul_rn(dr, rat)));
  return mkc(__dmul_rn(rat, scl), -scl);
}

constexpr int SX = 32, SY = 4, RB = 16;  // block 32x4 threads, 16 rows per thread

// one output by the per-point closure path (boundaries, ragged edges, pinned rows)
// MODE 4: the Jacobi sweep of MODE 2 plus a second output out2 = result + addt
// (the A-DEF1 sum r + t, madp.py:327, folded into the last post-smoothing sweep)
template <int MODE>
__device__ __forceinline__ void r1_point(const cd* __restrict__ u, const cd* __restrict__ b,
                                         const double* __restrict__ k, cd* __restrict__ out, const Geom& g,
                                         const OpCoef& c, double omega, int i, int j,
                                         const cd* __restrict__ addt = nullptr, cd* __restrict__ out2 = nullptr) {
  const int gj = j + g.row0;
  const long long p = (long long)j * g.nx + i;
  if (MODE == 3) {
    const cd bb = b[p];
    if (pinned(g, c, gj, i)) { out[p] = c_scale(omega, bb); return; }
    out[p] = c_mul(c_scale(omega, dinv_at(k, g, c, gj, i)), bb);
    return;
  }
  const cd uc = u[p];
  if (pinned(g, c, gj, i)) {
    if (MODE == 0) out[p] = uc;
    else if (MODE == 1) out[p] = c_sub(b[p], uc);
    else {
      const cd res = c_add(uc, c_scale(omega, c_sub(b[p], uc)));
      out[p] = res;
      if (MODE == 4) out2[p] = c_add(res, addt[p]);
    }
    return;
  }
  const cd Au = five_point(c.s, c.mc, k[p], uc, upad(u, k, g, c, gj, i - 1), upad(u, k, g, c, gj, i + 1),
                           upad(u, k, g, c, gj - 1, i), upad(u, k, g, c, gj + 1, i));
  if (MODE == 0) { out[p] = Au; return; }
  const cd r1 = c_sub(b[p], Au);
  if (MODE == 1) { out[p] = r1; return; }
  const cd res = c_add(uc, c_mul(c_scale(omega, dinv_at(k, g, c, gj, i)), r1));
  out[p] = res;
  if (MODE == 4) out2[p] = c_add(res, addt[p]);
}

// rows [j0, j0 + n) of column i by the sliding window: no closure, no pinning
// (the caller guarantees every point and its neighbours exist).  The whole
// warp runs the same rows (E/W come from lane shuffles).
template <int MODE, int UNR>
__device__ __forceinline__ void r1_run(const cd* __restrict__ u, const cd* __restrict__ b,
                                       const double* __restrict__ k, cd* __restrict__ out, const Geom& g,
                                       const OpCoef& c, double omega, int i, int j0, int n,
                                       const cd* __restrict__ addt = nullptr, cd* __restrict__ out2 = nullptr) {
  if (n <= 0) return;
  const int lane = threadIdx.x;
  const long long nx = g.nx;
  const cd* up = u + (long long)j0 * nx + i;
  if (MODE == 3) {
    const double* kp = k + (long long)j0 * nx + i;
    const cd* bp = b + (long long)j0 * nx + i;
    cd* op = out + (long long)j0 * nx + i;
    // the reciprocal depends on k^2 only: reuse it while k^2 repeats down the
    // column (constant and layered models), bit-identical either way
    double klast = kp[0];
    cd dlast = interior_dinv(c, klast);
#pragma unroll 4
    for (int r = 0; r < n; ++r) {
      const double kc = kp[r * nx];
      if (kc != klast) { klast = kc; dlast = interior_dinv(c, kc); }
      op[r * nx] = c_mul(c_scale(omega, dlast), bp[r * nx]);
    }
    return;
  }
  // software pipeline: row r+1's loads are issued before row r is computed
  const double* kp = k + (long long)j0 * nx + i;
  const cd* bp = b ? b + (long long)j0 * nx + i : nullptr;
  cd* op = out + (long long)j0 * nx + i;
  cd s_ = up[-nx], c_ = up[0], n_ = up[nx];
  double kc = kp[0];
  cd bc = (MODE != 0) ? bp[0] : mkc(0.0, 0.0);
  cd wl = (lane == 0) ? up[-1] : mkc(0.0, 0.0), el = (lane == SX - 1) ? up[1] : mkc(0.0, 0.0);
  double klast = 0.0;
  cd dlast = mkc(0.0, 0.0);
  if (MODE == 2 || MODE == 4) { klast = kc; dlast = interior_dinv(c, kc); }
  const cd* tp = MODE == 4 ? addt + (long long)j0 * nx + i : nullptr;
  cd* o2 = MODE == 4 ? out2 + (long long)j0 * nx + i : nullptr;
#pragma unroll (UNR)
  for (int r = 0; r < n; ++r) {
    const long long o = (long long)r * nx;
    // prefetch row r+1 (its north row r+2, k, b, warp-edge neighbours)
    const bool more = r + 1 < n;
    cd n2 = mkc(0.0, 0.0), b2 = mkc(0.0, 0.0), wl2 = mkc(0.0, 0.0), el2 = mkc(0.0, 0.0);
    double k2 = 0.0;
    if (more) {
      n2 = up[o + 2 * nx];
      k2 = kp[o + nx];
      if (MODE != 0) b2 = bp[o + nx];
      if (lane == 0) wl2 = up[o + nx - 1];
      if (lane == SX - 1) el2 = up[o + nx + 1];
    }
    cd w_, e_;
    w_.x = __shfl_up_sync(0xffffffffu, c_.x, 1);
    w_.y = __shfl_up_sync(0xffffffffu, c_.y, 1);
    e_.x = __shfl_down_sync(0xffffffffu, c_.x, 1);
    e_.y = __shfl_down_sync(0xffffffffu, c_.y, 1);
    if (lane == 0) w_ = wl;
    if (lane == SX - 1) e_ = el;
    const cd Au = five_point(c.s, c.mc, kc, c_, w_, e_, s_, n_);
    if (MODE == 0) {
      op[o] = Au;
    } else {
      const cd r1 = c_sub(bc, Au);
      if (MODE == 1) {
        op[o] = r1;
      } else {
        if (kc != klast) { klast = kc; dlast = interior_dinv(c, kc); }
        const cd res = c_add(c_, c_mul(c_scale(omega, dlast), r1));
        op[o] = res;
        if (MODE == 4) o2[o] = c_add(res, tp[o]);
      }
    }
    s_ = c_;
    c_ = n_;
    n_ = n2;
    kc = k2;
    bc = b2;
    wl = wl2;
    el = el2;
  }
}

template <int MODE>
__global__ void __launch_bounds__(SX * SY, MODE == 2 ? 5 : (MODE == 1 ? 6 : 8)) k_r1s(const cd* __restrict__ u, const cd* __restrict__ b,
                                                 const double* __restrict__ k, cd* __restrict__ out, Geom g,
                                                 OpCoef c, double omega) {
  if (c.skip && *c.skip) return;
  const int i = blockIdx.x * SX + threadIdx.x;
  const int jbeg = (blockIdx.y * SY + threadIdx.y) * RB;  // local row
  const int gi0 = blockIdx.x * SX, gj0 = g.row0 + blockIdx.y * SY * RB;
  const int gj1 = gj0 + SY * RB;  // exclusive
  const bool interior = gi0 >= 1 && gi0 + SX <= g.nx - 1 && gj0 >= 1 && gj1 <= g.nyg - 1 &&
                        blockIdx.y * SY * RB + SY * RB <= g.ny;
  if (!interior) {
    // generic per-point path (boundaries, ragged edges)
    if (i >= g.nx) return;
    for (int r = 0; r < RB; ++r) {
      const int j = jbeg + r;
      if (j >= g.ny) return;
      r1_point<MODE>(u, b, k, out, g, c, omega, i, j);
    }
    return;
  }
  r1_run<MODE, (MODE == 2 ? 2 : 4)>(u, b, k, out, g, c, omega, i, jbeg, RB);
}

// Same tiles as k_r1s with a run-time row count per thread (rb).  Shorter
// column runs are faster on the fine grids although each run re-reads its
// two halo rows (they hit L2: the block's other warps own them): measured
// (HDB_R1_RB sweep, profiles/r01e_r1_rows_sweep.txt) 4097^2 apply / residual
// 93.7 / 99.7 % of the copy peak at rb = 4 vs 83 / 91 % at rb = 16, 73.7 /
// 83 % at rb = 32; the Jacobi sweep (more registers, 5 CTAs/SM) peaks at rb = 8
// on 4097^2 and rb = 16 on 8193^2.
// The Jacobi form is held to 80 registers (6 CTAs/SM, 8 B of spill) -- measured
// faster than 94 registers at 5 CTAs/SM: 86.6 vs 83.4 % of the copy peak on
// 4097^2, 95.2 vs 91.8 % on 8193^2 (profiles/r01e_jacobi_occupancy.txt).
template <int MODE, int UNR>
__global__ void __launch_bounds__(SX * SY, (MODE == 1 || MODE == 2 || MODE == 4) ? 6 : 8) k_r1w(const cd* __restrict__ u, const cd* __restrict__ b,
                                                 const double* __restrict__ k, cd* __restrict__ out, Geom g,
                                                 OpCoef c, double omega, int rb,
                                                 const cd* __restrict__ addt = nullptr, cd* __restrict__ out2 = nullptr) {
  if (c.skip && *c.skip) return;
  const int i = blockIdx.x * SX + threadIdx.x;
  const int jbeg = (blockIdx.y * SY + threadIdx.y) * rb;  // local row
  const int gi0 = blockIdx.x * SX, gj0 = g.row0 + blockIdx.y * SY * rb;
  const int gj1 = gj0 + SY * rb;  // exclusive
  const bool interior = gi0 >= 1 && gi0 + SX <= g.nx - 1 && gj0 >= 1 && gj1 <= g.nyg - 1 &&
                        blockIdx.y * SY * rb + SY * rb <= g.ny;
  if (!interior) {
    if (i >= g.nx) return;
    const int je = min(jbeg + rb, g.ny);
    for (int j = jbeg; j < je; ++j) r1_point<MODE>(u, b, k, out, g, c, omega, i, j, addt, out2);
    return;
  }
  r1_run<MODE, UNR>(u, b, k, out, g, c, omega, i, jbeg, rb, addt, out2);
}

// ------------------------------------------------------------------------
// Fused residual norm (the MG divergence guard, mg.py:131-138, and any
// ||b - A u|| that only needs the norm): dst = (||b - A u||^2, ||b||^2) as one
// complex slot (re, im), read in one pass over u, b, k^2 (40 B/pt); the
// residual itself is never stored.  One block per 32 x (NRW*RBN) strip tile
// (interior tiles with the k_r1s sliding window, boundary tiles per point),
// per-tile partials in tile order, then one ordered sum (k_sum_partials):
// deterministic for a given grid.
constexpr int NRW = 4;  // warps per block (tile rows = NRW * RBN)
constexpr int RBN = 16;  // rows per warp (8 measured slower on 8193^2: 83 vs 90 % of peak)
__global__ void __launch_bounds__(32 * NRW) k_resnorm(const cd* __restrict__ u, const cd* __restrict__ b,
                                                      const double* __restrict__ k, Geom g, OpCoef c, cd* partials) {
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  double rr = 0.0, bb = 0.0;
  const long long nx = g.nx;
  const int bx = blockIdx.x, by = blockIdx.y;
  const int i = bx * 32 + lane;
  const int jbeg = (by * NRW + wy) * RBN;
  const int gi0 = bx * 32, gj0 = g.row0 + by * NRW * RBN, gj1 = gj0 + NRW * RBN;
  const bool interior = gi0 >= 1 && gi0 + 32 <= g.nx - 1 && gj0 >= 1 && gj1 <= g.nyg - 1 &&
                        by * NRW * RBN + NRW * RBN <= g.ny;
  if (!interior) {
    if (i < g.nx)
      for (int r = 0; r < RBN; ++r) {
        const int j = jbeg + r;
        if (j >= g.ny) break;
        const int gj = j + g.row0;
        const long long p = (long long)j * nx + i;
        const cd bc = b[p], uc = u[p];
        cd res;
        if (pinned(g, c, gj, i)) {
          res = c_sub(bc, uc);
        } else {
          const cd Au = five_point(c.s, c.mc, k[p], uc, upad(u, k, g, c, gj, i - 1), upad(u, k, g, c, gj, i + 1),
                                   upad(u, k, g, c, gj - 1, i), upad(u, k, g, c, gj + 1, i));
          res = c_sub(bc, Au);
        }
        rr = __fma_rn(res.x, res.x, rr); rr = __fma_rn(res.y, res.y, rr);
        bb = __fma_rn(bc.x, bc.x, bb); bb = __fma_rn(bc.y, bc.y, bb);
      }
  } else {
    const cd* up = u + (long long)jbeg * nx + i;
    const double* kp = k + (long long)jbeg * nx + i;
    const cd* bp = b + (long long)jbeg * nx + i;
    cd s_ = up[-nx], c_ = up[0], n_ = up[nx];
    double kc = kp[0];
    cd bc = bp[0];
    cd wl = (lane == 0) ? up[-1] : mkc(0.0, 0.0), el = (lane == 31) ? up[1] : mkc(0.0, 0.0);
#pragma unroll 4
    for (int r = 0; r < RBN; ++r) {
      const long long o = (long long)r * nx;
      const bool more = r + 1 < RBN;
      cd n2 = mkc(0.0, 0.0), b2 = mkc(0.0, 0.0), wl2 = mkc(0.0, 0.0), el2 = mkc(0.0, 0.0);
      double k2 = 0.0;
      if (more) {
        n2 = up[o + 2 * nx];
        k2 = kp[o + nx];
        b2 = bp[o + nx];
        if (lane == 0) wl2 = up[o + nx - 1];
        if (lane == 31) el2 = up[o + nx + 1];
      }
      cd w_, e_;
      w_.x = __shfl_up_sync(0xffffffffu, c_.x, 1);
      w_.y = __shfl_up_sync(0xffffffffu, c_.y, 1);
      e_.x = __shfl_down_sync(0xffffffffu, c_.x, 1);
      e_.y = __shfl_down_sync(0xffffffffu, c_.y, 1);
      if (lane == 0) w_ = wl;
      if (lane == 31) e_ = el;
      const cd res = c_sub(bc, five_point(c.s, c.mc, kc, c_, w_, e_, s_, n_));
      rr = __fma_rn(res.x, res.x, rr); rr = __fma_rn(res.y, res.y, rr);
      bb = __fma_rn(bc.x, bc.x, bb); bb = __fma_rn(bc.y, bc.y, bb);
      s_ = c_; c_ = n_; n_ = n2; kc = k2; bc = b2; wl = wl2; el = el2;
    }
  }
  const cd part = block_sum<32 * NRW>(mkc(rr, bb));
  if (threadIdx.x == 0) partials[(long long)by * gridDim.x + bx] = part;
}

// ordered sum of G partials (one block): thread t adds t, t + T, ... in order,
// then the fixed block tree
constexpr int kSumThreads = 1024;
__global__ void __launch_bounds__(kSumThreads) k_sum_partials(const cd* __restrict__ partials, long long G, cd* dst) {
  cd v = mkc(0.0, 0.0);
  for (long long q = threadIdx.x; q < G; q += kSumThreads) {
    const cd z = partials[q];
    v.x += z.x;
    v.y += z.y;
  }
  v = block_sum<kSumThreads>(v);
  if (threadIdx.x == 0) *dst = v;
}

// ------------------------------------------------------------------------
// radius 2/3: shared-memory tile of the ghost-closed u and k^2 windows, then
// the reference's row-major tap order (_kernels.py:44-50):
//   acc += (lap[o] + mass[o]*kpad) * upad
// mode 0: out = A u ; mode 1: out = b - A u (pinned rows: u / b - u)
// ------------------------------------------------------------------------
constexpr int TX = 32, TY = 8;

template <int R, int MODE>
__global__ void __launch_bounds__(TX * TY) k_rg(const cd* __restrict__ u, const cd* __restrict__ b,
                                               const double* __restrict__ k, cd* __restrict__ out,
                                               Geom g, OpCoef c) {
  if (c.skip && *c.skip) return;
  constexpr int W = TX + 2 * R, H = TY + 2 * R, N = 2 * R + 1;
  __shared__ cd su[H][W];
  __shared__ double sk[H][W];
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int t = tid; t < H * W; t += TX * TY) {
    const int ty = t / W, tx = t % W;
    const int gi = i0 + tx - R, gj = g.row0 + j0 + ty - R;
    const bool need = tile_row_needed(g, gj, R);
    su[ty][tx] = need ? upad(u, k, g, c, gj, gi) : mkc(0.0, 0.0);
    sk[ty][tx] = need ? kpad(k, g, c, gj, gi) : 0.0;
  }
  __syncthreads();
  const int i = i0 + threadIdx.x, j = j0 + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const int gj = j + g.row0;
  const long long p = (long long)j * g.nx + i;
  if (pinned(g, c, gj, i)) {
    const cd uc = su[threadIdx.y + R][threadIdx.x + R];
    out[p] = MODE == 0 ? uc : c_sub(b[p], uc);
    return;
  }
  cd acc = mkc(0.0, 0.0);
  // constant-k^2 level and a tile away from every boundary: every tap's k^2 is ku,
  // so the per-tap coefficient is the precomputed (identically rounded) ucoef
  const bool fast = c.uniform && i0 >= R && i0 + TX + R <= g.nx && g.row0 + j0 >= R &&
                    g.row0 + j0 + TY + R <= g.nyg && j0 + TY <= g.ny;  // (whole tile inside the slab)
  if (fast) {
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int bb = 0; bb < N; ++bb) acc = c_add(acc, c_mul(c.ucoef[a * N + bb], su[threadIdx.y + a][threadIdx.x + bb]));
    }
  } else {
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int bb = 0; bb < N; ++bb) {
        const double kp = sk[threadIdx.y + a][threadIdx.x + bb];
        const cd m = c.mass[a * N + bb];
        const cd coef = mkc(__dadd_rn(c.lap[a * N + bb], __dmul_rn(m.x, kp)), __dmul_rn(m.y, kp));
        acc = c_add(acc, c_mul(coef, su[threadIdx.y + a][threadIdx.x + bb]));
      }
    }
  }
  out[p] = MODE == 0 ? acc : c_sub(b[p], acc);
}

// Vertically register-blocked form (radius 3 on large grids): each thread owns
// the outputs (y, x) and (y+1, x).  Tile row r (r = 0 .. 2R+1) is loaded once
// (2R+1 values of u, and of k^2 on heterogeneous levels) and feeds tap row a = r
// of the upper output and a = r-1 of the lower one, so every output still
// receives its taps in the reference's row-major (a, b) order (bit-identical),
// while the shared-memory loads per output drop from (2R+1)^2 to
// (2R+2)(2R+1)/2.  Tile: 32 x 16 outputs (256 threads).  Four outputs per
// thread (17.5 loads per output) measured slower: 94 registers leave 20 warps
// per SM (41.0 vs 37.4 us on the 1025^2 level of config 2).
constexpr int VTY = 8, VROWS = 2 * VTY;
template <int R, int MODE>
__global__ void __launch_bounds__(TX * VTY) k_rgv(const cd* __restrict__ u, const cd* __restrict__ b,
                                                 const double* __restrict__ k, cd* __restrict__ out, Geom g,
                                                 OpCoef c) {
  if (c.skip && *c.skip) return;
  constexpr int W = TX + 2 * R, H = VROWS + 2 * R, N = 2 * R + 1;
  __shared__ cd su[H][W];
  __shared__ double sk[H][W];
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * VROWS;
  const bool fast = c.uniform && i0 >= R && i0 + TX + R <= g.nx && g.row0 + j0 >= R &&
                    g.row0 + j0 + VROWS + R <= g.nyg && j0 + VROWS <= g.ny;  // (whole tile inside the slab)
  const int tid = threadIdx.y * TX + threadIdx.x;
  for (int t = tid; t < H * W; t += TX * VTY) {
    const int ty = t / W, tx = t % W;
    const int gi = i0 + tx - R, gj = g.row0 + j0 + ty - R;
    if (fast) {
      su[ty][tx] = U(u, g, gj, gi);
    } else {
      const bool need = tile_row_needed(g, gj, R);
      su[ty][tx] = need ? upad(u, k, g, c, gj, gi) : mkc(0.0, 0.0);
      sk[ty][tx] = need ? kpad(k, g, c, gj, gi) : 0.0;
    }
  }
  __syncthreads();
  const int ly = 2 * threadIdx.y, lx = threadIdx.x;  // upper output at tile (ly, lx)
  cd a0 = mkc(0.0, 0.0), a1 = mkc(0.0, 0.0);
#pragma unroll
  for (int r = 0; r <= N; ++r) {
    cd uv[N];
#pragma unroll
    for (int bb = 0; bb < N; ++bb) uv[bb] = su[ly + r][lx + bb];
    if (fast) {
      if (r < N) {
#pragma unroll
        for (int bb = 0; bb < N; ++bb) a0 = c_add(a0, c_mul(c.ucoef[r * N + bb], uv[bb]));
      }
      if (r >= 1) {
#pragma unroll
        for (int bb = 0; bb < N; ++bb) a1 = c_add(a1, c_mul(c.ucoef[(r - 1) * N + bb], uv[bb]));
      }
    } else {
      double kv[N];
#pragma unroll
      for (int bb = 0; bb < N; ++bb) kv[bb] = sk[ly + r][lx + bb];
      if (r < N) {
#pragma unroll
        for (int bb = 0; bb < N; ++bb) {
          const cd m = c.mass[r * N + bb];
          const cd coef = mkc(__dadd_rn(c.lap[r * N + bb], __dmul_rn(m.x, kv[bb])), __dmul_rn(m.y, kv[bb]));
          a0 = c_add(a0, c_mul(coef, uv[bb]));
        }
      }
      if (r >= 1) {
#pragma unroll
        for (int bb = 0; bb < N; ++bb) {
          const cd m = c.mass[(r - 1) * N + bb];
          const cd coef =
              mkc(__dadd_rn(c.lap[(r - 1) * N + bb], __dmul_rn(m.x, kv[bb])), __dmul_rn(m.y, kv[bb]));
          a1 = c_add(a1, c_mul(coef, uv[bb]));
        }
      }
    }
  }
  const int i = i0 + lx;
  if (i >= g.nx) return;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int j = j0 + ly + o;
    if (j >= g.ny) return;
    const int gj = j + g.row0;
    const long long p = (long long)j * g.nx + i;
    const cd acc = o == 0 ? a0 : a1;
    if (pinned(g, c, gj, i)) {
      const cd uc = su[ly + o + R][lx + R];
      out[p] = MODE == 0 ? uc : c_sub(b[p], uc);
    } else {
      out[p] = MODE == 0 ? acc : c_sub(b[p], acc);
    }
  }
}

// Horizontally blocked radius-2 form for large grids (radius 3 keeps k_rg: its
// 49-tap body is already FP64/shared-memory co-limited and blocking measured
// slower): each thread owns HX
// adjacent outputs of one row.  For tap row a (a rolled, warp-uniform loop, so
// the per-tap coefficients come from uniform registers) it loads its HX + 2R
// window values once and feeds every (bb, r) tap; per output the taps still
// arrive in the reference's row-major (a, bb) order.  Shared-memory columns are
// skewed by one element every HX so a warp's 16-byte window loads are
// conflict-free (lane stride (HX + 1) * 16 B).
constexpr int HX = 4, HTY = 8, HTX = 32 * HX;
__device__ __forceinline__ int hskew(int col) { return col + col / HX; }
template <int R>
struct HTile {
  static constexpr int W = HTX + 2 * R, P = W + W / HX + 1, H = HTY + 2 * R;
  static constexpr size_t bytes = (size_t)H * P * (sizeof(cd) + sizeof(double));
};

template <int R, int MODE>
__global__ void __launch_bounds__(32 * HTY) k_rgh(const cd* __restrict__ u, const cd* __restrict__ b,
                                                 const double* __restrict__ k, cd* __restrict__ out,
                                                 Geom g, OpCoef c) {
  if (c.skip && *c.skip) return;
  using T = HTile<R>;
  constexpr int N = 2 * R + 1, W = T::W, P = T::P, H = T::H;
  extern __shared__ __align__(16) unsigned char hsm[];
  cd* su = reinterpret_cast<cd*>(hsm);
  double* sk = reinterpret_cast<double*>(su + H * P);
  const int i0 = blockIdx.x * HTX, j0 = blockIdx.y * HTY;
  const bool fast = c.uniform && i0 >= R && i0 + HTX + R <= g.nx && g.row0 + j0 >= R &&
                    g.row0 + j0 + HTY + R <= g.nyg && j0 + HTY <= g.ny;  // (whole tile inside the slab)
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int t = tid; t < H * W; t += 32 * HTY) {
    const int ty = t / W, tx = t % W;
    const int gi = i0 + tx - R, gj = g.row0 + j0 + ty - R;
    const int si = ty * P + hskew(tx);
    if (fast) {
      su[si] = U(u, g, gj, gi);
    } else {
      const bool need = tile_row_needed(g, gj, R);
      su[si] = need ? upad(u, k, g, c, gj, gi) : mkc(0.0, 0.0);
      sk[si] = need ? kpad(k, g, c, gj, gi) : 0.0;
    }
  }
  __syncthreads();
  const int ty = threadIdx.y, cx0 = threadIdx.x * HX;
  cd acc[HX];
#pragma unroll
  for (int r = 0; r < HX; ++r) acc[r] = mkc(0.0, 0.0);
#pragma unroll 1
  for (int a = 0; a < N; ++a) {
    const cd* row = su + (ty + a) * P;
    cd uv[HX + 2 * R];
#pragma unroll
    for (int q = 0; q < HX + 2 * R; ++q) uv[q] = row[hskew(cx0 + q)];
    if (fast) {
#pragma unroll
      for (int bb = 0; bb < N; ++bb) {
        const cd cf = c.ucoef[a * N + bb];
#pragma unroll
        for (int r = 0; r < HX; ++r) acc[r] = c_add(acc[r], c_mul(cf, uv[r + bb]));
      }
    } else {
      const double* krow = sk + (ty + a) * P;
      double kv[HX + 2 * R];
#pragma unroll
      for (int q = 0; q < HX + 2 * R; ++q) kv[q] = krow[hskew(cx0 + q)];
#pragma unroll
      for (int bb = 0; bb < N; ++bb) {
        const double lap = c.lap[a * N + bb];
        const cd m = c.mass[a * N + bb];
#pragma unroll
        for (int r = 0; r < HX; ++r) {
          const double kp = kv[r + bb];
          const cd coef = mkc(__dadd_rn(lap, __dmul_rn(m.x, kp)), __dmul_rn(m.y, kp));
          acc[r] = c_add(acc[r], c_mul(coef, uv[r + bb]));
        }
      }
    }
  }
  const int j = j0 + ty;
  if (j >= g.ny) return;
#pragma unroll
  for (int r = 0; r < HX; ++r) {
    const int i = i0 + cx0 + r;
    if (i >= g.nx) break;
    const long long p = (long long)j * g.nx + i;
    if (pinned(g, c, j + g.row0, i)) {
      const cd uc = su[(ty + R) * P + hskew(cx0 + r + R)];
      out[p] = MODE == 0 ? uc : c_sub(b[p], uc);
    } else {
      out[p] = MODE == 0 ? acc[r] : c_sub(b[p], acc[r]);
    }
  }
}

template <int R, int MODE>
static void launch_rgh(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* out,
                       cudaStream_t st) {
  ensure_smem_attr((const void*)k_rgh<R, MODE>, HTile<R>::bytes);
  const dim3 blk(32, HTY), grd((g.nx + HTX - 1) / HTX, (g.ny + HTY - 1) / HTY);
  k_rgh<R, MODE><<<grd, blk, HTile<R>::bytes, st>>>(u, b, k, out, g, c);
}

// ---------------------------------------------------------------------------
// Separable Galerkin stencil (K2).  Every level kernel factorises exactly
// (SURVEY §0): lap = lsc (a (x) m + m (x) a), mass = msc (m (x) m), so
//   A u = lsc [ sum_r a_r (M u)_r + sum_r m_r (A u)_r ] + msc sum_r m_r (M (k u))_r
// with row-wise 1D passes  (M u)(y, x) = sum_c m_c u(y, x + c)  etc. over the
// SAME ghost-closed u and k^2 samples as the tap form (upad / kpad), then the
// Dirichlet identity rows.  ~100 FP64 operations per output instead of 392-539:
// the kernel becomes memory-bound.  Not bit-identical to the reference's
// row-major 49-tap sum (a different association of the same products):
// within a few ulp of it (tests hold it to 4e-15 of the field's max).
// CTA: 32 x 32 outputs, 256 threads.  Horizontal pass: a thread forms the three
// row sums of 4 adjacent columns from one register window of 4 + 2R samples
// (tile columns skewed by one element every 4 so a quarter-warp's 16-byte window
// loads hit distinct banks); vertical pass: a thread forms 4 vertically adjacent
// outputs of one column from a window of 4 + 2R row sums.
constexpr int GS_T = 32;          // outputs per tile side
__device__ __forceinline__ int gskew(int col) { return col + (col >> 2); }
template <int R>
struct GSTile {
  static constexpr int TR = GS_T + 2 * R, TC = GS_T + 2 * R, PC = TC + TC / 4 + 1;
  static constexpr size_t u_bytes = (size_t)TR * PC * sizeof(cd);
  static constexpr size_t k_bytes = (size_t)TR * PC * sizeof(double);
  static constexpr size_t h_bytes = (size_t)3 * TR * GS_T * sizeof(cd);
  static constexpr size_t bytes = u_bytes + k_bytes + h_bytes;
};

template <int R, int MODE>
__global__ void __launch_bounds__(256, 2) k_rgs(const cd* __restrict__ u, const cd* __restrict__ b,
                                                const double* __restrict__ k, cd* __restrict__ out, Geom g,
                                                OpCoef c) {
  if (c.skip && *c.skip) return;
  using T = GSTile<R>;
  constexpr int N = 2 * R + 1, TR = T::TR, TC = T::TC, PC = T::PC, W = 4 + 2 * R;
  extern __shared__ __align__(16) unsigned char gsm[];
  cd* su = reinterpret_cast<cd*>(gsm);
  double* sk = reinterpret_cast<double*>(gsm + T::u_bytes);
  cd* hm = reinterpret_cast<cd*>(gsm + T::u_bytes + T::k_bytes);  // (M u) rows
  cd* ha = hm + TR * GS_T;                                        // (A u) rows
  cd* hk = ha + TR * GS_T;                                        // (M (k u)) rows
  const int i0 = blockIdx.x * GS_T, j0 = blockIdx.y * GS_T;
  const bool fast = c.uniform && i0 >= R && i0 + GS_T + R <= g.nx && g.row0 + j0 >= R &&
                    g.row0 + j0 + GS_T + R <= g.nyg && j0 + GS_T <= g.ny;  // (whole tile inside the slab)
  const int tid = threadIdx.x;
  constexpr int NL = (TR * TC + 255) / 256;
  if (fast) {  // interior tile: every sample in range, all NL loads in flight before the stores
    cd v[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int t = tid + l * 256;
      const int ty = t / TC, tx = t - ty * TC;
      v[l] = t < TR * TC ? U(u, g, g.row0 + j0 + ty - R, i0 + tx - R) : mkc(0.0, 0.0);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int t = tid + l * 256;
      const int ty = t / TC, tx = t - ty * TC;
      if (t < TR * TC) su[ty * PC + gskew(tx)] = v[l];
    }
  } else {
    for (int t = tid; t < TR * TC; t += 256) {
      const int ty = t / TC, tx = t - ty * TC;
      const int gi = i0 + tx - R, gj = g.row0 + j0 + ty - R;
      const int si = ty * PC + gskew(tx);
      const bool need = tile_row_needed(g, gj, R);
      su[si] = need ? upad(u, k, g, c, gj, gi) : mkc(0.0, 0.0);
      sk[si] = need ? kpad(k, g, c, gj, gi) : 0.0;
    }
  }
  __syncthreads();
  // horizontal pass: item = (tile row r, column group xg of 4)
  for (int it = tid; it < TR * (GS_T / 4); it += 256) {
    const int r = it >> 3, x0 = (it & 7) * 4;
    const cd* row = su + r * PC;
    cd uv[W];
#pragma unroll
    for (int q = 0; q < W; ++q) uv[q] = row[gskew(x0 + q)];
    cd am[4], aa[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) { am[o] = mkc(0.0, 0.0); aa[o] = mkc(0.0, 0.0); }
#pragma unroll
    for (int bb = 0; bb < N; ++bb) {
      const double mb = c.sm[bb], ab = c.sa[bb];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const cd v = uv[o + bb];
        am[o].x = fma(mb, v.x, am[o].x); am[o].y = fma(mb, v.y, am[o].y);
        aa[o].x = fma(ab, v.x, aa[o].x); aa[o].y = fma(ab, v.y, aa[o].y);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      hm[r * GS_T + x0 + o] = am[o];
      ha[r * GS_T + x0 + o] = aa[o];
    }
    if (!fast) {
      const double* krow = sk + r * PC;
      cd ak[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) ak[o] = mkc(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const double kq = krow[gskew(x0 + q)];
        const cd ku = mkc(kq * uv[q].x, kq * uv[q].y);
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int bb = q - o;
          if (bb >= 0 && bb < N) {
            ak[o].x = fma(c.sm[bb], ku.x, ak[o].x);
            ak[o].y = fma(c.sm[bb], ku.y, ak[o].y);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) hk[r * GS_T + x0 + o] = ak[o];
    }
  }
  __syncthreads();
  // vertical pass: thread = (column x, row group y0 of 4)
  const int x = tid & 31, y0 = (tid >> 5) * 4;
  cd lm[4], lk[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) { lm[o] = mkc(0.0, 0.0); lk[o] = mkc(0.0, 0.0); }
  {
    cd w[W];
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = hm[(y0 + q) * GS_T + x];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const double aa = c.sa[a], ma = c.sm[a];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        lm[o].x = fma(aa, w[o + a].x, lm[o].x); lm[o].y = fma(aa, w[o + a].y, lm[o].y);
        lk[o].x = fma(ma, w[o + a].x, lk[o].x); lk[o].y = fma(ma, w[o + a].y, lk[o].y);
      }
    }
#pragma unroll
    for (int q = 0; q < W; ++q) w[q] = ha[(y0 + q) * GS_T + x];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const double ma = c.sm[a];
#pragma unroll
      for (int o = 0; o < 4; ++o) { lm[o].x = fma(ma, w[o + a].x, lm[o].x); lm[o].y = fma(ma, w[o + a].y, lm[o].y); }
    }
    if (!fast) {  // lk = sum_a m_a (M (k u))_a; the uniform form scales sum_a m_a (M u)_a by k
#pragma unroll
      for (int q = 0; q < W; ++q) w[q] = hk[(y0 + q) * GS_T + x];
#pragma unroll
      for (int o = 0; o < 4; ++o) lk[o] = mkc(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double ma = c.sm[a];
#pragma unroll
        for (int o = 0; o < 4; ++o) { lk[o].x = fma(ma, w[o + a].x, lk[o].x); lk[o].y = fma(ma, w[o + a].y, lk[o].y); }
      }
    } else {
#pragma unroll
      for (int o = 0; o < 4; ++o) lk[o] = mkc(c.ku * lk[o].x, c.ku * lk[o].y);
    }
  }
  const int i = i0 + x;
  if (i >= g.nx) return;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int j = j0 + y0 + o;
    if (j >= g.ny) return;
    const int gj = j + g.row0;
    const long long p = (long long)j * g.nx + i;
    cd v;
    if (pinned(g, c, gj, i)) {
      v = su[(y0 + o + R) * PC + gskew(x + R)];
    } else {
      // lsc * lap sums + msc * mass sum (complex msc)
      v.x = fma(c.lsc, lm[o].x, fma(c.msc.x, lk[o].x, -c.msc.y * lk[o].y));
      v.y = fma(c.lsc, lm[o].y, fma(c.msc.x, lk[o].y, c.msc.y * lk[o].x));
    }
    out[p] = MODE == 0 ? v : c_sub(b[p], v);
  }
}

template <int R, int MODE>
static void launch_rgs(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* out,
                       cudaStream_t st) {
  ensure_smem_attr((const void*)k_rgs<R, MODE>, GSTile<R>::bytes);
  const dim3 grd((g.nx + GS_T - 1) / GS_T, (g.ny + GS_T - 1) / GS_T);
  k_rgs<R, MODE><<<grd, 256, GSTile<R>::bytes, st>>>(u, b, k, out, g, c);
}

static int g_rg_exact = -1;  // -1: from HDB_RG_EXACT (default 0 = separable form where available)
void set_rg_exact(int on) { g_rg_exact = on ? 1 : 0; }
static bool rg_exact() {
  if (g_rg_exact < 0) {
    const char* e = getenv("HDB_RG_EXACT");
    g_rg_exact = e ? (atoi(e) != 0) : 0;
  }
  return g_rg_exact != 0;
}
bool rg_exact_on() { return rg_exact(); }

// ------------------------------------------------------------------------
// Fused multigrid residual + restriction (mg.py:116-117):
//     coarse = Z^T (b - M x)        with the coarse Dirichlet rows zeroed
// in ONE pass over x, b, k^2 (40 B per fine point) plus the coarse write (4 B
// per fine point) -- the residual is never stored (the unfused pair moves 56 +
// 20 B per fine point).  A warp owns 30 coarse columns and FRB coarse rows:
// lane L holds the fine columns E = 2 (c0 + L), O = E + 1 and walks the strip's
// 2 FRB + 3 fine rows top to bottom with rows y-1, y, y+1 of x in registers
// (k_r1w's sliding window, two columns per lane; the x-neighbours come from
// lane shuffles); the residuals of one fine row then feed the (1,4,6,4,1)/16
// taps of the coarse points through shuffles (lanes 0 / 31 only supply the
// neighbours' residuals).  Residuals use k_r1's arithmetic and every coarse sum
// the reference's (b, a) term order, so the result is bit-identical to
// launch_apply(mode 1) followed by launch_restrict.  Fine points on the boundary
// ring or outside the grid (the reference's zero extension) take the per-point
// closure path (rr_point) -- a few lanes / rows per boundary strip.  Unsharded
// radius-1 levels only.
constexpr int FWY = 4;              // warps per block
constexpr int FCX = 30;             // coarse columns per warp
__host__ __device__ constexpr double fw16(int i) { return (i == 0 || i == 4 ? 1.0 : (i == 2 ? 6.0 : 4.0)) / 16; }

// b - M x at fine (y, x) by the closure path; zero outside the grid.  Out of line (it
// serves the few boundary-ring points of a strip) and fed by value: a reference to
// the kernel's OpCoef parameter would force a per-thread stack copy of the whole
// coefficient block.  Same operations as r1_point<1> (upad / pinned / five_point).
struct R1C {
  int nx, ny, bc[4];
  double two_h, s;
  cd mc;
};
__device__ __noinline__ cd rr_point(const cd* __restrict__ u, const cd* __restrict__ b,
                                    const double* __restrict__ k, R1C q, int y, int x) {
  if (y < 0 || y >= q.ny || x < 0 || x >= q.nx) return mkc(0.0, 0.0);
  const long long nx = q.nx, p = (long long)y * nx + x;
  const cd uc = u[p];
  if ((q.bc[0] == HDB_BC_DIRICHLET && x == 0) || (q.bc[1] == HDB_BC_DIRICHLET && x == q.nx - 1) ||
      (q.bc[2] == HDB_BC_DIRICHLET && y == 0) || (q.bc[3] == HDB_BC_DIRICHLET && y == q.ny - 1))
    return c_sub(b[p], uc);
  const double kc = k[p];
  // neighbours: in the grid, or the first ghost layer closed from (boundary point = centre, inner point)
  const cd w = x > 0 ? u[p - 1] : ghost_val(q.bc[0], q.two_h, kc, uc, u[p + 1]);
  const cd e = x < q.nx - 1 ? u[p + 1] : ghost_val(q.bc[1], q.two_h, kc, uc, u[p - 1]);
  const cd so = y > 0 ? u[p - nx] : ghost_val(q.bc[2], q.two_h, kc, uc, u[p + nx]);
  const cd no = y < q.ny - 1 ? u[p + nx] : ghost_val(q.bc[3], q.two_h, kc, uc, u[p - nx]);
  return c_sub(b[p], five_point(q.s, q.mc, kc, uc, w, e, so, no));
}

// Every strip runs the sliding window with row and column indices clamped into the
// grid (so all loads are legal); a fine point that is not strictly interior -- the
// boundary ring (closure, pinned rows) or a position outside the grid (zero
// extension) -- has its window value replaced by rr_point.  Only the lanes / rows
// that own such points diverge.
template <int FRB>
__global__ void __launch_bounds__(32 * FWY, 4) k_resrestrict(const cd* __restrict__ u, const cd* __restrict__ b,
                                                          const double* __restrict__ k, cd* __restrict__ coarse,
                                                          Geom g, OpCoef c, int ncx, int ncy, int zero_mask) {
  constexpr int FNR = 2 * FRB + 3;  // fine rows per strip
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  const int c0 = blockIdx.x * FCX - 1;  // coarse column of lane 0 (a neighbour-only lane)
  const int cx = c0 + lane;
  const int cy0 = (blockIdx.y * FWY + wy) * FRB;
  if (cy0 >= ncy) return;
  const int nrows = min(FRB, ncy - cy0);
  const int xE = 2 * cx, y0 = 2 * cy0 - 2;
  const int nx = g.nx, ny = g.nyg;
  R1C rc;
  rc.nx = nx; rc.ny = ny; rc.two_h = 2.0 * c.h; rc.s = c.s; rc.mc = c.mc;
#pragma unroll
  for (int q = 0; q < 4; ++q) rc.bc[q] = c.bc[q];
  const bool inE = xE >= 1 && xE <= nx - 2, inO = xE + 1 >= 1 && xE + 1 <= nx - 2;  // strictly interior columns
  auto cl = [](int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); };
  const int qE = cl(xE, nx - 1), qO = cl(xE + 1, nx - 1), qW = cl(xE - 1, nx - 1), qX = cl(xE + 2, nx - 1);
  auto row = [&](int y) { return (long long)cl(y, ny - 1) * nx; };
  double ar[FRB], ai[FRB];
#pragma unroll
  for (int q = 0; q < FRB; ++q) ar[q] = ai[q] = 0.0;
  cd sE = u[row(y0 - 1) + qE], sO = u[row(y0 - 1) + qO];
  cd cE = u[row(y0) + qE], cO = u[row(y0) + qO];
  cd nE = u[row(y0 + 1) + qE], nO = u[row(y0 + 1) + qO];
  cd bE = b[row(y0) + qE], bO = b[row(y0) + qO];
  double kE = k[row(y0) + qE], kO = k[row(y0) + qO];
  cd wl = mkc(0.0, 0.0), el = wl;
  if (lane == 0) wl = u[row(y0) + qW];
  if (lane == 31) el = u[row(y0) + qX];
#pragma unroll
  for (int r = 0; r < FNR; ++r) {
    const int y = y0 + r;
    cd n2E = mkc(0.0, 0.0), n2O = n2E, b2E = n2E, b2O = n2E, wl2 = n2E, el2 = n2E;
    double k2E = 0.0, k2O = 0.0;
    if (r + 1 < FNR) {  // next row's loads before this row's arithmetic
      const long long o2 = row(y + 2), o1 = row(y + 1);
      n2E = u[o2 + qE]; n2O = u[o2 + qO];
      b2E = b[o1 + qE]; b2O = b[o1 + qO];
      k2E = k[o1 + qE]; k2O = k[o1 + qO];
      if (lane == 0) wl2 = u[o1 + qW];
      if (lane == 31) el2 = u[o1 + qX];
    }
    cd wE, eO;
    wE.x = __shfl_up_sync(0xffffffffu, cO.x, 1);
    wE.y = __shfl_up_sync(0xffffffffu, cO.y, 1);
    eO.x = __shfl_down_sync(0xffffffffu, cE.x, 1);
    eO.y = __shfl_down_sync(0xffffffffu, cE.y, 1);
    if (lane == 0) wE = wl;
    if (lane == 31) eO = el;
    cd rE = c_sub(bE, five_point(c.s, c.mc, kE, cE, wE, cO, sE, nE));
    cd rO = c_sub(bO, five_point(c.s, c.mc, kO, cO, cE, eO, sO, nO));
    const bool rin = y >= 1 && y <= ny - 2;  // strictly interior row (warp-uniform)
    if (!(rin && inE)) rE = rr_point(u, b, k, rc, y, xE);
    if (!(rin && inO)) rO = rr_point(u, b, k, rc, y, xE + 1);
    sE = cE; sO = cO; cE = nE; cO = nO; nE = n2E; nO = n2O;
    bE = b2E; bO = b2O; kE = k2E; kO = k2O; wl = wl2; el = el2;
    // the five fine residuals under coarse column cx: columns 2cx-2 .. 2cx+2
    cd v[5];
    v[2] = rE;
    v[3] = rO;
    v[0].x = __shfl_up_sync(0xffffffffu, rE.x, 1);
    v[0].y = __shfl_up_sync(0xffffffffu, rE.y, 1);
    v[1].x = __shfl_up_sync(0xffffffffu, rO.x, 1);
    v[1].y = __shfl_up_sync(0xffffffffu, rO.y, 1);
    v[4].x = __shfl_down_sync(0xffffffffu, rE.x, 1);
    v[4].y = __shfl_down_sync(0xffffffffu, rE.y, 1);
    // fine row r is tap b = r - 2q of coarse row q (compile-time after unrolling)
#pragma unroll
    for (int q = 0; q < FRB; ++q) {
      const int bt = r - 2 * q;
      if (bt < 0 || bt > 4) continue;
#pragma unroll
      for (int a = 0; a < 5; ++a) {
        const double w = fw16(bt) * fw16(a);  // exact (dyadic)
        ar[q] = __dadd_rn(ar[q], __dmul_rn(w, v[a].x));
        ai[q] = __dadd_rn(ai[q], __dmul_rn(w, v[a].y));
      }
    }
    if (r >= 4 && ((r - 4) & 1) == 0) {  // coarse row q complete after its b = 4 row
      const int q = (r - 4) / 2;
      if (q < nrows && lane >= 1 && lane <= FCX && cx < ncx) {
        const int cy = cy0 + q;
        const bool z = ((zero_mask & 1) && cx == 0) || ((zero_mask & 2) && cx == ncx - 1) ||
                       ((zero_mask & 4) && cy == 0) || ((zero_mask & 8) && cy == ncy - 1);
        coarse[(long long)cy * ncx + cx] = z ? mkc(0.0, 0.0) : mkc(ar[q], ai[q]);
      }
    }
  }
}

bool resrestrict_fits(const OpCoef& c, const Geom& g) {
  static const bool on = [] {
    const char* e = getenv("HDB_FUSE_RR");
    return !e || atoi(e) != 0;
  }();
  // small grids: most strips are boundary strips (per-point path); keep the unfused pair there
  static const int minn = [] {  // HDB_RR_MIN: smallest fine extent that takes the fused kernel
    const char* e = getenv("HDB_RR_MIN");
    return e ? atoi(e) : 513;
  }();
  return on && c.radius == 1 && g.row0 == 0 && g.ny == g.nyg && g.nx >= minn && g.ny >= minn && (g.nx & 1) && (g.ny & 1);
}

void launch_resrestrict(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* coarse,
                        int zero_mask, cudaStream_t st) {
  const int ncx = (g.nx - 1) / 2 + 1, ncy = (g.nyg - 1) / 2 + 1;
  static const int forced = [] {  // HDB_RR_FRB=4|8: coarse rows per warp
    const char* e = getenv("HDB_RR_FRB");
    return e ? atoi(e) : 0;
  }();
  const int frb = forced ? forced : 4;  // measured: 4 rows per warp is as fast or faster at every size (profiles/r02z_fusion_microbench.log)
  if (frb == 8) {
    const dim3 grd((ncx + FCX - 1) / FCX, (ncy + FWY * 8 - 1) / (FWY * 8));
    k_resrestrict<8><<<grd, 32 * FWY, 0, st>>>(u, b, k, coarse, g, c, ncx, ncy, zero_mask);
  } else {
    const dim3 grd((ncx + FCX - 1) / FCX, (ncy + FWY * 4 - 1) / (FWY * 4));
    k_resrestrict<4><<<grd, 32 * FWY, 0, st>>>(u, b, k, coarse, g, c, ncx, ncy, zero_mask);
  }
}

// ------------------------------------------------------------------------
static inline dim3 grid_r1(const Geom& g) { return dim3((g.nx + 31) / 32, (g.ny + 7) / 8); }
static inline dim3 grid_r1s(const Geom& g) { return dim3((g.nx + SX - 1) / SX, (g.ny + SY * RB - 1) / (SY * RB)); }
static inline bool use_strip(const Geom& g) { return g.nx >= 512 && g.ny >= 512; }  // small grids: all blocks are boundary blocks

// HDB_R1_WAVE=0 selects the fixed 16-row k_r1s; HDB_R1_RB=n forces rb
static int r1_rows(int mode, const Geom& g) {
  static const int forced = [] {
    const char* e = getenv("HDB_R1_RB");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  if (forced) return forced;
  if (mode == 0 || mode == 1) return 4;
  return (long long)g.nx * g.ny >= (32LL << 20) ? 16 : 8;
}
static bool r1_wave() {
  static const bool v = [] {
    const char* e = getenv("HDB_R1_WAVE");
    return !e || atoi(e) != 0;
  }();
  return v;
}
template <int MODE>
static void launch_r1_strip(const Geom& g, const cd* u, const cd* b, const double* k, cd* out, const OpCoef& c,
                            double omega, cudaStream_t st) {
  const dim3 blk(SX, SY);
  if (!r1_wave()) {
    k_r1s<MODE><<<grid_r1s(g), blk, 0, st>>>(u, b, k, out, g, c, omega);
    return;
  }
  const int rb = r1_rows(MODE, g);
  const dim3 grd((g.nx + SX - 1) / SX, (g.ny + SY * rb - 1) / (SY * rb));
  k_r1w<MODE, (MODE == 2 ? 2 : 4)><<<grd, blk, 0, st>>>(u, b, k, out, g, c, omega, rb);
}

void launch_apply(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* out,
                  int mode, cudaStream_t st) {
  if (c.radius == 1) {
    if (use_strip(g)) {
      if (mode == 0) launch_r1_strip<0>(g, u, b, k, out, c, 0.0, st);
      else launch_r1_strip<1>(g, u, b, k, out, c, 0.0, st);
      return;
    }
    const dim3 blk(32, 8), grd = grid_r1(g);
    if (mode == 0) k_r1<0><<<grd, blk, 0, st>>>(u, b, k, out, g, c, 0.0);
    else k_r1<1><<<grd, blk, 0, st>>>(u, b, k, out, g, c, 0.0);
    return;
  }
  if (c.sep && !rg_exact()) {
    if (c.radius == 2) {
      if (mode == 0) launch_rgs<2, 0>(c, g, u, b, k, out, st);
      else launch_rgs<2, 1>(c, g, u, b, k, out, st);
    } else {
      if (mode == 0) launch_rgs<3, 0>(c, g, u, b, k, out, st);
      else launch_rgs<3, 1>(c, g, u, b, k, out, st);
    }
    return;
  }
  static const bool blocked = [] {
    const char* e = getenv("HDB_RG_BLOCKED");
    return !e || atoi(e) != 0;
  }();
  if (blocked && c.radius == 2 && g.nx >= 256 && g.ny >= 64) {
    if (mode == 0) launch_rgh<2, 0>(c, g, u, b, k, out, st);
    else launch_rgh<2, 1>(c, g, u, b, k, out, st);
    return;
  }
  static const bool vblock = [] {
    const char* e = getenv("HDB_RG_VBLOCK");
    return !e || atoi(e) != 0;
  }();
  if (vblock && c.radius == 3 && g.nx >= 64 && g.ny >= 64) {
    const dim3 blk(TX, VTY), grd((g.nx + TX - 1) / TX, (g.ny + VROWS - 1) / VROWS);
    if (mode == 0) k_rgv<3, 0><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
    else k_rgv<3, 1><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
    return;
  }
  const dim3 blk(TX, TY), grd((g.nx + TX - 1) / TX, (g.ny + TY - 1) / TY);
  if (c.radius == 2) {
    if (mode == 0) k_rg<2, 0><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
    else k_rg<2, 1><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
  } else {
    if (mode == 0) k_rg<3, 0><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
    else k_rg<3, 1><<<grd, blk, 0, st>>>(u, b, k, out, g, c);
  }
}

void launch_jacobi(const OpCoef& c, const Geom& g, const cd* x, const cd* b, const double* k, cd* out,
                   double omega, bool from_zero, cudaStream_t st) {
  if (use_strip(g)) {
    if (from_zero) launch_r1_strip<3>(g, x, b, k, out, c, omega, st);
    else launch_r1_strip<2>(g, x, b, k, out, c, omega, st);
    return;
  }
  const dim3 blk(32, 8), grd = grid_r1(g);
  if (from_zero) k_r1<3><<<grd, blk, 0, st>>>(x, b, k, out, g, c, omega);
  else k_r1<2><<<grd, blk, 0, st>>>(x, b, k, out, g, c, omega);
}

// the last post-smoothing sweep with the A-DEF1 sum folded in: out = Jacobi(x), out2 = out + addt
bool jacobi_add_fits(const Geom& g) {
  static const bool on = [] {
    const char* e = getenv("HDB_FUSE_RT");
    return !e || atoi(e) != 0;
  }();
  return on && use_strip(g) && r1_wave();
}
void launch_jacobi_add(const OpCoef& c, const Geom& g, const cd* x, const cd* b, const double* k, cd* out,
                       double omega, const cd* addt, cd* out2, cudaStream_t st) {
  const int rb = r1_rows(2, g);
  const dim3 blk(SX, SY), grd((g.nx + SX - 1) / SX, (g.ny + SY * rb - 1) / (SY * rb));
  k_r1w<4, 2><<<grd, blk, 0, st>>>(x, b, k, out, g, c, omega, rb, addt, out2);
}

long long resnorm_partials(const Geom& g) {
  return (long long)((g.nx + 31) / 32) * ((g.ny + NRW * RBN - 1) / (NRW * RBN));
}
void launch_resnorm(const OpCoef& c, const Geom& g, const cd* u, const cd* b, const double* k, cd* partials,
                    cd* dst, cudaStream_t st) {
  const dim3 grd((g.nx + 31) / 32, (g.ny + NRW * RBN - 1) / (NRW * RBN));
  k_resnorm<<<grd, 32 * NRW, 0, st>>>(u, b, k, g, c, partials);
  k_sum_partials<<<1, kSumThreads, 0, st>>>(partials, (long long)grd.x * grd.y, dst);
}

}  // namespace hdb
