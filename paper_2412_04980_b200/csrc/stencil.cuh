// Ghost-closure sampling shared by all level-operator kernels.
//
// Restates operators.py:44-93 (ghost_pad / ksq_ghost_pad) as on-the-fly
// sampling: first ghost layer synthesised (Dirichlet 2u_b - u_in,
// Sommerfeld u_in + (2ih k_b) u_b), deeper layers and ghost corners zero;
// ghost k^2 = 2k_b - k_in on Dirichlet sides, else zero.  k_b = sqrt(k^2_b)
// (IEEE-correctly-rounded sqrt = numpy's np.sqrt, operators.py:114-115).
#pragma once
#include "hdb_common.cuh"

namespace hdb {

__device__ __forceinline__ const cd& U(const cd* u, const Geom& g, int gj, int i) {
  return u[(long long)(gj - g.row0) * g.nx + i];
}
__device__ __forceinline__ double K(const double* k, const Geom& g, int gj, int i) {
  return k[(long long)(gj - g.row0) * g.nx + i];
}

// Sommerfeld ghost  u_in + (0, B) * u_b  with B = (2h) * k_b  (exactly the numpy
// evaluation two_ih * k_edge * u_b followed by the add)
__device__ __forceinline__ cd ghost_val(int bc, double two_h, double kb2, cd ub, cd uin) {
  if (bc == HDB_BC_DIRICHLET) {
    return mkc(__dsub_rn(__dmul_rn(2.0, ub.x), uin.x), __dsub_rn(__dmul_rn(2.0, ub.y), uin.y));
  }
  const double B = __dmul_rn(two_h, sqrt(kb2));
  return mkc(__dsub_rn(uin.x, __dmul_rn(B, ub.y)), __dadd_rn(uin.y, __dmul_rn(B, ub.x)));
}

// padded u at global (gj, i); (gj, i) may lie outside the grid by up to r
__device__ __forceinline__ cd upad(const cd* u, const double* k, const Geom& g, const OpCoef& c,
                                   int gj, int i) {
  const bool xin = (i >= 0) & (i < g.nx);
  const bool yin = (gj >= 0) & (gj < g.nyg);
  if (xin & yin) return U(u, g, gj, i);
  const double two_h = 2.0 * c.h;
  if (yin) {
    if (i == -1) return ghost_val(c.bc[0], two_h, K(k, g, gj, 0), U(u, g, gj, 0), U(u, g, gj, 1));
    if (i == g.nx)
      return ghost_val(c.bc[1], two_h, K(k, g, gj, g.nx - 1), U(u, g, gj, g.nx - 1), U(u, g, gj, g.nx - 2));
  } else if (xin) {
    if (gj == -1) return ghost_val(c.bc[2], two_h, K(k, g, 0, i), U(u, g, 0, i), U(u, g, 1, i));
    if (gj == g.nyg)
      return ghost_val(c.bc[3], two_h, K(k, g, g.nyg - 1, i), U(u, g, g.nyg - 1, i), U(u, g, g.nyg - 2, i));
  }
  return mkc(0.0, 0.0);
}

// Tile loaders of the radius-2/3 kernels: a block whose outputs run past the slab's last row
// would sample rows beyond the slab's halo (local row >= ny + R).  No valid output needs
// them and on a row slab they are not addressable (only H >= R halo rows exist around a
// vector; on the whole grid they are ghost rows anyway): such samples are not loaded.
__device__ __forceinline__ bool tile_row_needed(const Geom& g, int gj, int R) { return gj - g.row0 < g.ny + R; }

// padded k^2 (operators.py:78-93)
__device__ __forceinline__ double kpad(const double* k, const Geom& g, const OpCoef& c, int gj, int i) {
  const bool xin = (i >= 0) & (i < g.nx);
  const bool yin = (gj >= 0) & (gj < g.nyg);
  if (xin & yin) return K(k, g, gj, i);
  if (yin) {
    if (i == -1 && c.bc[0] == HDB_BC_DIRICHLET)
      return __dsub_rn(__dmul_rn(2.0, K(k, g, gj, 0)), K(k, g, gj, 1));
    if (i == g.nx && c.bc[1] == HDB_BC_DIRICHLET)
      return __dsub_rn(__dmul_rn(2.0, K(k, g, gj, g.nx - 1)), K(k, g, gj, g.nx - 2));
  } else if (xin) {
    if (gj == -1 && c.bc[2] == HDB_BC_DIRICHLET)
      return __dsub_rn(__dmul_rn(2.0, K(k, g, 0, i)), K(k, g, 1, i));
    if (gj == g.nyg && c.bc[3] == HDB_BC_DIRICHLET)
      return __dsub_rn(__dmul_rn(2.0, K(k, g, g.nyg - 1, i)), K(k, g, g.nyg - 2, i));
  }
  return 0.0;
}

// Dirichlet identity row?  (operators.py:163-166, dirichlet_slices 149-161)
__device__ __forceinline__ bool pinned(const Geom& g, const OpCoef& c, int gj, int i) {
  return (c.bc[0] == HDB_BC_DIRICHLET && i == 0) || (c.bc[1] == HDB_BC_DIRICHLET && i == g.nx - 1) ||
         (c.bc[2] == HDB_BC_DIRICHLET && gj == 0) || (c.bc[3] == HDB_BC_DIRICHLET && gj == g.nyg - 1);
}

// radius-1 contraction (_kernels.py:24-31):
//   s*((((4c - W) - E) - S) - N) + (mc*k)*c
__device__ __forceinline__ cd five_point(double s, cd mc, double kc, cd c, cd w, cd e, cd so, cd no) {
  double lr = __dmul_rn(4.0, c.x), li = __dmul_rn(4.0, c.y);
  lr = __dsub_rn(lr, w.x);  li = __dsub_rn(li, w.y);
  lr = __dsub_rn(lr, e.x);  li = __dsub_rn(li, e.y);
  lr = __dsub_rn(lr, so.x); li = __dsub_rn(li, so.y);
  lr = __dsub_rn(lr, no.x); li = __dsub_rn(li, no.y);
  const cd mk = mkc(__dmul_rn(mc.x, kc), __dmul_rn(mc.y, kc));
  const cd m = c_mul(mk, c);
  return mkc(__dadd_rn(__dmul_rn(s, lr), m.x), __dadd_rn(__dmul_rn(s, li), m.y));
}

// reciprocal of the radius-1 diagonal (operators.py:180-208), numpy Smith
// division 1.0/d (CDOUBLE_divide)
__device__ __forceinline__ cd dinv_at(const double* k, const Geom& g, const OpCoef& c, int gj, int i) {
  if (pinned(g, c, gj, i)) return mkc(1.0, 0.0);
  const double kc = K(k, g, gj, i);
  double dr = __dadd_rn(4.0 * c.s, __dmul_rn(c.mc.x, kc));
  double di = __dmul_rn(c.mc.y, kc);
  if (c.bc[0] == HDB_BC_SOMMERFELD && i == 0) di = __dadd_rn(di, __dmul_rn(c.E, sqrt(K(k, g, gj, 0))));
  if (c.bc[1] == HDB_BC_SOMMERFELD && i == g.nx - 1) di = __dadd_rn(di, __dmul_rn(c.E, sqrt(K(k, g, gj, g.nx - 1))));
  if (c.bc[2] == HDB_BC_SOMMERFELD && gj == 0) di = __dadd_rn(di, __dmul_rn(c.E, sqrt(K(k, g, 0, i))));
  if (c.bc[3] == HDB_BC_SOMMERFELD && gj == g.nyg - 1) di = __dadd_rn(di, __dmul_rn(c.E, sqrt(K(k, g, g.nyg - 1, i))));
  if (fabs(dr) >= fabs(di)) {
    const double rat = __ddiv_rn(di, dr);
    const double scl = __ddiv_rn(1.0, __dadd_rn(dr, __dmul_rn(di, rat)));
    return mkc(scl, __dmul_rn(-rat, scl));
  }
  const double rat = __ddiv_rn(dr, di);
  const double scl = __ddiv_rn(1.0, __dadd_rn(di, __dmul_rn(dr, rat)));
  return mkc(__dmul_rn(rat, scl), -scl);
}

}  // namespace hdb
