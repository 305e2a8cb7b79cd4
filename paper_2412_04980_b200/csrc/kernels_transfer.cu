// Higher-order transfers Z^T (restriction, (1,4,6,4,1)/16 per dim) and Z
// (prolongation, (1,4,6,4,1)/8 per dim, scatter form), zero extension.
//
// Reference: transfers.py:59-88.  The reference accumulates 25 strided numpy
// passes in (b, a) row-major order starting from zeros; each pass adds
// round(w_b w_a * v) (w products are exact dyadic rationals).  The gather
// kernels below add the same terms in the same order, so results are
// bit-identical.  Algorithmic traffic: 20 B per fine point each way
// (fine 16 B read/write + coarse 16 B / 4).
//
// Slab form (TGeom): fine rows [f_row0, f_row0 + f_ny) of a grid with nfy_g
// rows are local; rows just outside are halo rows (filled by the exchange) or,
// at the physical edges, zero extension.  Coarse rows likewise.
#include <cstdlib>

#include "kernels.h"
#include "hdb_common.cuh"

namespace hdb {

__constant__ double cW16[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
__constant__ double cW8[5] = {1.0 / 8, 4.0 / 8, 6.0 / 8, 4.0 / 8, 1.0 / 8};

__device__ __forceinline__ cd ldf(const cd* f, const TGeom& t, int yg, int x) {
  return (yg >= 0 && yg < t.nfy_g && x >= 0 && x < t.nfx) ? f[(long long)(yg - t.f_row0) * t.nfx + x]
                                                           : mkc(0.0, 0.0);
}
__device__ __forceinline__ cd ldc(const cd* c, const TGeom& t, int yg, int x) {
  return (yg >= 0 && yg < t.ncy_g && x >= 0 && x < t.ncx) ? c[(long long)(yg - t.c_row0) * t.ncx + x]
                                                          : mkc(0.0, 0.0);
}
__device__ __forceinline__ bool zrow(int zero_mask, int cx, int cyg, const TGeom& t) {
  return ((zero_mask & 1) && cx == 0) || ((zero_mask & 2) && cx == t.ncx - 1) || ((zero_mask & 4) && cyg == 0) ||
         ((zero_mask & 8) && cyg == t.ncy_g - 1);
}

// coarse point (cy, cx) = sum_{b,a} (w16_b w16_a) fine(2cy+b-2, 2cx+a-2); thread per coarse point
__global__ void __launch_bounds__(256) k_restrict(const cd* __restrict__ f, cd* __restrict__ c, TGeom t,
                                                  int zero_mask) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= t.ncx || cy >= t.c_ny) return;
  const int cyg = cy + t.c_row0;
  const long long p = (long long)cy * t.ncx + cx;
  if (zrow(zero_mask, cx, cyg, t)) { c[p] = mkc(0.0, 0.0); return; }
  double ar = 0.0, ai = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int y = 2 * cyg + b - 2;
    if (y < 0 || y >= t.nfy_g) continue;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      if (x < 0 || x >= t.nfx) continue;
      const double w = cW16[b] * cW16[a];
      const cd v = f[(long long)(y - t.f_row0) * t.nfx + x];
      ar = __dadd_rn(ar, __dmul_rn(w, v.x));
      ai = __dadd_rn(ai, __dmul_rn(w, v.y));
    }
  }
  c[p] = mkc(ar, ai);
}

// fine-level form: two coarse rows per thread (cy, cy+1) share fine rows
// 2cy-2..2cy+4, each loaded once and fed to two independent ordered chains
__global__ void __launch_bounds__(256) k_restrict2(const cd* __restrict__ f, cd* __restrict__ c, TGeom t,
                                                   int zero_mask) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = 2 * (blockIdx.y * blockDim.y + threadIdx.y);
  if (cx >= t.ncx || cy >= t.c_ny) return;
  const int cyg = cy + t.c_row0;
  double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
#pragma unroll
  for (int r = 0; r < 7; ++r) {
    const int y = 2 * cyg - 2 + r;
    if (y < 0 || y >= t.nfy_g) continue;
    cd v[5];
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      v[a] = (x >= 0 && x < t.nfx) ? f[(long long)(y - t.f_row0) * t.nfx + x] : mkc(0.0, 0.0);
    }
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      if (x < 0 || x >= t.nfx) continue;
      if (r <= 4) {
        const double w = cW16[r] * cW16[a];
        ar = __dadd_rn(ar, __dmul_rn(w, v[a].x));
        ai = __dadd_rn(ai, __dmul_rn(w, v[a].y));
      }
      if (r >= 2) {
        const double w = cW16[r - 2] * cW16[a];
        br = __dadd_rn(br, __dmul_rn(w, v[a].x));
        bi = __dadd_rn(bi, __dmul_rn(w, v[a].y));
      }
    }
  }
  c[(long long)cy * t.ncx + cx] = zrow(zero_mask, cx, cyg, t) ? mkc(0.0, 0.0) : mkc(ar, ai);
  if (cy + 1 < t.c_ny)
    c[(long long)(cy + 1) * t.ncx + cx] = zrow(zero_mask, cx, cyg + 1, t) ? mkc(0.0, 0.0) : mkc(br, bi);
}

// Strip form for large grids: one thread per coarse column, RRB coarse rows
// per thread.  Fine rows are streamed top to bottom; each is read once per warp
// as a coalesced even/odd pair (fine 2cx, 2cx+1) and the (2cx-2, 2cx-1, 2cx+2)
// neighbours come from warp shuffles.  A fine row y contributes to the coarse
// rows with b = y - 2cy + 2 in [0, 4] in increasing-b order, so every coarse
// sum is accumulated in the reference's (b, a) order (bit-identical).
constexpr int RSX = 32, RSY = 4, RRB = 8;
__host__ __device__ constexpr double kw5(int i) { return i == 0 || i == 4 ? 1.0 : (i == 2 ? 6.0 : 4.0); }
__host__ __device__ constexpr double kW16(int i) { return kw5(i) / 16; }

__global__ void __launch_bounds__(RSX * RSY) k_restrict_s(const cd* __restrict__ f, cd* __restrict__ c, TGeom t,
                                                          int zero_mask) {
  const int lane = threadIdx.x;
  const int cx = blockIdx.x * RSX + lane;
  const int cy0 = (blockIdx.y * RSY + threadIdx.y) * RRB;  // local coarse row (warp-uniform)
  if (cy0 >= t.c_ny) return;
  const int ncy = min(RRB, t.c_ny - cy0);
  const int cyg0 = cy0 + t.c_row0;
  const int x0 = 2 * cx;
  bool va[5];
#pragma unroll
  for (int a = 0; a < 5; ++a) va[a] = (x0 + a - 2 >= 0) && (x0 + a - 2 < t.nfx);
  double ar[RRB], ai[RRB];
#pragma unroll
  for (int k = 0; k < RRB; ++k) ar[k] = ai[k] = 0.0;
#pragma unroll
  for (int r = 0; r < 2 * RRB + 3; ++r) {
    const int y = 2 * cyg0 - 2 + r;
    if (r <= 2 * (ncy - 1) + 4 && y >= 0 && y < t.nfy_g) {  // warp-uniform
      const cd* row = f + (long long)(y - t.f_row0) * t.nfx;
      const cd E = (x0 < t.nfx) ? row[x0] : mkc(0.0, 0.0);
      const cd O = (x0 + 1 < t.nfx) ? row[x0 + 1] : mkc(0.0, 0.0);
      cd v[5];
      v[2] = E;
      v[3] = O;
      v[0].x = __shfl_up_sync(0xffffffffu, E.x, 1);
      v[0].y = __shfl_up_sync(0xffffffffu, E.y, 1);
      v[1].x = __shfl_up_sync(0xffffffffu, O.x, 1);
      v[1].y = __shfl_up_sync(0xffffffffu, O.y, 1);
      v[4].x = __shfl_down_sync(0xffffffffu, E.x, 1);
      v[4].y = __shfl_down_sync(0xffffffffu, E.y, 1);
      if (lane == 0) {
        v[0] = va[0] ? row[x0 - 2] : mkc(0.0, 0.0);
        v[1] = va[1] ? row[x0 - 1] : mkc(0.0, 0.0);
      }
      if (lane == RSX - 1) v[4] = va[4] ? row[x0 + 2] : mkc(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < RRB; ++k) {
        const int b = r - 2 * k;
        if (b < 0 || b > 4) continue;  // compile-time
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          if (!va[a]) continue;
          const double w = kW16(b) * kW16(a);
          ar[k] = __dadd_rn(ar[k], __dmul_rn(w, v[a].x));
          ai[k] = __dadd_rn(ai[k], __dmul_rn(w, v[a].y));
        }
      }
    }
    // coarse row k is complete after its b = 4 fine row (r = 2k + 4)
    if (r >= 4 && ((r - 4) & 1) == 0) {
      const int k = (r - 4) / 2;
      if (k < ncy && cx < t.ncx) {
        const int cyg = cyg0 + k;
        c[(long long)(cy0 + k) * t.ncx + cx] = zrow(zero_mask, cx, cyg, t) ? mkc(0.0, 0.0) : mkc(ar[k], ai[k]);
      }
    }
  }
}

// fine point (y, x) gathers (w8_b w8_a) coarse((y+2-b)/2, (x+2-a)/2) over the
// (b, a) pairs of the right parity, in the reference's (b, a) order.
__global__ void __launch_bounds__(256) k_prolong(const cd* __restrict__ c, const cd* __restrict__ base,
                                                 cd* __restrict__ f, TGeom t, int accumulate) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int yl = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= t.nfx || yl >= t.f_ny) return;
  const int y = yl + t.f_row0;
  double ar = 0.0, ai = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int ty = y + 2 - b;
    if (ty & 1) continue;
    const int cy = ty >> 1;
    if (cy < 0 || cy >= t.ncy_g) continue;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int tx = x + 2 - a;
      if (tx & 1) continue;
      const int cx = tx >> 1;
      if (cx < 0 || cx >= t.ncx) continue;
      const double w = cW8[b] * cW8[a];
      const cd v = c[(long long)(cy - t.c_row0) * t.ncx + cx];
      ar = __dadd_rn(ar, __dmul_rn(w, v.x));
      ai = __dadd_rn(ai, __dmul_rn(w, v.y));
    }
  }
  const long long p = (long long)yl * t.nfx + x;
  if (accumulate) {
    const cd o = base[p];
    f[p] = mkc(__dadd_rn(o.x, ar), __dadd_rn(o.y, ai));
  } else {
    f[p] = mkc(ar, ai);
  }
}

// fine-level form: thread per coarse point writes the fine 2x2 block
// (2cy..2cy+1, 2cx..2cx+1) from the coarse 3x3 neighbourhood (same term order)
__global__ void __launch_bounds__(128) k_prolong_s(const cd* __restrict__ c, const cd* __restrict__ base,
                                                   cd* __restrict__ f, TGeom t, int cy_lo, int cy_cnt,
                                                   int accumulate) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= t.ncx || k >= cy_cnt) return;
  const int cy = cy_lo + k;  // global coarse row
  cd n[3][3];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) n[dy + 1][dx + 1] = ldc(c, t, cy + dy, cx + dx);
#pragma unroll
  for (int oy = 0; oy < 2; ++oy) {
    const int y = 2 * cy + oy;
    if (y < t.f_row0 || y >= t.f_row0 + t.f_ny) continue;
#pragma unroll
    for (int ox = 0; ox < 2; ++ox) {
      const int x = 2 * cx + ox;
      if (x >= t.nfx) continue;
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        if ((oy + 2 - b) & 1) continue;  // compile-time parity
        const int dy = (oy + 2 - b) / 2;
        if (cy + dy < 0 || cy + dy >= t.ncy_g) continue;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          if ((ox + 2 - a) & 1) continue;
          const int dx = (ox + 2 - a) / 2;
          if (cx + dx < 0 || cx + dx >= t.ncx) continue;
          const double w = cW8[b] * cW8[a];
          const cd v = n[dy + 1][dx + 1];
          ar = __dadd_rn(ar, __dmul_rn(w, v.x));
          ai = __dadd_rn(ai, __dmul_rn(w, v.y));
        }
      }
      const long long p = (long long)(y - t.f_row0) * t.nfx + x;
      if (accumulate) {
        const cd o = base[p];
        f[p] = mkc(__dadd_rn(o.x, ar), __dadd_rn(o.y, ai));
      } else {
        f[p] = mkc(ar, ai);
      }
    }
  }
}

TGeom full_tgeom(int nfx, int nfy) {
  TGeom t;
  t.nfx = nfx; t.f_row0 = 0; t.f_ny = nfy; t.nfy_g = nfy;
  t.ncx = (nfx - 1) / 2 + 1; t.ncy_g = (nfy - 1) / 2 + 1; t.c_row0 = 0; t.c_ny = t.ncy_g;
  return t;
}

void launch_restrict(const cd* fine, cd* coarse, const TGeom& t, int zero_mask, cudaStream_t st) {
  static const int mode = [] {
    const char* e = getenv("HDB_RESTRICT");
    return e ? atoi(e) : 2;
  }();
  if (mode == 2 && t.ncx >= 256 && t.c_ny >= 256) {
    const dim3 blk(RSX, RSY), grd((t.ncx + RSX - 1) / RSX, (t.c_ny + RSY * RRB - 1) / (RSY * RRB));
    k_restrict_s<<<grd, blk, 0, st>>>(fine, coarse, t, zero_mask);
    return;
  }
  if (mode >= 1 && t.ncx >= 64 && t.c_ny >= 64) {
    const dim3 blk(32, 8), grd((t.ncx + 31) / 32, ((t.c_ny + 1) / 2 + 7) / 8);
    k_restrict2<<<grd, blk, 0, st>>>(fine, coarse, t, zero_mask);
    return;
  }
  const dim3 blk(32, 8), grd((t.ncx + 31) / 32, (t.c_ny + 7) / 8);
  k_restrict<<<grd, blk, 0, st>>>(fine, coarse, t, zero_mask);
}

void launch_prolong(const cd* coarse, const cd* base, cd* fine, const TGeom& t, int accumulate, cudaStream_t st) {
  if (t.ncx >= 64 && t.f_ny >= 128) {
    const int cy_lo = t.f_row0 / 2, cy_hi = (t.f_row0 + t.f_ny - 1) / 2;  // coarse rows owning the fine rows
    const int cnt = cy_hi - cy_lo + 1;
    const dim3 blk(32, 4), grd((t.ncx + 31) / 32, (cnt + 3) / 4);
    k_prolong_s<<<grd, blk, 0, st>>>(coarse, base, fine, t, cy_lo, cnt, accumulate);
    return;
  }
  const dim3 blk(32, 8), grd((t.nfx + 31) / 32, (t.f_ny + 7) / 8);
  k_prolong<<<grd, blk, 0, st>>>(coarse, base, fine, t, accumulate);
}

}  // namespace hdb
