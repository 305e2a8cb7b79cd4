// Higher-order transfers Z^T (restriction, (1,4,6,4,1)/16 per dim) and Z
// (prolongation, (1,4,6,4,1)/8 per dim, scatter form), zero extension.
//
// Reference: transfers.py:59-88.  The reference accumulates 25 strided numpy
// passes in (b, a) row-major order starting from zeros; each pass adds
// round(w_b w_a * v) (w products are exact dyadic rationals).  The gather
// kernels below add the same terms in the same order, so results are
// bit-identical.  Algorithmic traffic: 20 B per fine point each way
// (fine 16 B read/write + coarse 16 B / 4).
#include "kernels.h"
#include "hdb_common.cuh"

namespace hdb {

__constant__ double cW16[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
__constant__ double cW8[5] = {1.0 / 8, 4.0 / 8, 6.0 / 8, 4.0 / 8, 1.0 / 8};

// coarse point (cy, cx) = sum_{b,a} (w16_b w16_a) fine(2cy+b-2, 2cx+a-2)
// zero_rows/zero_cols: coarse Dirichlet rows set to 0 (mg.py:118-119), bit mask
// (1 west, 2 east, 4 south, 8 north); 0 for the deflation path.
__global__ void __launch_bounds__(256) k_restrict(const cd* __restrict__ f, cd* __restrict__ c, int nfx,
                                                  int nfy, int ncx, int ncy, int zero_mask) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= ncx || cy >= ncy) return;
  const long long p = (long long)cy * ncx + cx;
  if (((zero_mask & 1) && cx == 0) || ((zero_mask & 2) && cx == ncx - 1) ||
      ((zero_mask & 4) && cy == 0) || ((zero_mask & 8) && cy == ncy - 1)) {
    c[p] = mkc(0.0, 0.0);
    return;
  }
  double ar = 0.0, ai = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int y = 2 * cy + b - 2;
    if (y < 0 || y >= nfy) continue;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      if (x < 0 || x >= nfx) continue;
      const double w = cW16[b] * cW16[a];
      const cd v = f[(long long)y * nfx + x];
      ar = __dadd_rn(ar, __dmul_rn(w, v.x));
      ai = __dadd_rn(ai, __dmul_rn(w, v.y));
    }
  }
  c[p] = mkc(ar, ai);
}

// fine point (y, x) gathers (w8_b w8_a) coarse((y+2-b)/2, (x+2-a)/2) over the
// (b, a) pairs of the right parity, in the reference's (b, a) order.
// accumulate: out = base + Zc  (mg.py:121 x + prolong(ec)); else out = Zc.
__global__ void __launch_bounds__(256) k_prolong(const cd* __restrict__ c, const cd* __restrict__ base,
                                                 cd* __restrict__ f, int nfx, int nfy, int ncx, int ncy,
                                                 int accumulate) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= nfx || y >= nfy) return;
  double ar = 0.0, ai = 0.0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const int ty = y + 2 - b;
    if (ty & 1) continue;
    const int cy = ty >> 1;
    if (cy < 0 || cy >= ncy) continue;
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int tx = x + 2 - a;
      if (tx & 1) continue;
      const int cx = tx >> 1;
      if (cx < 0 || cx >= ncx) continue;
      const double w = cW8[b] * cW8[a];
      const cd v = c[(long long)cy * ncx + cx];
      ar = __dadd_rn(ar, __dmul_rn(w, v.x));
      ai = __dadd_rn(ai, __dmul_rn(w, v.y));
    }
  }
  const long long p = (long long)y * nfx + x;
  if (accumulate) {
    const cd o = base[p];
    f[p] = mkc(__dadd_rn(o.x, ar), __dadd_rn(o.y, ai));
  } else {
    f[p] = mkc(ar, ai);
  }
}

// ------------------------------------------------------------------------
// Fine-level forms.
__device__ __forceinline__ cd ldf(const cd* f, int nfx, int nfy, int y, int x) {
  return (y >= 0 && y < nfy && x >= 0 && x < nfx) ? f[(long long)y * nfx + x] : mkc(0.0, 0.0);
}

// Prolongation: a thread owns coarse point (cy, cx) and writes the fine 2x2
// block (2cy..2cy+1, 2cx..2cx+1) from the coarse 3x3 neighbourhood; each fine
// value adds its terms in the reference's (b, a) order.
__device__ __forceinline__ cd ldc(const cd* c, int ncx, int ncy, int y, int x) {
  return (y >= 0 && y < ncy && x >= 0 && x < ncx) ? c[(long long)y * ncx + x] : mkc(0.0, 0.0);
}

__global__ void __launch_bounds__(128) k_prolong_s(const cd* __restrict__ c, const cd* __restrict__ base,
                                                   cd* __restrict__ f, int nfx, int nfy, int ncx, int ncy,
                                                   int accumulate) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= ncx || cy >= ncy) return;
  cd n[3][3];  // n[dy+1][dx+1] = coarse(cy+dy, cx+dx)
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) n[dy + 1][dx + 1] = ldc(c, ncx, ncy, cy + dy, cx + dx);
#pragma unroll
  for (int oy = 0; oy < 2; ++oy) {
    const int y = 2 * cy + oy;
    if (y >= nfy) continue;
#pragma unroll
    for (int ox = 0; ox < 2; ++ox) {
      const int x = 2 * cx + ox;
      if (x >= nfx) continue;
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        if ((oy + 2 - b) & 1) continue;          // compile-time parity
        const int dy = (oy + 2 - b) / 2;         // coarse row offset in {-1, 0, 1}
        if (cy + dy < 0 || cy + dy >= ncy) continue;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          if ((ox + 2 - a) & 1) continue;
          const int dx = (ox + 2 - a) / 2;
          if (cx + dx < 0 || cx + dx >= ncx) continue;
          const double wgt = cW8[b] * cW8[a];
          const cd v = n[dy + 1][dx + 1];
          ar = __dadd_rn(ar, __dmul_rn(wgt, v.x));
          ai = __dadd_rn(ai, __dmul_rn(wgt, v.y));
        }
      }
      const long long p = (long long)y * nfx + x;
      if (accumulate) {
        const cd o = base[p];
        f[p] = mkc(__dadd_rn(o.x, ar), __dadd_rn(o.y, ai));
      } else {
        f[p] = mkc(ar, ai);
      }
    }
  }
}

// two coarse rows per thread (cy, cy+1): fine rows 2cy-2..2cy+4, each loaded
// once and fed to two independent (b, a)-ordered accumulation chains
__global__ void __launch_bounds__(256) k_restrict2(const cd* __restrict__ f, cd* __restrict__ c, int nfx, int nfy,
                                                   int ncx, int ncy, int zero_mask) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int cy = 2 * (blockIdx.y * blockDim.y + threadIdx.y);
  if (cx >= ncx || cy >= ncy) return;
  double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
#pragma unroll
  for (int r = 0; r < 7; ++r) {
    const int y = 2 * cy - 2 + r;
    if (y < 0 || y >= nfy) continue;
    cd v[5];
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      v[a] = (x >= 0 && x < nfx) ? f[(long long)y * nfx + x] : mkc(0.0, 0.0);
    }
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      const int x = 2 * cx + a - 2;
      if (x < 0 || x >= nfx) continue;
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
  auto zero = [&](int yy) {
    return ((zero_mask & 1) && cx == 0) || ((zero_mask & 2) && cx == ncx - 1) || ((zero_mask & 4) && yy == 0) ||
           ((zero_mask & 8) && yy == ncy - 1);
  };
  c[(long long)cy * ncx + cx] = zero(cy) ? mkc(0.0, 0.0) : mkc(ar, ai);
  if (cy + 1 < ncy) c[(long long)(cy + 1) * ncx + cx] = zero(cy + 1) ? mkc(0.0, 0.0) : mkc(br, bi);
}

void launch_restrict(const cd* fine, cd* coarse, int nfx, int nfy, int zero_mask, cudaStream_t st) {
  const int ncx0 = (nfx - 1) / 2 + 1, ncy0 = (nfy - 1) / 2 + 1;
  if (ncx0 >= 64 && ncy0 >= 64) {
    const dim3 blk(32, 8), grd((ncx0 + 31) / 32, ((ncy0 + 1) / 2 + 7) / 8);
    k_restrict2<<<grd, blk, 0, st>>>(fine, coarse, nfx, nfy, ncx0, ncy0, zero_mask);
    return;
  }
  const int ncx = (nfx - 1) / 2 + 1, ncy = (nfy - 1) / 2 + 1;
  const dim3 blk(32, 8), grd((ncx + 31) / 32, (ncy + 7) / 8);
  k_restrict<<<grd, blk, 0, st>>>(fine, coarse, nfx, nfy, ncx, ncy, zero_mask);
}

void launch_prolong(const cd* coarse, const cd* base, cd* fine, int nfx, int nfy, int accumulate,
                    cudaStream_t st) {
  const int ncx = (nfx - 1) / 2 + 1, ncy = (nfy - 1) / 2 + 1;
  if (ncx >= 64 && ncy >= 64) {
    const dim3 blk(32, 4), grd((ncx + 31) / 32, (ncy + 3) / 4);
    k_prolong_s<<<grd, blk, 0, st>>>(coarse, base, fine, nfx, nfy, ncx, ncy, accumulate);
    return;
  }
  const dim3 blk(32, 8), grd((nfx + 31) / 32, (nfy + 7) / 8);
  k_prolong<<<grd, blk, 0, st>>>(coarse, base, fine, nfx, nfy, ncx, ncy, accumulate);
}

}  // namespace hdb
