// Problem setup on the device: the k^2 field of the fine level
// from a velocity model, its injection down the hierarchy, range checks and the
// point-source right-hand side, without a host array of the fine grid.
//
// Reference: grid.py:220-287 (build_hierarchy / _fine_ksq: k^2 = (2 pi f / c)^2 at
// the vertices x = x0 + h i, coarse levels by injection at coincident vertices),
// grid.py:120-160 (wedge layers, bilinear raster sampling), grid.py:309-320 (point
// source 1 / (hx hy)).  Every expression is evaluated with explicit
// round-to-nearest operations in numpy's order, so the device fields are
// bit-identical to the host ones (tests/test_gpu_parity.py::test_device_setup_*).
// All kernels stream: 8 B written per fine point (+ 8 B read per coarse point).
#include "kernels.h"
#include "hdb_common.cuh"

namespace hdb {

__device__ __forceinline__ double coord(double o, double h, int i) { return __dadd_rn(o, __dmul_rn(h, (double)i)); }
__device__ __forceinline__ double ksq_of(double w, double c) {
  const double q = __ddiv_rn(w, c);
  return __dmul_rn(q, q);
}

__global__ void k_setup_fill(double* __restrict__ out, long long n, double v) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    out[p] = v;
}

// wedge (grid.py:120-135): layers (y at first x, y at last x, velocity) top to bottom; a
// vertex on or below a layer's interface that no earlier layer claimed takes its velocity
__global__ void k_setup_wedge(double* __restrict__ out, int nx, int ny, double ox, double oy, double hx, double hy,
                              double w, SetupLayers L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  const double x = coord(ox, hx, i), y = coord(oy, hy, j);
  const double x0 = coord(ox, hx, 0);
  const double span = nx > 1 ? __dsub_rn(coord(ox, hx, nx - 1), x0) : 1.0;
  double vel = L.v[L.n - 1];
  for (int q = 0; q < L.n - 1; ++q) {
    // y_first + (y_last - y_first) * (x - x0) / span
    const double surface =
        __dadd_rn(L.y0[q], __ddiv_rn(__dmul_rn(__dsub_rn(L.y1[q], L.y0[q]), __dsub_rn(x, x0)), span));
    if (y >= surface) {
      vel = L.v[q];
      break;
    }
  }
  out[(long long)j * nx + i] = ksq_of(w, vel);
}

// one raster axis (grid.py:138-143): cell, upper neighbour, fractional weight
__device__ __forceinline__ void raster_axis(double c, double origin, double step, int n, int& lo, int& hi, double& t) {
  double frac = __ddiv_rn(__dsub_rn(c, origin), step);
  frac = fmin(fmax(frac, 0.0), (double)n - 1.0);
  lo = n > 1 ? min((int)frac, n - 2) : 0;
  hi = min(lo + 1, n - 1);
  t = __dsub_rn(frac, (double)lo);
}

// bilinear raster (grid.py:146-160): corner order 00, 01, 10, 11, term = (g * w_col) * w_row
__global__ void k_setup_raster(double* __restrict__ out, int nx, int ny, double ox, double oy, double hx, double hy,
                               double w, const double* __restrict__ g, int rnx, int rny, double rx0, double ry0,
                               double rdx, double rdy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= nx || j >= ny) return;
  int ix0, ix1, iy0, iy1;
  double tx, ty;
  raster_axis(coord(ox, hx, i), rx0, rdx, rnx, ix0, ix1, tx);
  raster_axis(coord(oy, hy, j), ry0, rdy, rny, iy0, iy1, ty);
  const double ux = __dsub_rn(1.0, tx), uy = __dsub_rn(1.0, ty);
  const double* r0 = g + (long long)iy0 * rnx;
  const double* r1 = g + (long long)iy1 * rnx;
  double tot = __dmul_rn(__dmul_rn(r0[ix0], ux), uy);
  tot = __dadd_rn(tot, __dmul_rn(__dmul_rn(r0[ix1], tx), uy));
  tot = __dadd_rn(tot, __dmul_rn(__dmul_rn(r1[ix0], ux), ty));
  tot = __dadd_rn(tot, __dmul_rn(__dmul_rn(r1[ix1], tx), ty));
  out[(long long)j * nx + i] = ksq_of(w, tot);
}

// injection at coincident vertices (grid.py:285): coarse[j][i] = fine[2j][2i]
__global__ void k_setup_inject(const double* __restrict__ f, int nfx, double* __restrict__ c, int ncx, int ncy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= ncx || j >= ncy) return;
  c[(long long)j * ncx + i] = f[(long long)(2 * j) * nfx + 2 * i];
}

// (min, max, count of non-finite values): block partials, the last block combines them
constexpr int kStatThreads = 256;
__global__ void __launch_bounds__(kStatThreads) k_setup_stats(const double* __restrict__ a, long long n, double* part,
                                                              unsigned* ticket, double* out3) {
  __shared__ double smin[kStatThreads], smax[kStatThreads], sbad[kStatThreads];
  __shared__ bool last;
  double mn = INFINITY, mx = -INFINITY, bad = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const double v = a[p];
    if (!isfinite(v)) bad += 1.0;
    else { mn = fmin(mn, v); mx = fmax(mx, v); }
  }
  auto block_reduce = [&] {
    smin[threadIdx.x] = mn; smax[threadIdx.x] = mx; sbad[threadIdx.x] = bad;
    __syncthreads();
    for (int s = kStatThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
        smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
        sbad[threadIdx.x] += sbad[threadIdx.x + s];
      }
      __syncthreads();
    }
  };
  block_reduce();
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = smin[0]; part[3 * blockIdx.x + 1] = smax[0]; part[3 * blockIdx.x + 2] = sbad[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  mn = INFINITY; mx = -INFINITY; bad = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kStatThreads) {
    const volatile double* q = part + 3 * b;
    mn = fmin(mn, q[0]); mx = fmax(mx, q[1]); bad += q[2];
  }
  __syncthreads();
  block_reduce();
  if (threadIdx.x == 0) {
    out3[0] = smin[0]; out3[1] = smax[0]; out3[2] = sbad[0];
    *ticket = 0u;
  }
}

__global__ void k_setup_point(cd* rhs, long long idx, double v) { rhs[idx] = mkc(v, 0.0); }

static inline dim3 grid2(int nx, int ny) { return dim3((nx + 31) / 32, (ny + 7) / 8); }

void launch_setup_fill(double* out, long long n, double v, cudaStream_t st) {
  const int blocks = (int)std::min<long long>((n + 1023) / 1024, 148 * 8);
  k_setup_fill<<<blocks < 1 ? 1 : blocks, 256, 0, st>>>(out, n, v);
}
void launch_setup_wedge(double* out, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                        const SetupLayers& L, cudaStream_t st) {
  k_setup_wedge<<<grid2(nx, ny), dim3(32, 8), 0, st>>>(out, nx, ny, ox, oy, hx, hy, w, L);
}
void launch_setup_raster(double* out, int nx, int ny, double ox, double oy, double hx, double hy, double w,
                         const double* g, int rnx, int rny, double rx0, double ry0, double rdx, double rdy,
                         cudaStream_t st) {
  k_setup_raster<<<grid2(nx, ny), dim3(32, 8), 0, st>>>(out, nx, ny, ox, oy, hx, hy, w, g, rnx, rny, rx0, ry0, rdx, rdy);
}
void launch_setup_inject(const double* fine, int nfx, double* coarse, int ncx, int ncy, cudaStream_t st) {
  k_setup_inject<<<grid2(ncx, ncy), dim3(32, 8), 0, st>>>(fine, nfx, coarse, ncx, ncy);
}
int setup_stats_blocks(long long n) {
  const long long b = (n + kStatThreads * 8 - 1) / (kStatThreads * 8);
  return (int)std::max<long long>(1, std::min<long long>(b, kMaxReduceBlocks));
}
void launch_setup_stats(const double* a, long long n, double* part, unsigned* ticket, double* out3, cudaStream_t st) {
  k_setup_stats<<<setup_stats_blocks(n), kStatThreads, 0, st>>>(a, n, part, ticket, out3);
}
void launch_setup_point(cd* rhs, long long n, long long idx, double v, cudaStream_t st) {
  cudaMemsetAsync(rhs, 0, sizeof(cd) * (size_t)n, st);
  k_setup_point<<<1, 1, 0, st>>>(rhs, idx, v);
}

}  // namespace hdb
