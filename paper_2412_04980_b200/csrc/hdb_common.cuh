// Shared device/host definitions for the B200 MADP-FGMRES library.
//
// Arithmetic policy: the library is compiled with -fmad=false and every
// operation that has a reference counterpart is written with explicit
// round-to-nearest intrinsics in the reference's operation order, so level
// operators, Jacobi sweeps and transfers are bit-identical to the reference
// (numba loops without fastmath, numpy strided passes).  Reductions (dots)
// use FMA and a fixed tree order: deterministic, but not bit-identical to
// OpenBLAS zdotc.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

#define HDB_BC_SOMMERFELD 0
#define HDB_BC_DIRICHLET 1

namespace hdb {

typedef double2 cd;  // complex128, interleaved (re, im) = numpy complex128 layout

__host__ __device__ inline cd mkc(double r, double i) { cd z; z.x = r; z.y = i; return z; }

// ---- exact (no-FMA) complex helpers -------------------------------------
__device__ __forceinline__ cd c_add(cd a, cd b) { return mkc(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ cd c_sub(cd a, cd b) { return mkc(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
// textbook product (numba complex multiply, no contraction)
__device__ __forceinline__ cd c_mul(cd a, cd b) {
  return mkc(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
             __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// real * complex, componentwise (exact equivalent of (s+0i)*z for finite values)
__device__ __forceinline__ cd c_scale(double s, cd z) { return mkc(__dmul_rn(s, z.x), __dmul_rn(s, z.y)); }
// numpy's AVX-512 complex128 multiply of scalar a by array element b:
//   re = fma(a.re, b.re, -(a.im*b.im)),  im = fma(a.re, b.im, a.im*b.re)
__device__ __forceinline__ cd c_mul_np(cd a, cd b) {
  return mkc(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
// conj(a) * b with FMA (reductions only)
__device__ __forceinline__ cd c_conjmul_acc(cd acc, cd a, cd b) {
  acc.x = __fma_rn(a.x, b.x, acc.x); acc.x = __fma_rn(a.y, b.y, acc.x);
  acc.y = __fma_rn(a.x, b.y, acc.y); acc.y = __fma_rn(-a.y, b.x, acc.y);
  return acc;
}

// ---- level geometry ----------------------------------------------------------
// A level array holds rows [0, ny) of a slab whose first row is global row
// `row0` of a grid with `nyg` rows; physical boundaries (closure rules) apply
// only at global rows 0 / nyg-1 and columns 0 / nx-1.  Arrays are row-major
// (x fastest), pitch nx; for a slab, `halo` rows above and below row 0 / ny-1
// are addressable (filled by the halo exchange).  Single GPU: row0 = 0, ny = nyg.
struct Geom {
  int nx, ny;      // local extent
  int row0, nyg;   // global offset / global rows
};

// Coefficients of one level operator  -Lap - shift*I(k^2)  (operators.py:99-117)
struct OpCoef {
  int radius;            // 1, 2 or 3
  int bc[4];             // west, east, south, north
  double h;
  double s;              // radius 1: lap_coef[1,1] / 4
  cd mc;                 // radius 1: mass_coef[1,1]
  double E;              // radius 1: (-s*2)*h  (Sommerfeld diagonal increment factor)
  double lap[49];        // (2r+1)^2 row-major lap_coef
  cd mass[49];           // (2r+1)^2 row-major mass_coef
  int uniform;           // k^2 is one constant on this level (host-checked): ucoef valid
  double ku;             // that constant
  cd ucoef[49];          // lap + mass * ku per tap, same rounded operations as the per-point form
  const int* skip = nullptr;  // device flag: nonzero -> the launch does nothing (device-driven loops)
  // separable form of a radius-2/3 Galerkin level:
  //   lap[a][b] = lsc * (sa[a] sm[b] + sm[a] sa[b]),  mass[a][b] = msc * sm[a] sm[b]
  // (host-verified reconstruction); used unless the exact tap order is requested
  int sep = 0;
  double sa[7], sm[7];
  double lsc;
  cd msc;
};

// Raise a kernel's dynamic shared-memory limit to >= bytes on the current device,
// once per (device, kernel) and size; thread-safe (rank threads share a process).
inline bool ensure_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{dev, fn}];
  if (bytes <= cur) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) return false;
  cur = bytes;
  return true;
}

constexpr int kReduceThreads = 256;
constexpr int kMaxReduceBlocks = 592;  // 4 x 148 SMs

}  // namespace hdb
