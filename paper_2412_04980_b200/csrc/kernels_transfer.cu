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
#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime's driver entry point)

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
    if (r >= 5 && cy + 1 >= t.c_ny) continue;  // rows only the absent second coarse row needs (beyond a slab's halo)
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
__host__ __device__ constexpr double kW8(int i) { return kw5(i) / 8; }

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

// ---------------------------------------------------------------------------
// TMA-staged restriction (fine levels).  A CTA owns 62 coarse columns (two
// consumer warps, lane = coarse column) and a strip of TSR coarse rows; a third
// warp is the producer: its lane 0 streams the strip's 2*TSR + 3 fine rows,
// two rows per tensor copy (box = 256 doubles x 2 rows: fine columns
// 2*cx0 - 2 .. 2*cx0 + 125, 2 KB contiguous per row), HBM -> shared memory through a TST-stage ring
// (full barriers completed by the copy engine, empty barriers by the two
// consumer warps).  The tensor map spans the GLOBAL fine grid, so columns and
// rows outside it arrive as zeros -- exactly the reference's zero extension
// (transfers.py:59-72) -- and no CTA needs a boundary path.  The consumers sum
// the 25 terms of each coarse point in the reference's (b, a) order with the
// rotating-accumulator walk (pairs of fine rows; products shared between b =
// 0/4 and b = 1/3), so results are bit-identical to k_restrict.
constexpr int TCC = 62;        // coarse columns per CTA (2*62 + 3 fine columns fit one 128-point box row)
constexpr int TBC = 128;       // box columns (fine points per staged row: 2 KB contiguous)
constexpr uint32_t kTBoxBytes = 2u * TBC * 16u;
template <int TST>
struct TRing {
  uint64_t full[TST], empty[TST];
  double scratch[64];  // consumer-side release dependencies
};
__device__ __forceinline__ uint32_t s_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arm(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.b32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(s_addr(b)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(s_addr(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s_addr(bar))
      : "memory");
}
// the five fine values v[a] = fine(2cx + a - 2) of one staged row (E/O loads,
// neighbours by shuffles, warp-edge lanes read their outer values directly)
__device__ __forceinline__ void srow_taps(cd v[5], const cd* row, int col, int lane) {
  const cd E = row[col + 2], O = row[col + 3];
  v[2] = E;
  v[3] = O;
  v[0].x = __shfl_up_sync(0xffffffffu, E.x, 1);
  v[0].y = __shfl_up_sync(0xffffffffu, E.y, 1);
  v[1].x = __shfl_up_sync(0xffffffffu, O.x, 1);
  v[1].y = __shfl_up_sync(0xffffffffu, O.y, 1);
  v[4].x = __shfl_down_sync(0xffffffffu, E.x, 1);
  v[4].y = __shfl_down_sync(0xffffffffu, E.y, 1);
  if (lane == 0) { v[0] = row[col]; v[1] = row[col + 1]; }
  if (lane == 31) v[4] = row[min(col + 4, TBC - 1)];
}
__device__ __forceinline__ void wprod(cd p[5], const cd v[5], double wb) {
#pragma unroll
  for (int a = 0; a < 5; ++a) {
    const double w = wb * kW16(a);  // exact (dyadic)
    p[a] = mkc(__dmul_rn(w, v[a].x), __dmul_rn(w, v[a].y));
  }
}
__device__ __forceinline__ void wacc(cd& acc, const cd p[5]) {
#pragma unroll
  for (int a = 0; a < 5; ++a) acc = mkc(__dadd_rn(acc.x, p[a].x), __dadd_rn(acc.y, p[a].y));
}

template <int TST, int TSR>  // ring stages (row pairs), coarse rows per CTA
__global__ void __launch_bounds__(96) k_restrict_t(const __grid_constant__ CUtensorMap fmap, cd* __restrict__ c,
                                                   TGeom t, int zero_mask) {
  extern __shared__ __align__(128) unsigned char tsm[];
  cd* ring = reinterpret_cast<cd*>(tsm);                          // TST x (2 rows x TBC)
  TRing<TST>& rb = *reinterpret_cast<TRing<TST>*>(tsm + (size_t)TST * kTBoxBytes);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cx0 = blockIdx.x * TCC;
  const int cy0 = blockIdx.y * TSR;                 // local coarse row
  const int cyg0 = cy0 + t.c_row0;
  const int y0 = 2 * cyg0 - 2;                      // first fine row (global; may be -2 -> zero rows)
  if (threadIdx.x == 0) {
    for (int q = 0; q < TST; ++q) {
      bar_init(&rb.full[q], 1);
      bar_init(&rb.empty[q], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ncy = min(TSR, t.c_ny - cy0);
  const int np = ncy + 2;  // row pairs this strip needs (slab strips may be short)
  if (wid == 2) {  // producer
    if (lane == 0) {
      for (int p = 0; p < np; ++p) {
        const int q = p % TST;
        if (p >= TST) bar_wait(&rb.empty[q], (uint32_t)((p / TST - 1) & 1));
        bar_arm(&rb.full[q], kTBoxBytes);
        tma_load_2d(ring + (size_t)q * 2 * TBC, &fmap, 2 * (2 * cx0 - 2), y0 + 2 * p, &rb.full[q]);
      }
    }
    return;
  }
  const int cc = wid * 32 + lane;         // coarse column within the CTA (62, 63: idle lanes)
  const int col = 2 * min(cc, TCC);       // staged index of fine column 2cx - 2 (idle lanes clamped in range)
  const int cx = cc < TCC ? cx0 + cc : t.ncx;
  cd A0 = mkc(0.0, 0.0), A1 = mkc(0.0, 0.0), A2 = mkc(0.0, 0.0);  // coarse rows p-2, p-1, p
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
    const int q = p % TST;
    bar_wait(&rb.full[q], (uint32_t)((p / TST) & 1));
    const cd* r0 = ring + (size_t)q * 2 * TBC;
    cd v0[5], v1[5];
    srow_taps(v0, r0, col, lane);
    srow_taps(v1, r0 + TBC, col, lane);
    cd pr[5], pr1[5];
    wprod(pr, v0, kW16(0));
    wprod(pr1, v1, kW16(1));
    // The stage is released only once every value read from it has been
    // consumed: this scratch store depends on all of them (the products of the
    // lane-0 / lane-31 halo loads included), so no shared load can still be in
    // flight when the copy engine refills the stage.
    rb.scratch[threadIdx.x] = __dadd_rn(__dadd_rn(__dadd_rn(pr[0].x, pr[1].x), pr[4].x),
                                        __dadd_rn(__dadd_rn(pr1[0].x, pr1[1].x), pr1[4].x));
    __syncwarp();
    if (lane == 0) bar_arrive(&rb.empty[q]);
    // even row 2p: b = 4 -> A0, b = 2 -> A1, b = 0 -> A2 (w_4 = w_0)
    if (p >= 2) wacc(A0, pr);
    if (p >= 1 && p - 1 < TSR) {
      cd p2[5];
      wprod(p2, v0, kW16(2));
      wacc(A1, p2);
    }
    if (p < TSR) wacc(A2, pr);
    if (p >= 2) {
      const int k = p - 2;
      if (k < ncy && cx < t.ncx)
        c[(long long)(cy0 + k) * t.ncx + cx] = zrow(zero_mask, cx, cyg0 + k, t) ? mkc(0.0, 0.0) : A0;
    }
    // odd row 2p+1: b = 3 -> A1, b = 1 -> A2 (w_3 = w_1); not needed in the last pair
    if (p + 1 < np) {
      if (p >= 1 && p - 1 < TSR) wacc(A1, pr1);
      if (p < TSR) wacc(A2, pr1);
    }
    A0 = A1;
    A1 = A2;
    A2 = mkc(0.0, 0.0);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}
// fine grid (global rows 0..nfy_g) as a 2-D f64 tensor {2 * column + re/im, row};
// false when the encoder is unavailable or rejects the geometry
static bool fine_map(CUtensorMap* m, const cd* fine, const TGeom& t) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cd* base = fine - (long long)t.f_row0 * t.nfx;  // global row 0 (rows outside the slab + halo are never requested)
  const cuuint64_t dims[2] = {2 * (cuuint64_t)t.nfx, (cuuint64_t)t.nfy_g};  // doubles (re, im interleaved) x rows
  const cuuint64_t strides[1] = {(cuuint64_t)t.nfx * 16};
  const cuuint32_t box[2] = {2 * TBC, 2};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// encoded maps of recently used fine vectors (a solve reuses its level vectors)
struct MapEntry {
  const cd* ptr;
  int nfx, nfy_g, f_row0;
  CUtensorMap map;
};
static bool cached_fine_map(CUtensorMap* m, const cd* fine, const TGeom& t) {
  static thread_local MapEntry cache[32];
  static thread_local int n = 0, next = 0;
  for (int i = 0; i < n; ++i) {
    const MapEntry& e = cache[i];
    if (e.ptr == fine && e.nfx == t.nfx && e.nfy_g == t.nfy_g && e.f_row0 == t.f_row0) {
      *m = e.map;
      return true;
    }
  }
  if (!fine_map(m, fine, t)) return false;
  MapEntry& e = cache[next];
  e.ptr = fine; e.nfx = t.nfx; e.nfy_g = t.nfy_g; e.f_row0 = t.f_row0; e.map = *m;
  next = (next + 1) % 32;
  if (n < 32) ++n;
  return true;
}
template <int TST, int TSR>
static void launch_restrict_tk(const CUtensorMap& m, cd* coarse, const TGeom& t, int zero_mask, cudaStream_t st) {
  constexpr size_t smem = (size_t)TST * kTBoxBytes + sizeof(TRing<TST>);
  ensure_smem_attr((const void*)k_restrict_t<TST, TSR>, smem);
  const dim3 grd((t.ncx + TCC - 1) / TCC, (t.c_ny + TSR - 1) / TSR);
  k_restrict_t<TST, TSR><<<grd, 96, smem, st>>>(m, coarse, t, zero_mask);
}
static bool launch_restrict_t(const cd* fine, cd* coarse, const TGeom& t, int zero_mask, int variant,
                              cudaStream_t st) {
  CUtensorMap m;
  if (!cached_fine_map(&m, fine, t)) return false;
  if (variant == 4) launch_restrict_tk<4, 32>(m, coarse, t, zero_mask, st);
  else if (variant == 5) launch_restrict_tk<3, 32>(m, coarse, t, zero_mask, st);
  else if (variant == 6) launch_restrict_tk<4, 16>(m, coarse, t, zero_mask, st);
  else launch_restrict_tk<3, 32>(m, coarse, t, zero_mask, st);  // default: 3 stages (more CTAs per SM beat deeper rings, measured)
  return true;
}

// ---------------------------------------------------------------------------
// TMA-staged prolongation (fine levels).  A CTA owns 62 coarse columns (two
// consumer warps, lane = coarse column) and a strip of PSR coarse rows; the
// producer warp's lane 0 streams coarse rows cy0-1 .. cy0+PSR (box 128
// doubles = coarse columns cx0-1 .. cx0+62; columns / rows outside the grid
// arrive as zeros, whose +0 terms leave every sum unchanged -- the reference
// drops them) and, for the accumulate form, the two base rows of each output
// pair.  Consumers keep a 3-row register window, form the fine rows 2cy and
// 2cy+1 (E = 2cx, O = 2cx+1, (b, a) term order of k_prolong: bit-identical),
// stage them in shared memory and one thread writes them back with a tensor
// store (clipped at the grid edge), double-buffered against the next pair.
constexpr int PSR = 32;                    // coarse rows per CTA
constexpr int PST = 4;                     // ring stages
constexpr int PCC = 62;                    // coarse columns per CTA
constexpr int POB = 2 * PCC;               // fine points per staged output row (124)
constexpr uint32_t kPCoarseBytes = 128u * 8u;          // one coarse row box (64 points)
constexpr uint32_t kPBaseBytes = 2u * POB * 16u;        // two base rows
struct PRing {
  uint64_t full[PST], empty[PST];
};
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s_addr(src)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(96) k_prolong_t(const __grid_constant__ CUtensorMap cmap,
                                                  const __grid_constant__ CUtensorMap bmap,
                                                  const __grid_constant__ CUtensorMap fmap, TGeom t, int cy_lo,
                                                  int cy_cnt, int accumulate) {
  extern __shared__ __align__(128) unsigned char psm[];
  // layout: coarse ring (PST x 1 KB) | base ring (PST x 3968 B, accumulate) | out (2 x 3968 B) | 2 scratch | barriers
  cd* cring = reinterpret_cast<cd*>(psm);
  cd* bring = reinterpret_cast<cd*>(psm + PST * kPCoarseBytes);
  cd* obuf = reinterpret_cast<cd*>(psm + PST * (kPCoarseBytes + kPBaseBytes));
  PRing& rb = *reinterpret_cast<PRing*>(psm + PST * (kPCoarseBytes + kPBaseBytes) + 2 * kPBaseBytes + 2 * sizeof(cd));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cx0 = blockIdx.x * PCC;
  const int k0 = blockIdx.y * PSR;
  const int cy0 = cy_lo + k0;                   // first coarse row (global)
  const int nrow = min(PSR, cy_cnt - k0);       // output coarse rows of this strip
  const int nitems = nrow + 2;                  // coarse rows cy0-1 .. cy0+nrow
  if (threadIdx.x == 0) {
    for (int q = 0; q < PST; ++q) {
      bar_init(&rb.full[q], 1);
      bar_init(&rb.empty[q], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == 2) {  // producer
    if (lane == 0) {
      for (int k = 0; k < nitems; ++k) {
        const int q = k % PST;
        if (k >= PST) bar_wait(&rb.empty[q], (uint32_t)((k / PST - 1) & 1));
        const bool wb = accumulate && k >= 2;
        bar_arm(&rb.full[q], kPCoarseBytes + (wb ? kPBaseBytes : 0u));
        tma_load_2d(cring + (size_t)q * 64, &cmap, 2 * (cx0 - 1), cy0 - 1 + k, &rb.full[q]);
        if (wb) tma_load_2d(bring + (size_t)q * 2 * POB, &bmap, 4 * cx0, 2 * (cy0 + k - 2), &rb.full[q]);
      }
    }
    return;
  }
  const int cc = min(wid * 32 + lane, PCC - 1);  // idle lanes (62, 63) mirror column 61 (never stored)
  const bool live = wid * 32 + lane < PCC;
  cd L0, C0, R0, L1, C1, R1;
  // window rows cy0-1 (item 0) and cy0 (item 1).  A stage is released only
  // after the values read from it have been consumed by arithmetic (a shared
  // load still in flight must not race the copy engine refilling the stage),
  // so items 0 and 1 are released after output 0.
  for (int k = 0; k < 2; ++k) {
    bar_wait(&rb.full[k], 0);
    const cd* row = cring + (size_t)k * 64;
    if (k == 0) { L0 = row[cc]; C0 = row[cc + 1]; R0 = row[cc + 2]; }
    else { L1 = row[cc]; C1 = row[cc + 1]; R1 = row[cc + 2]; }
  }
  const double w0 = kW8(0), w1 = kW8(1), w2 = kW8(2), w3 = kW8(3), w4 = kW8(4);
#pragma unroll 1
  for (int i = 0; i < nrow; ++i) {
    const int k = i + 2, q = k % PST;
    bar_wait(&rb.full[q], (uint32_t)((k / PST) & 1));
    const cd* row = cring + (size_t)q * 64;
    const cd L2 = row[cc], C2 = row[cc + 1], R2 = row[cc + 2];  // coarse row cy+1
    cd bE0, bO0, bE1, bO1;
    if (accumulate) {
      const cd* br = bring + (size_t)q * 2 * POB;
      bE0 = br[2 * cc]; bO0 = br[2 * cc + 1]; bE1 = br[POB + 2 * cc]; bO1 = br[POB + 2 * cc + 1];
    }
    // fine row 2cy: b = 0 -> cy+1, b = 2 -> cy, b = 4 -> cy-1;  E: a = 0, 2, 4 (R, C, L), O: a = 1, 3 (R, C)
    double er = 0.0, ei = 0.0, orr = 0.0, oi = 0.0;
#define PT(wb, LL, CC_, RR)                                                                                  \
    er = __dadd_rn(er, __dmul_rn((wb) * w0, RR.x)); ei = __dadd_rn(ei, __dmul_rn((wb) * w0, RR.y));           \
    er = __dadd_rn(er, __dmul_rn((wb) * w2, CC_.x)); ei = __dadd_rn(ei, __dmul_rn((wb) * w2, CC_.y));         \
    er = __dadd_rn(er, __dmul_rn((wb) * w4, LL.x)); ei = __dadd_rn(ei, __dmul_rn((wb) * w4, LL.y));           \
    orr = __dadd_rn(orr, __dmul_rn((wb) * w1, RR.x)); oi = __dadd_rn(oi, __dmul_rn((wb) * w1, RR.y));         \
    orr = __dadd_rn(orr, __dmul_rn((wb) * w3, CC_.x)); oi = __dadd_rn(oi, __dmul_rn((wb) * w3, CC_.y));
    PT(w0, L2, C2, R2)
    PT(w2, L1, C1, R1)
    PT(w4, L0, C0, R0)
    cd E0 = mkc(er, ei), O0 = mkc(orr, oi);
    er = ei = orr = oi = 0.0;
    PT(w1, L2, C2, R2)
    PT(w3, L1, C1, R1)
#undef PT
    cd E1 = mkc(er, ei), O1 = mkc(orr, oi);
    if (accumulate) {
      E0 = mkc(__dadd_rn(bE0.x, E0.x), __dadd_rn(bE0.y, E0.y));
      O0 = mkc(__dadd_rn(bO0.x, O0.x), __dadd_rn(bO0.y, O0.y));
      E1 = mkc(__dadd_rn(bE1.x, E1.x), __dadd_rn(bE1.y, E1.y));
      O1 = mkc(__dadd_rn(bO1.x, O1.x), __dadd_rn(bO1.y, O1.y));
    }
    // stage and store: the store that last read this buffer (pair i-2) has been
    // waited for by thread 0 before the previous iteration's closing barrier
    cd* ob = obuf + (size_t)(i & 1) * 2 * POB;
    named_sync(1, 64);
    if (live) {
      ob[2 * cc] = E0; ob[2 * cc + 1] = O0;
      ob[POB + 2 * cc] = E1; ob[POB + 2 * cc + 1] = O1;
    } else {
      obuf[4 * POB + (wid * 32 + lane - PCC)] = E0;  // idle lanes: scratch slots after both buffers
    }
    // Release stage q (and, at i = 0, items 0 and 1) only now: these shared
    // stores depend on every value read from the stage, so no shared load can
    // still be in flight when the copy engine refills it.
    __syncwarp();
    if (lane == 0) {
      bar_arrive(&rb.empty[q]);
      if (i == 0) { bar_arrive(&rb.empty[0]); bar_arrive(&rb.empty[1]); }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    named_sync(1, 64);
    if (threadIdx.x == 0) {
      tma_store_2d(&fmap, 4 * cx0, 2 * (cy0 + i), ob);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    L0 = L1; C0 = C1; R0 = R1;
    L1 = L2; C1 = C2; R1 = R2;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static bool map2d(CUtensorMap* m, const cd* base_row0, int ncols, int nrows, uint32_t box_doubles, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {2 * (cuuint64_t)ncols, (cuuint64_t)nrows};
  const cuuint64_t strides[1] = {(cuuint64_t)ncols * 16};
  const cuuint32_t box[2] = {box_doubles, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base_row0, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
struct PMapEntry {
  const cd *c, *b, *f;
  int nfx, nfy_g, f_row0, c_row0;
  CUtensorMap cm, bm, fm;
};
static bool launch_prolong_t(const cd* coarse, const cd* base, cd* fine, const TGeom& t, int accumulate,
                             cudaStream_t st) {
  static thread_local PMapEntry cache[32];
  static thread_local int n = 0, next = 0;
  PMapEntry* e = nullptr;
  for (int i = 0; i < n && !e; ++i)
    if (cache[i].c == coarse && cache[i].b == base && cache[i].f == fine && cache[i].nfx == t.nfx &&
        cache[i].nfy_g == t.nfy_g && cache[i].f_row0 == t.f_row0 && cache[i].c_row0 == t.c_row0)
      e = &cache[i];
  if (!e) {
    PMapEntry ne;
    ne.c = coarse; ne.b = base; ne.f = fine; ne.nfx = t.nfx; ne.nfy_g = t.nfy_g; ne.f_row0 = t.f_row0;
    ne.c_row0 = t.c_row0;
    const cd* c0 = coarse - (long long)t.c_row0 * t.ncx;  // global coarse row 0
    const cd* f0 = fine - (long long)t.f_row0 * t.nfx;
    const cd* b0 = base ? base - (long long)t.f_row0 * t.nfx : f0;
    if (!map2d(&ne.cm, c0, t.ncx, t.ncy_g, 128, 1) || !map2d(&ne.bm, b0, t.nfx, t.nfy_g, 2 * POB, 2) ||
        !map2d(&ne.fm, f0, t.nfx, t.nfy_g, 2 * POB, 2))
      return false;
    cache[next] = ne;
    e = &cache[next];
    next = (next + 1) % 32;
    if (n < 32) ++n;
  }
  constexpr size_t smem = PST * (kPCoarseBytes + kPBaseBytes) + 2 * kPBaseBytes + 2 * sizeof(cd) + sizeof(PRing);
  ensure_smem_attr((const void*)k_prolong_t, smem);
  const int cy_lo = t.f_row0 / 2, cy_hi = (t.f_row0 + t.f_ny - 1) / 2;
  const int cnt = cy_hi - cy_lo + 1;
  const dim3 grd((t.ncx + PCC - 1) / PCC, (cnt + PSR - 1) / PSR);
  k_prolong_t<<<grd, 96, smem, st>>>(e->cm, e->bm, e->fm, t, cy_lo, cnt, accumulate);
  return true;
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

// the 2x2 fine block (2cy..2cy+1, 2cx..2cx+1) of coarse point (cy, cx) from its
// 3x3 coarse neighbourhood, every bound checked (same term order as k_prolong)
__device__ __forceinline__ void prolong_point(const cd* __restrict__ c, const cd* __restrict__ base,
                                              cd* __restrict__ f, const TGeom& t, int cx, int cy, int accumulate) {
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

// fine-level form: thread per coarse point writes the fine 2x2 block
// (2cy..2cy+1, 2cx..2cx+1) from the coarse 3x3 neighbourhood (same term order)
__global__ void __launch_bounds__(128) k_prolong_s(const cd* __restrict__ c, const cd* __restrict__ base,
                                                   cd* __restrict__ f, TGeom t, int cy_lo, int cy_cnt,
                                                   int accumulate) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y * blockDim.y + threadIdx.y;
  if (cx >= t.ncx || k >= cy_cnt) return;
  prolong_point(c, base, f, t, cx, cy_lo + k, accumulate);
}

// Half-warp-interleaved prolongation for fine levels: lane l of a warp owns
// coarse column c = cxw + (l & 15) and fine parity p = l >> 4, i.e. fine column
// 2c + p, so every store (and the base load of the accumulate form) of the
// warp is one contiguous 512-byte access.  Each lane forms its fine value as
// wR*R + wC*C + wL*L per contributing coarse row (R, C, L = coarse columns
// c+1, c, c-1; odd columns have wL = 0, whose +0 term leaves the sum
// unchanged), which is the reference's (b, a) term order.  Coarse rows stream
// through a 3-row register window (one new row per coarse row).  Blocks that
// touch a boundary or the slab edge take the per-point path of k_prolong_s.
constexpr int PHB = 16;  // coarse rows per thread
__device__ __forceinline__ void ld_crow(const cd* q, cd& L, cd& C, cd& R) {
  L = q[-1];
  C = q[0];
  R = q[1];
}
__device__ __forceinline__ void pterm(double& ar, double& ai, double wr, double wc, double wl, cd L, cd C, cd R) {
  ar = __dadd_rn(ar, __dmul_rn(wr, R.x)); ai = __dadd_rn(ai, __dmul_rn(wr, R.y));
  ar = __dadd_rn(ar, __dmul_rn(wc, C.x)); ai = __dadd_rn(ai, __dmul_rn(wc, C.y));
  ar = __dadd_rn(ar, __dmul_rn(wl, L.x)); ai = __dadd_rn(ai, __dmul_rn(wl, L.y));
}
__device__ __noinline__ void prolong_block_generic(const cd* __restrict__ c, const cd* __restrict__ base,
                                                   cd* __restrict__ f, TGeom t, int cx, int cy0, int kend,
                                                   int accumulate) {
  for (int kk = 0; kk < kend; ++kk) prolong_point(c, base, f, t, cx, cy0 + kk, accumulate);
}
__global__ void __launch_bounds__(128) k_prolong_h(const cd* __restrict__ c, const cd* __restrict__ base,
                                                   cd* __restrict__ f, TGeom t, int cy_lo, int cy_cnt, int accumulate) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cxw = blockIdx.x * 64 + wid * 16;  // this warp's 16 coarse columns
  const int k0 = blockIdx.y * PHB;
  if (k0 >= cy_cnt) return;
  const int cy0 = cy_lo + k0;
  const int bx0 = blockIdx.x * 64;
  const bool interior = bx0 >= 1 && bx0 + 63 <= t.ncx - 2 && cy0 >= 1 && cy0 + PHB <= t.ncy_g - 1 &&
                        k0 + PHB <= cy_cnt && 2 * cy0 >= t.f_row0 && 2 * (cy0 + PHB - 1) + 1 < t.f_row0 + t.f_ny;
  if (!interior) {
    // generic: thread per coarse point (the block's 64 columns x PHB rows)
    const int cx = bx0 + (threadIdx.x & 63);
    if (cx >= t.ncx) return;
    const int half = threadIdx.x >> 6;  // two threads per column: rows split in halves
    const int kb = k0 + half * (PHB / 2), ke = min(k0 + (half + 1) * (PHB / 2), cy_cnt);
    if (kb < ke) prolong_block_generic(c, base, f, t, cx, cy_lo + kb, ke - kb, accumulate);
    return;
  }
  const int cc = cxw + (lane & 15), par = lane >> 4;
  // weights of (R, C, L) for this lane's parity: even fine column a = 0, 2, 4; odd a = 1, 3
  const double wr = par ? kW8(1) : kW8(0), wc = par ? kW8(3) : kW8(2), wl = par ? 0.0 : kW8(4);
  const long long ncx = t.ncx, nfx = t.nfx;
  const cd* cp = c + (long long)(cy0 - 1 - t.c_row0) * ncx + cc;
  cd L0, C0, R0, L1, C1, R1, L2, C2, R2;
  ld_crow(cp, L0, C0, R0);
  ld_crow(cp + ncx, L1, C1, R1);
  cd nL, nC, nR;
  ld_crow(cp + 2 * ncx, nL, nC, nR);
  cd* fp = f + (long long)(2 * cy0 - t.f_row0) * nfx + 2 * cc + par;
  const cd* bp = accumulate ? base + (long long)(2 * cy0 - t.f_row0) * nfx + 2 * cc + par : nullptr;
#pragma unroll 2
  for (int k = 0; k < PHB; ++k) {
    L2 = nL; C2 = nC; R2 = nR;  // coarse row cy0 + k + 1
    if (k + 1 < PHB) ld_crow(cp + (long long)(k + 3) * ncx, nL, nC, nR);
    const double w0 = kW8(0), w1 = kW8(1), w2 = kW8(2), w3 = kW8(3), w4 = kW8(4);
    // fine row 2cy: b = 0 -> cy+1, b = 2 -> cy, b = 4 -> cy-1
    double ar = 0.0, ai = 0.0;
    pterm(ar, ai, w0 * wr, w0 * wc, w0 * wl, L2, C2, R2);
    pterm(ar, ai, w2 * wr, w2 * wc, w2 * wl, L1, C1, R1);
    pterm(ar, ai, w4 * wr, w4 * wc, w4 * wl, L0, C0, R0);
    cd* o = fp + (long long)(2 * k) * nfx;
    if (bp) {
      const cd ob = bp[(long long)(2 * k) * nfx];
      *o = mkc(__dadd_rn(ob.x, ar), __dadd_rn(ob.y, ai));
    } else {
      *o = mkc(ar, ai);
    }
    // fine row 2cy+1: b = 1 -> cy+1, b = 3 -> cy
    ar = ai = 0.0;
    pterm(ar, ai, w1 * wr, w1 * wc, w1 * wl, L2, C2, R2);
    pterm(ar, ai, w3 * wr, w3 * wc, w3 * wl, L1, C1, R1);
    o += nfx;
    if (bp) {
      const cd ob = bp[(long long)(2 * k + 1) * nfx];
      *o = mkc(__dadd_rn(ob.x, ar), __dadd_rn(ob.y, ai));
    } else {
      *o = mkc(ar, ai);
    }
    L0 = L1; C0 = C1; R0 = R1;
    L1 = L2; C1 = C2; R1 = R2;
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
    return e ? atoi(e) : 3;
  }();
  // TMA-staged form on large grids (its per-strip pipeline latency does not pay on small ones)
  if (mode >= 3 && t.ncx >= 1024 && t.c_ny >= 512 && launch_restrict_t(fine, coarse, t, zero_mask, mode, st)) return;
  if (mode >= 2 && t.ncx >= 256 && t.c_ny >= 256) {
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
  static const int pmode = [] {
    const char* e = getenv("HDB_PROLONG");
    return e ? atoi(e) : 3;
  }();
  // TMA-staged form on large grids (its per-strip pipeline latency does not pay on small ones)
  if (pmode == 3 && t.ncx >= 1024 && t.f_ny >= 1024 && launch_prolong_t(coarse, base, fine, t, accumulate, st)) return;
  if (pmode == 2 && t.ncx >= 256 && t.f_ny >= 256) {
    const int cy_lo = t.f_row0 / 2, cy_hi = (t.f_row0 + t.f_ny - 1) / 2;
    const int cnt = cy_hi - cy_lo + 1;
    const dim3 grd((t.ncx + 63) / 64, (cnt + PHB - 1) / PHB);
    k_prolong_h<<<grd, 128, 0, st>>>(coarse, base, fine, t, cy_lo, cnt, accumulate);
    return;
  }
  if (pmode >= 1 && t.ncx >= 64 && t.f_ny >= 128) {
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
