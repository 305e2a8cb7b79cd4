// Deterministic single-launch grid reductions (shared by the BLAS and the fused
// stencil kernels): warp/block trees in a fixed order, per-block partials, and
// the last block to finish (threadfence + ticket) combining them in block order.
#pragma once
#include "hdb_common.cuh"

namespace hdb {

__device__ __forceinline__ cd warp_sum(cd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// block-wide sum in fixed order (1-D block of NT threads); result valid in thread 0
template <int NT = kReduceThreads>
__device__ __forceinline__ cd block_sum(cd v) {
  __shared__ cd sw[NT / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sw[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < NT / 32 ? sw[lane] : mkc(0.0, 0.0);
    v = warp_sum(v);
  }
  __syncthreads();
  return v;
}

// finish a grid reduction: every block deposits its partial; the last one
// sums partials[0..G) in order and stores to *dst (optionally only the real
// part as a squared norm).
// Returns true (block-uniform) in the block that wrote *dst -- callers hang small
// single-thread epilogues on it (the value is visible to that block's thread 0).
template <int NT = kReduceThreads>
__device__ __forceinline__ bool grid_finish(cd part, cd* partials, unsigned* ticket, cd* dst) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = part;
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  cd v = mkc(0.0, 0.0);
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const volatile double* q = (const volatile double*)(partials + b);
    v.x += q[0];
    v.y += q[1];
  }
  v = block_sum<NT>(v);
  if (threadIdx.x == 0) {
    *dst = v;
    *ticket = 0u;
  }
  return true;
}

}  // namespace hdb
