// Microbenchmark: cost of one MGS-style reduction step inside a 16-CTA cluster.
// variants: 0 block reduce only; 1 + DSMEM push/mbarrier all-gather;
// 2 + cluster.sync instead; 3 = 1 + global loads of a fresh vector chunk.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double2 wsum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) { v.x += __shfl_down_sync(~0u, v.x, o); v.y += __shfl_down_sync(~0u, v.y, o); }
  return v;
}

template <int T, int V>
__global__ void k(const double2* __restrict__ vec, long long n, int steps, double* out) {
  __shared__ uint64_t mbar[2];
  __shared__ double2 gather[2][16];
  __shared__ double2 warp[T / 32];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), rank = cl.block_rank();
  uint32_t par[2] = {0, 0};
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar[0])), "r"(16 * C));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar[1])), "r"(16 * C));
  }
  cl.sync();
  double2 acc = {1e-3 * threadIdx.x, 0.0};
  int b = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double2 v = acc;
    if (V == 3) {
      const long long p = ((long long)s * C * T + rank * T + threadIdx.x) % n;
      const double2 q = vec[p];
      v.x += q.x; v.y += q.y;
    }
    v = wsum(v);
    if ((threadIdx.x & 31) == 0) warp[threadIdx.x >> 5] = v;
    __syncthreads();
    double2 tt = {0, 0};
    if (threadIdx.x < 32) { tt = threadIdx.x < T / 32 ? warp[threadIdx.x] : double2{0, 0}; tt = wsum(tt); }
    if (V == 0) {
      if (threadIdx.x == 0) gather[b][0] = tt;
      __syncthreads();
      acc.x += gather[b][0].x * 1e-9;
    } else if (V == 2) {
      if (threadIdx.x == 0) gather[b][rank] = tt;
      cl.sync();
      double2 q = {0, 0};
      if (threadIdx.x < 32 && threadIdx.x < C) q = *cl.map_shared_rank(&gather[b][rank], threadIdx.x);
      if (threadIdx.x < 32) q = wsum(q);
      if (threadIdx.x == 0) warp[0] = q;
      __syncthreads();
      acc.x += warp[0].x * 1e-9;
    } else {
      if (threadIdx.x == 0) {
        const uint32_t la = sa(&gather[b][rank]), lb = sa(&mbar[b]);
        for (int r = 0; r < C; ++r) {
          uint32_t ra, rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(r));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                       ::"r"(ra), "d"(tt.x), "d"(tt.y), "r"(rb) : "memory");
        }
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.b32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(sa(&mbar[b])), "r"(par[b]) : "memory");
      par[b] ^= 1;
      double2 q = {0, 0};
      for (int r = 0; r < C; ++r) { q.x += gather[b][r].x; q.y += gather[b][r].y; }
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar[b])), "r"(16 * C));
      acc.x += q.x * 1e-9;
    }
    b ^= 1;
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && rank == 0) { out[0] = (double)(t1 - t0) / steps; out[1] = acc.x; }
}

template <int T, int V>
void run(const char* name, int C, double2* vec, long long n, double* d) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(C); cfg.blockDim = dim3(T); cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<T, V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int steps = 2000;
  cudaLaunchKernelEx(&cfg, k<T, V>, (const double2*)vec, n, steps, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<T, V>, (const double2*)vec, n, steps, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-28s C=%2d T=%4d  %7.1f cycles/step  %6.3f us/step  err=%s\n", name, C, T, h[0], ms * 1e3 / steps,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double2* vec; double* d; long long n = 1 << 22;
  cudaMalloc(&vec, n * 16); cudaMemset(vec, 0, n * 16); cudaMalloc(&d, 64);
  for (int C : {16, 8}) {
    run<512, 0>("block reduce only", C, vec, n, d);
    run<512, 1>("push all-gather", C, vec, n, d);
    run<512, 2>("cluster.sync + DSMEM", C, vec, n, d);
    run<512, 3>("push + fresh global load", C, vec, n, d);
    run<256, 1>("push all-gather", C, vec, n, d);
    run<128, 1>("push all-gather", C, vec, n, d);
    run<128, 3>("push + fresh global load", C, vec, n, d);
  }
  return 0;
}
