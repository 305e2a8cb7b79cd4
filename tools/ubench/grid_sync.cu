// Microbenchmark: cost of a grid-wide barrier / deterministic reduction in a
// cooperative launch over all SMs.
// 0: cg::grid.sync(); 1: partial store + grid.sync + read all partials (GridSync::reduce);
// 2: custom barrier: per-CTA atomicAdd on a counter + spin on the generation word;
// 3: custom all-reduce: partials + counter; the last CTA sums, publishes, bumps generation.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int V>
__global__ void k(double* part, unsigned* bar, double* out, int steps) {
  cg::grid_group g = cg::this_grid();
  double acc = threadIdx.x * 1e-3;
  const int P = gridDim.x;
  __shared__ double bc;
  unsigned gen = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    if (V == 0) {
      g.sync();
    } else if (V == 1) {
      if (threadIdx.x == 0) part[(s & 1) * P + blockIdx.x] = acc;
      g.sync();
      if (threadIdx.x < 32) {
        double q = 0;
        for (int r = threadIdx.x; r < P; r += 32) q += __ldcg(&part[(s & 1) * P + r]);
        for (int o = 16; o > 0; o >>= 1) q += __shfl_down_sync(~0u, q, o);
        if (threadIdx.x == 0) bc = q;
      }
      __syncthreads();
      acc += bc * 1e-12;
    } else if (V == 2) {
      __syncthreads();
      if (threadIdx.x == 0) {
        gen++;
        __threadfence();
        const unsigned t = atomicAdd(&bar[0], 1u);
        if (t == (unsigned)P * gen - 1) atomicExch(&bar[1], gen);
        while (ld_acquire(&bar[1]) < gen) {}
      }
      __syncthreads();
    } else {
      // last-arriver reduction: partial, fence, ticket; last CTA sums in order and publishes
      if (threadIdx.x == 0) {
        gen++;
        part[(s & 1) * P + blockIdx.x] = acc;
        __threadfence();
        const unsigned t = atomicAdd(&bar[0], 1u);
        if (t == (unsigned)P * gen - 1) {
          double q = 0;
          for (int r = 0; r < P; ++r) q += __ldcg(&part[(s & 1) * P + r]);
          __stcg(&out[2 + (s & 1)], q);
          __threadfence();
          atomicExch(&bar[1], gen);
        }
        while (ld_acquire(&bar[1]) < gen) {}
        bc = __ldcg(&out[2 + (s & 1)]);
      }
      __syncthreads();
      acc += bc * 1e-12;
    }
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = (double)(t1 - t0) / steps; out[1] = acc; }
}

template <int V>
void run(const char* name, int P, int T) {
  double *part, *out; unsigned* bar;
  cudaMalloc(&part, 2 * P * 8); cudaMalloc(&out, 64); cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  int steps = 2000;
  void* args[] = {&part, &bar, &out, &steps};
  cudaLaunchCooperativeKernel((void*)k<V>, dim3(P), dim3(T), args, 0, 0);
  cudaMemset(bar, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)k<V>, dim3(P), dim3(T), args, 0, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("%-34s P=%3d T=%4d  %8.1f cycles/step  %6.3f us/step  %s\n", name, P, T, h[0], ms * 1e3 / steps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(part); cudaFree(out); cudaFree(bar);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int P : {sms, 64, 16}) {
    run<0>("cg grid.sync", P, 512);
    run<1>("GridSync::reduce (partials+sync)", P, 512);
    run<2>("custom counter barrier", P, 512);
    run<3>("last-arriver reduction", P, 512);
  }
  return 0;
}
