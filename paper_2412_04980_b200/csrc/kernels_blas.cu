// Krylov vector kernels: deterministic conj-dots, fused MGS steps, scaling,
// solution update, combine.  Reference: krylov.py:121-174, parallel.py:168-199.
//
// Reductions are single-launch and deterministic: a fixed grid (function of
// n only) writes per-block partials, the last block to finish (threadfence +
// ticket) sums them in a fixed order and writes the scalar to device memory.
// Nothing returns to the host here; the Krylov driver reads the Hessenberg
// column once per Arnoldi step.
#include <cstdio>
#include <cstdlib>
#include <functional>

#include "kernels.h"
#include "hdb_common.cuh"
#include "reduce.cuh"

namespace hdb {

int reduce_blocks(long long n) {
  long long b = (n + kReduceThreads * 4 - 1) / (kReduceThreads * 4);
  if (b < 1) b = 1;
  if (b > kMaxReduceBlocks) b = kMaxReduceBlocks;
  return (int)b;
}

// dst = <u, v> = sum conj(u) v
__global__ void __launch_bounds__(kReduceThreads) k_dot(const cd* __restrict__ u, const cd* __restrict__ v,
                                                        long long n, cd* partials, unsigned* ticket, cd* dst) {
  cd acc = mkc(0.0, 0.0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    acc = c_conjmul_acc(acc, u[p], v[p]);
  acc = block_sum(acc);
  grid_finish(acc, partials, ticket, dst);
}

// the one-iteration FGMRES scalar update (krylov.py:126-168 for m = 1): Givens, y_0, count
__device__ __forceinline__ void step1_update(const cd* b2, const cd* h0p, const cd* hn2, cd* y_out, int* its_out, cd* flag) {
  const double beta = sqrt(fmax(b2->x, 0.0));
  if (beta == 0.0) {
    *y_out = mkc(0.0, 0.0);
    *its_out = 0;
    return;
  }
  const cd h1 = *h0p;
  const double hn = sqrt(fmax(hn2->x, 0.0));
  const bool finite = isfinite(h1.x) && isfinite(h1.y) && isfinite(hn) && isfinite(beta);
  const double a1 = hypot(h1.x, h1.y), a2 = hn;
  double c, sr, si;  // s = (sr, si)
  if (a2 == 0.0) { c = 1.0; sr = 0.0; si = 0.0; }
  else if (a1 == 0.0) { c = 0.0; sr = 1.0; si = 0.0; }
  else {
    const double t = hypot(a1, a2);
    c = a1 / t;
    sr = (h1.x / a1) * hn / t;  // (h1/|h1|) conj(hn) / t with hn real
    si = (h1.y / a1) * hn / t;
  }
  const double rr = c * h1.x + sr * hn, ri = c * h1.y + si * hn;  // R00 = c h1 + s h2
  const double g = c * beta;
  const double d = rr * rr + ri * ri;
  *y_out = mkc(g * rr / d, -g * ri / d);
  *its_out = 1;
  if (!finite || !(d > 0.0)) flag->x = 2.0;
}

// Fused MGS step (krylov.py:121-124):  w -= h * vi  (h = *hsrc, numpy complex
// scalar*array then subtract);  then dst = <vn, w_new> (vn = w for the norm).
// vi == nullptr skips the update (first dot of the chain).
// epi.b2 != null: the block that finishes the reduction also runs the one-iteration FGMRES
// update on (b2, h0, *dst) -- the step1 control kernel folded into the norm launch
__global__ void __launch_bounds__(kReduceThreads) k_mgs(cd* __restrict__ w, const cd* __restrict__ vi,
                                                        const cd* hsrc, const cd* __restrict__ vn, long long n,
                                                        cd* partials, unsigned* ticket, cd* dst, Step1Epi epi) {
  const cd h = vi ? *hsrc : mkc(0.0, 0.0);
  cd acc = mkc(0.0, 0.0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    cd x = w[p];
    if (vi) {
      x = c_sub(x, c_mul_np(h, vi[p]));
      w[p] = x;
    }
    const cd a = vn ? vn[p] : x;
    acc = c_conjmul_acc(acc, a, x);
  }
  acc = block_sum(acc);
  if (grid_finish(acc, partials, ticket, dst) && epi.b2 && threadIdx.x == 0)
    step1_update(epi.b2, epi.h0, dst, epi.y, epi.its, epi.flag);
}

// dst = ||b - t||^2 (real part) without storing the difference (krylov.py:174)
// guard != null: a non-finite result raises the NumericalError flag (k_finite_guard folded in)
__global__ void __launch_bounds__(kReduceThreads) k_subnorm(const cd* __restrict__ b, const cd* __restrict__ t,
                                                            long long n, cd* partials, unsigned* ticket, cd* dst,
                                                            cd* guard) {
  cd acc = mkc(0.0, 0.0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd d = c_sub(b[p], t[p]);
    acc = c_conjmul_acc(acc, d, d);
  }
  acc = block_sum(acc);
  if (grid_finish(acc, partials, ticket, dst) && guard && threadIdx.x == 0 && !isfinite(dst->x)) guard->x = 2.0;
}

// out = x * inv   (numpy  x / beta  ==  (x.re * (1/beta), x.im * (1/beta)))
__global__ void k_scale(const cd* __restrict__ x, cd* __restrict__ out, double inv, long long n) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd v = x[p];
    out[p] = mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv));
  }
}

// x = x0 + sum_i y_i * B_i, terms added in order (krylov.py:169-172); x0 may be null (zeros)
__global__ void k_lincomb(const cd* const* __restrict__ basis, const cd* __restrict__ y, int m,
                          const cd* __restrict__ x0, cd* __restrict__ x, long long n) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    cd acc = x0 ? x0[p] : mkc(0.0, 0.0);
    for (int i = 0; i < m; ++i) acc = c_add(acc, c_mul_np(y[i], basis[i][p]));
    x[p] = acc;
  }
}

// out = a + b   /  out = a - b
__global__ void k_add(const cd* __restrict__ a, const cd* __restrict__ b, cd* __restrict__ out, long long n, int sub) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    out[p] = sub ? c_sub(a[p], b[p]) : c_add(a[p], b[p]);
}

// out = y + a x  (sub = 0)  /  out = y - a x  (sub = 1); numpy scalar*array then add/sub
__global__ void k_axpy(const cd* __restrict__ y, cd a, const cd* __restrict__ x, cd* __restrict__ out, long long n,
                       int sub) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd t = c_mul_np(a, x[p]);
    out[p] = sub ? c_sub(y[p], t) : c_add(y[p], t);
  }
}

// Bi-CGSTAB direction (krylov.py:218): p = r + beta * (p - omega * v)
__global__ void k_bicg_p(const cd* __restrict__ r, cd* __restrict__ pv, const cd* __restrict__ v, cd beta, cd omega,
                         long long n) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    pv[p] = c_add(r[p], c_mul_np(beta, c_sub(pv[p], c_mul_np(omega, v[p]))));
}

// small dense complex GEMV  x = Ainv b  (MG coarsest solve, n <= 4096)
__global__ void __launch_bounds__(256) k_gemv(const cd* __restrict__ A, const cd* __restrict__ b, cd* __restrict__ x,
                                              int n) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const cd* row = A + (long long)warp * n;
  cd acc = mkc(0.0, 0.0);
  for (int c = lane; c < n; c += 32) {
    const cd a = row[c], v = b[c];
    acc.x = __fma_rn(a.x, v.x, acc.x); acc.x = __fma_rn(-a.y, v.y, acc.x);
    acc.y = __fma_rn(a.x, v.y, acc.y); acc.y = __fma_rn(a.y, v.x, acc.y);
  }
  acc = warp_sum(acc);
  if (lane == 0) x[warp] = acc;
}

// out = x * (1/sqrt(max(nrm2->x, 0)))  (V0 = r0 / beta with beta on device; 0 if beta == 0)
__global__ void k_scale_dev(const cd* __restrict__ x, cd* __restrict__ out, const cd* nrm2, long long n,
                            const int* skip) {
  if (skip && *skip) return;
  const double beta = sqrt(fmax(nrm2->x, 0.0));
  const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd v = x[p];
    out[p] = mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv));
  }
}

// One-step FGMRES closure on device (krylov.py:130-168 with m = 1): from
// b2 = ||b||^2, h0 = <V0, A z0>, hn2 = ||w||^2 form the Givens rotation, the
// recurrence residual and y0 = c*beta / (c h0 + s hn).  Writes y0, the
// iteration count (0 when b = 0) and raises the non-finite flag (2.0).
__global__ void k_step1(const cd* b2, const cd* h0p, const cd* hn2, cd* y_out, int* its_out, cd* flag) {
  step1_update(b2, h0p, hn2, y_out, its_out, flag);
}

// non-finite guard on a device scalar (explicit final residual, krylov.py:174-176)
__global__ void k_finite_guard(const cd* v, cd* flag) {
  if (!isfinite(v->x)) flag->x = 2.0;
}

// MG divergence guard (mg.py:133-138): flag |= sqrt(post2) > guard*sqrt(bn2)
__global__ void k_guard(const cd* post2, const cd* bn2, const cd* r02, double guard, cd* flag) {
  // bn2 == nullptr: ||b||^2 rides in post2's imaginary part (fused k_resnorm)
  const double post = sqrt(fmax(post2->x, 0.0)), bn = sqrt(fmax(bn2 ? bn2->x : post2->y, 0.0));
  const double r0 = r02 ? sqrt(fmax(r02->x, 0.0)) : bn;
  if (bn > 0.0 && post > guard * fmax(r0, bn)) flag->x = 1.0;
}

static inline int ew_blocks(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------
// Low-synchronisation MGS step for levels whose w does not fit on chip (the fine
// level of config 2: 16.8M points): the same algorithm as k_mgs_ls (h = (I + L)^{-1}
// V^H w, T = (I + L)^{-1} rows kept across the Arnoldi steps) as streaming passes
// over HBM instead of the fused MGS chain's j + 2 launches of 64 B/pt:
//   pass A  groups of kLsG basis vectors: g_k = <V_k, w>, l_k = <V_j, V_k>, and
//           <V_j, w> with the first group -> per-block partials;
//   finish  one block: ordered sum of the partials, the new T row, h = T g;
//   pass B  groups: w -= h_j V_j, then h_k V_k for k = j-1 .. 0; the last group
//           also forms the per-block partials of ||w||^2;
//   norm    one block: ordered sum -> hout[j + 1].
// At Arnoldi step j it moves (ceil(j/8) + ceil((j+1)/8)) 32 + 2 (j+1) 16 B/pt instead of
// (j+2) 64: 640 vs 1024 B/pt at j = 14.
constexpr int kLsG = 8;
constexpr int kLsPE = 2 * kLsG + 1;  // partial elements per block per group

__global__ void __launch_bounds__(kReduceThreads, 2) k_lsh_a(const cd* __restrict__ w, const cd* __restrict__ vj,
                                                          const cd* const* V, int k0, int kn, int with_gj,
                                                          long long n, cd* part, const int* skip) {
  if (skip && *skip) return;  // device-driven loops: the solve is already done
  cd g[kLsG], l[kLsG], gj = mkc(0.0, 0.0);
  const cd* vk[kLsG];
#pragma unroll
  for (int u = 0; u < kLsG; ++u) {
    g[u] = mkc(0.0, 0.0);
    l[u] = mkc(0.0, 0.0);
    vk[u] = u < kn ? V[k0 + u] : nullptr;
  }
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd wv = w[p], vv = vj[p];
    cd r[kLsG];
#pragma unroll
    for (int u = 0; u < kLsG; ++u) r[u] = u < kn ? vk[u][p] : mkc(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kLsG; ++u) {
      if (u < kn) {
        g[u] = c_conjmul_acc(g[u], r[u], wv);
        l[u] = c_conjmul_acc(l[u], vv, r[u]);
      }
    }
    if (with_gj) gj = c_conjmul_acc(gj, vv, wv);
  }
  cd* out = part + (long long)blockIdx.x * kLsPE;
#pragma unroll
  for (int u = 0; u < kLsG; ++u) {
    if (u < kn) {  // kn is grid-uniform: every thread takes part in the block sums
      const cd a = block_sum(g[u]);
      const cd b = block_sum(l[u]);
      if (threadIdx.x == 0) { out[u] = a; out[kLsG + u] = b; }
    }
  }
  if (with_gj) {
    const cd a = block_sum(gj);
    if (threadIdx.x == 0) out[2 * kLsG] = a;
  }
}

__device__ __forceinline__ void cfma_(cd& a, cd x, cd y) {  // a += x * y
  a.x = __fma_rn(x.x, y.x, a.x); a.x = __fma_rn(-x.y, y.y, a.x);
  a.y = __fma_rn(x.x, y.y, a.y); a.y = __fma_rn(x.y, y.x, a.y);
}

// ordered sum of the block partials -> sums[0 .. 2j] (g_0..g_j, l_0..l_{j-1}); one block
// of 1024 threads; part: [group][block][kLsPE].  A sharded level all-reduces `sums`
// (one collective per Arnoldi step) before k_lsh_th.
constexpr int kLshF = 1024;
__global__ void __launch_bounds__(kLshF) k_lsh_sum(const cd* part, int nblocks, int j, cd* sums, const int* skip) {
  if (skip && *skip) return;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int ne = 2 * j + 1;
  for (int e = wid; e < ne; e += kLshF / 32) {
    // element e -> (group, slot): g_k and l_k live in group k / kLsG; g_j in group 0's extra slot
    int grp, slot;
    if (e < j) { grp = e / kLsG; slot = e % kLsG; }
    else if (e == j) { grp = 0; slot = 2 * kLsG; }
    else { const int k = e - j - 1; grp = k / kLsG; slot = kLsG + k % kLsG; }
    const cd* src = part + (long long)grp * nblocks * kLsPE + slot;
    cd a = mkc(0.0, 0.0);
    for (int b0 = lane; b0 < nblocks; b0 += 32 * 8) {  // 8 loads in flight per lane, block order per lane
      cd z[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + 32 * u;
        z[u] = b < nblocks ? src[(long long)b * kLsPE] : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { a.x += z[u].x; a.y += z[u].y; }
    }
    a = warp_sum(a);
    if (lane == 0) sums[e] = a;
  }
}

// the new T row and h = T g from the reduced sums (every rank identically)
__global__ void __launch_bounds__(kLshF) k_lsh_th(const cd* sums, int j, cd* Tg, cd* hout, const int* skip) {
  __shared__ cd tot[2 * 512 + 1];
  __shared__ cd trow[512];
  if (skip && *skip) return;
  const int t = threadIdx.x;
  for (int e = t; e < 2 * j + 1; e += kLshF) tot[e] = sums[e];
  __syncthreads();
  const long long rj = (long long)j * (j + 1) / 2;
  if (t < j) {  // t_jk = -sum_{m=k}^{j-1} l_m T_mk
    cd a = mkc(0.0, 0.0);
    for (int m0 = t; m0 < j; m0 += 8) {
      cd tm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tm[u] = m0 + u < j ? Tg[(long long)(m0 + u) * (m0 + u + 1) / 2 + t] : mkc(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (m0 + u < j) cfma_(a, tot[j + 1 + m0 + u], tm[u]);
    }
    trow[t] = mkc(-a.x, -a.y);
    Tg[rj + t] = trow[t];
  }
  if (t == 0) Tg[rj + j] = mkc(1.0, 0.0);
  __syncthreads();
  if (t <= j) {  // h_i = sum_{k <= i} T_ik g_k
    cd a = mkc(0.0, 0.0);
    const long long ri = (long long)t * (t + 1) / 2;
    for (int k0 = 0; k0 <= t; k0 += 8) {
      cd tk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        tk[u] = k > t ? mkc(0.0, 0.0) : (t < j ? (k < t ? Tg[ri + k] : mkc(1.0, 0.0)) : (k < j ? trow[k] : mkc(1.0, 0.0)));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u <= t) cfma_(a, tk[u], tot[k0 + u]);
    }
    hout[t] = a;
  }
}

// w -= h_k V_k for k = kfirst, kfirst-1, ..., kfirst-kn+1 (descending); norm != 0: per-block ||w||^2
__global__ void __launch_bounds__(kReduceThreads) k_lsh_b(cd* __restrict__ w, const cd* const* V, const cd* h,
                                                          int kfirst, int kn, int norm, long long n, cd* part,
                                                          const int* skip) {
  if (skip && *skip) return;
  cd hk[kLsG];
  const cd* vk[kLsG];
#pragma unroll
  for (int u = 0; u < kLsG; ++u) {
    hk[u] = u < kn ? h[kfirst - u] : mkc(0.0, 0.0);
    vk[u] = u < kn ? V[kfirst - u] : nullptr;
  }
  cd acc = mkc(0.0, 0.0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    cd x = w[p];
    cd r[kLsG];
#pragma unroll
    for (int u = 0; u < kLsG; ++u) r[u] = u < kn ? vk[u][p] : mkc(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kLsG; ++u)
      if (u < kn) x = c_sub(x, c_mul_np(hk[u], r[u]));
    w[p] = x;
    if (norm) acc = c_conjmul_acc(acc, x, x);
  }
  if (norm) {
    const cd a = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = a;
  }
}

__global__ void __launch_bounds__(kReduceThreads) k_lsh_norm(const cd* part, int nblocks, cd* dst, const int* skip) {
  if (skip && *skip) return;
  cd v = mkc(0.0, 0.0);
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) { v.x += part[b].x; v.y += part[b].y; }
  v = block_sum(v);
  if (threadIdx.x == 0) *dst = v;
}

// buffer layout: [0, 1024) reduced sums (2j + 1 <= 1023), [1024, 1024 + G) norm partials,
// then one region of G * kLsPE block partials per pass-A group
constexpr int kLshSums = 1024;
long long lsh_part_elems(long long n, int maxj) {
  const long long G = reduce_blocks(n);
  return kLshSums + G + (long long)((maxj + kLsG) / kLsG + 1) * G * kLsPE;
}

int launch_mgs_lsh(cd* w, const cd* const* Vtab, const cd* const* Vhost, int j, long long n, cd* part, cd* Tg,
                   cd* hout, cudaStream_t st, const std::function<void(cd*, int)>& allreduce, const int* skip) {
  if (j > 511) return 1;
  const int G = reduce_blocks(n);
  // HDB_DEBUG_SYNC=1: synchronise after every kernel of the step and name a faulting one
  static const bool dbg = [] {
    const char* e = getenv("HDB_DEBUG_SYNC");
    return e && *e && *e != '0';
  }();
  auto chk = [&](const char* what, int q) {
    if (!dbg) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
      fprintf(stderr, "lsh fault after %s (group %d): j=%d n=%lld G=%d w=%p part=%p Tg=%p hout=%p: %s\n", what, q, j, n, G,
              (void*)w, (void*)part, (void*)Tg, (void*)hout, cudaGetErrorString(e));
  };
  cd* sums = part;
  cd* npart = part + kLshSums;
  cd* apart = npart + G;
  // pass A (the first group also carries <V_j, w>; with j = 0 it carries only that)
  const int ga = j == 0 ? 1 : (j + kLsG - 1) / kLsG;
  for (int q = 0; q < ga; ++q) {
    const int k0 = q * kLsG, kn = j - k0 < kLsG ? j - k0 : kLsG;
    k_lsh_a<<<G, kReduceThreads, 0, st>>>(w, Vhost[j], Vtab, k0, kn > 0 ? kn : 0, q == 0, n,
                                          apart + (long long)q * G * kLsPE, skip);
    chk("k_lsh_a", q);
  }
  k_lsh_sum<<<1, kLshF, 0, st>>>(apart, G, j, sums, skip);
  chk("k_lsh_sum", 0);
  if (allreduce) allreduce(sums, 2 * j + 1);
  chk("allreduce(sums)", 0);
  k_lsh_th<<<1, kLshF, 0, st>>>(sums, j, Tg, hout, skip);
  chk("k_lsh_th", 0);
  const int gb = (j + 1 + kLsG - 1) / kLsG;
  for (int q = 0; q < gb; ++q) {
    const int kfirst = j - q * kLsG, kn = kfirst + 1 < kLsG ? kfirst + 1 : kLsG;
    k_lsh_b<<<G, kReduceThreads, 0, st>>>(w, Vtab, hout, kfirst, kn, q == gb - 1, n, npart, skip);
    chk("k_lsh_b", q);
  }
  k_lsh_norm<<<1, kReduceThreads, 0, st>>>(npart, G, hout + j + 1, skip);
  chk("k_lsh_norm", 0);
  if (allreduce) allreduce(hout + j + 1, 1);
  return 0;
}

// ---------------------------------------------------------------------------
// Rank-count-invariant reductions (parallel.py:168-195: reduce_dot is bitwise
// invariant to the worker count).  One block per grid ROW forms that row's
// partial with a fixed in-row order (thread-strided sums, then the block tree:
// a function of nx only); the row partials of ALL ranks are then gathered in
// global row order and summed by k_rowsum in a fixed order (a function of the
// global row count only).  A slab decomposition cuts between rows, so every
// rank count -- one GPU included -- produces the same bits.
// op 0: <u, v>;  op 1: the fused MGS step of k_mgs (w -= h vi, then <vn, w>);
// op 2: ||b - t||^2.
template <int OP>
__global__ void __launch_bounds__(kReduceThreads) k_rowred(cd* __restrict__ w, const cd* __restrict__ a,
                                                           const cd* hsrc, const cd* __restrict__ c, int nx,
                                                           cd* __restrict__ rowpart) {
  const long long base = (long long)blockIdx.x * nx;
  const cd h = (OP == 1 && a) ? *hsrc : mkc(0.0, 0.0);
  cd acc = mkc(0.0, 0.0);
  for (int i = threadIdx.x; i < nx; i += kReduceThreads) {
    const long long p = base + i;
    if (OP == 0) {
      acc = c_conjmul_acc(acc, a[p], c[p]);
    } else if (OP == 1) {
      cd x = w[p];
      if (a) {
        x = c_sub(x, c_mul_np(h, a[p]));
        w[p] = x;
      }
      acc = c_conjmul_acc(acc, c ? c[p] : x, x);
    } else {
      const cd d = c_sub(a[p], c[p]);
      acc = c_conjmul_acc(acc, d, d);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) rowpart[blockIdx.x] = acc;
}

constexpr int kRowSumThreads = 1024;
__global__ void __launch_bounds__(kRowSumThreads) k_rowsum(const cd* __restrict__ rows, int nyg, cd* dst) {
  cd v = mkc(0.0, 0.0);
  for (int q = threadIdx.x; q < nyg; q += kRowSumThreads) {
    const cd z = rows[q];
    v.x += z.x;
    v.y += z.y;
  }
  v = block_sum<kRowSumThreads>(v);
  if (threadIdx.x == 0) *dst = v;
}

void launch_rowdot(const cd* u, const cd* v, int nx, int ny, cd* rowpart, cudaStream_t st) {
  k_rowred<0><<<ny, kReduceThreads, 0, st>>>(nullptr, u, nullptr, v, nx, rowpart);
}
void launch_rowmgs(cd* w, const cd* vi, const cd* hsrc, const cd* vn, int nx, int ny, cd* rowpart, cudaStream_t st) {
  k_rowred<1><<<ny, kReduceThreads, 0, st>>>(w, vi, hsrc, vn, nx, rowpart);
}
void launch_rowsubnorm(const cd* b, const cd* t, int nx, int ny, cd* rowpart, cudaStream_t st) {
  k_rowred<2><<<ny, kReduceThreads, 0, st>>>(nullptr, b, nullptr, t, nx, rowpart);
}
void launch_rowsum(const cd* rows, int nyg, cd* dst, cudaStream_t st) {
  k_rowsum<<<1, kRowSumThreads, 0, st>>>(rows, nyg, dst);
}

void launch_dot(const cd* u, const cd* v, long long n, RedWS& ws, cd* dst, cudaStream_t st) {
  k_dot<<<reduce_blocks(n), kReduceThreads, 0, st>>>(u, v, n, ws.partials, ws.ticket, dst);
}
void launch_mgs(cd* w, const cd* vi, const cd* hsrc, const cd* vn, long long n, RedWS& ws, cd* dst, cudaStream_t st,
                const Step1Epi* epi) {
  const Step1Epi e = epi ? *epi : Step1Epi{nullptr, nullptr, nullptr, nullptr, nullptr};
  k_mgs<<<reduce_blocks(n), kReduceThreads, 0, st>>>(w, vi, hsrc, vn, n, ws.partials, ws.ticket, dst, e);
}
void launch_subnorm(const cd* b, const cd* t, long long n, RedWS& ws, cd* dst, cudaStream_t st, cd* guard) {
  k_subnorm<<<reduce_blocks(n), kReduceThreads, 0, st>>>(b, t, n, ws.partials, ws.ticket, dst, guard);
}
void launch_scale(const cd* x, cd* out, double inv, long long n, cudaStream_t st) {
  k_scale<<<ew_blocks(n), 256, 0, st>>>(x, out, inv, n);
}
void launch_lincomb(const cd* const* basis, const cd* y, int m, const cd* x0, cd* x, long long n, cudaStream_t st) {
  k_lincomb<<<ew_blocks(n), 256, 0, st>>>(basis, y, m, x0, x, n);
}
void launch_add(const cd* a, const cd* b, cd* out, long long n, int sub, cudaStream_t st) {
  k_add<<<ew_blocks(n), 256, 0, st>>>(a, b, out, n, sub);
}
void launch_axpy(const cd* y, cd a, const cd* x, cd* out, long long n, int sub, cudaStream_t st) {
  k_axpy<<<ew_blocks(n), 256, 0, st>>>(y, a, x, out, n, sub);
}
void launch_bicg_p(const cd* r, cd* p, const cd* v, cd beta, cd omega, long long n, cudaStream_t st) {
  k_bicg_p<<<ew_blocks(n), 256, 0, st>>>(r, p, v, beta, omega, n);
}
void launch_gemv(const cd* A, const cd* b, cd* x, int n, cudaStream_t st) {
  k_gemv<<<(n * 32 + 255) / 256, 256, 0, st>>>(A, b, x, n);
}
void launch_scale_dev(const cd* x, cd* out, const cd* nrm2, long long n, cudaStream_t st, const int* skip) {
  k_scale_dev<<<ew_blocks(n), 256, 0, st>>>(x, out, nrm2, n, skip);
}
void launch_step1(const cd* b2, const cd* h0, const cd* hn2, cd* y, int* its, cd* flag, cudaStream_t st) {
  k_step1<<<1, 1, 0, st>>>(b2, h0, hn2, y, its, flag);
}
void launch_finite_guard(const cd* v, cd* flag, cudaStream_t st) { k_finite_guard<<<1, 1, 0, st>>>(v, flag); }
__global__ void k_pack_im(cd* dst, const cd* src) { dst->y = src->x; }
void launch_pack_im(cd* dst, const cd* src, cudaStream_t st) { k_pack_im<<<1, 1, 0, st>>>(dst, src); }
void launch_guard(const cd* post2, const cd* bn2, const cd* r02, double guard, cd* flag, cudaStream_t st) {
  k_guard<<<1, 1, 0, st>>>(post2, bn2, r02, guard, flag);
}

}  // namespace hdb
