// Device-resident GMRES: a whole unrestarted GMRES solve (krylov.py:61-177
// with apply_M = None) — operator applies, modified Gram-Schmidt, Givens
// rotations, stopping test, least squares, solution update and the explicit
// final residual — in ONE launch.  Used for every CSLP-GMRES and MG-coarsest
// GMRES on levels that fit the resident working set.
//
// Why: in the launch-driven engine every MGS coefficient is a kernel launch
// and every Arnoldi step a host round trip for the Hessenberg column
// (measured 168 us per GMRES iteration on the 65^2 level of BASELINE config 2,
// profiles/).  Resident, a step costs one barrier + a deterministic reduction.
//
// Two synchronisation policies share the solver body:
//   ClusterSync  one thread-block cluster (<= 16 CTAs), partials through DSMEM,
//                barrier.cluster — small levels (<= ~70k points);
//   GridSync     cooperative launch over all SMs, partials through global
//                memory, grid barrier — mid-size levels (<= ~2M points).
// CTA r owns the flat point range [r*N/P, (r+1)*N/P); its slice of the Arnoldi
// vector w lives in shared memory for the whole solve; basis vectors live in
// global memory (L2-resident on small levels).  Reductions are deterministic
// (fixed warp/block tree, then the P CTA partials combined in rank order by
// every CTA, so all CTAs hold bit-identical scalars).  Stencil and vector
// arithmetic is the same as the launch path.
#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>

#include "kernels.h"
#include "stencil.cuh"

namespace cg = cooperative_groups;

namespace hdb {

constexpr int kRT = 512;        // threads per CTA
constexpr int kMaxCap = 400;    // iteration cap supported by the device solver

struct ResidentArgs {
  OpCoef c;
  Geom g;
  const double* ksq;
  const cd* b;
  cd* x;
  cd* basis;          // (cap + 1) vectors of n points
  cd* Rg;             // packed upper-triangular R (cap*(cap+1)/2) + y (cap), written by rank 0;
                      // then (cap+1)(cap+2)/2 rows of T = (I + L)^{-1} (ORTHO 3)
  cd* gpart;          // GridSync: 2 * nranks partials
  long long n;
  double tol;
  int cap;
  int* its_out;
  double* relres_out;
  cd* flag;           // .x = 2.0 on a non-finite value (NumericalError)
  long long* prof;    // optional: per-phase cycles of CTA 0 thread 0 (telemetry), may be null
  int tiled;          // stencil windows staged in shared memory
  int tile_elems;     // window elements (max over CTAs)
  int sbasis;         // 1: this CTA's basis slices also kept in shared memory (dots / updates read them)
  int sstride;        // their stride (points per CTA, rounded up)
  int rsm;            // 1: the packed R factor is also kept in shared memory (least squares reads it there)
};

// phase clock (CTA 0, thread 0) — only when A.prof != nullptr
#define PHASE(k)                                                   \
  do {                                                             \
    if (A.prof && rank == 0 && t == 0) {                           \
      const long long now_ = clock64();                            \
      A.prof[k] += now_ - tprev_;                                  \
      tprev_ = now_;                                               \
    }                                                              \
  } while (0)

constexpr int kVecCap = 402;     // CGS2 coefficient vectors (cap + 1), grid mode
constexpr int kGatherCap = 130;  // cluster all-gather vector length (DSMEM buffers)

typedef cd GatherBuf[2][16][kGatherCap];  // [buffer][source rank][element] (cluster mode only)

constexpr int kOnePhaseMax = 64;  // grid reductions of up to this many elements take one barrier

struct RSmem {
  uint64_t mbar[2];
  cd sub[kRT];                // one-barrier grid reduction: per-thread sub-sums
  cd coef[49];    // per-tap coefficients when this CTA's k^2 window is uniform
  int uniform;
  cd pv[kVecCap];             // this CTA's block partial vector
  cd hv[kVecCap];             // reduced vector (CGS2 coefficients)
  cd warp[kRT / 32];
  cd part[2];
  cd bcast[2];
  cd hcol[kMaxCap + 2];
  cd sn[kMaxCap];
  double cs[kMaxCap];
  cd g[kMaxCap + 2];
  int decision;
};

template <int R>
__device__ __forceinline__ cd op_point(const OpCoef& c, const Geom& g, const cd* u, const double* k, int gj, int i) {
  const long long p = (long long)(gj - g.row0) * g.nx + i;
  if (pinned(g, c, gj, i)) return u[p];
  if (R == 1) {
    return five_point(c.s, c.mc, k[p], u[p], upad(u, k, g, c, gj, i - 1), upad(u, k, g, c, gj, i + 1),
                      upad(u, k, g, c, gj - 1, i), upad(u, k, g, c, gj + 1, i));
  }
  constexpr int N = 2 * R + 1;
  cd acc = mkc(0.0, 0.0);
#pragma unroll 1
  for (int a = 0; a < N; ++a) {
#pragma unroll
    for (int bb = 0; bb < N; ++bb) {
      const int jj = gj + a - R, ii = i + bb - R;
      const double kp = kpad(k, g, c, jj, ii);
      const cd m = c.mass[a * N + bb];
      const cd coef = mkc(__dadd_rn(c.lap[a * N + bb], __dmul_rn(m.x, kp)), __dmul_rn(m.y, kp));
      acc = c_add(acc, c_mul(coef, upad(u, k, g, c, jj, ii)));
    }
  }
  return acc;
}

// Shared-memory stencil window of this CTA's rows: rows [rlo-R, rhi+R] x columns
// [-R, nx+R) of the ghost-closed field (upad) and of k^2 (kpad).  Taps then read
// shared memory only; the window is loaded with all loads in flight.
struct Tile {
  int rlo, rows, cols;  // first own global row, window rows / cols
};

template <int R>
__device__ __forceinline__ Tile make_tile(const Geom& g, long long p0, long long p1) {
  Tile T;
  T.rlo = (int)(p0 / g.nx) + g.row0;
  const int rhi = (int)((p1 - 1) / g.nx) + g.row0;
  T.rows = rhi - T.rlo + 1 + 2 * R;
  T.cols = g.nx + 2 * R;
  return T;
}

template <int R>
__device__ __forceinline__ void load_u_tile(cd* ut, const Tile& T, const cd* u, const double* k, const Geom& g,
                                            const OpCoef& c) {
  const int n = T.rows * T.cols;
#pragma unroll 4
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int tr = e / T.cols, tc = e - tr * T.cols;
    ut[e] = upad(u, k, g, c, T.rlo - R + tr, tc - R);
  }
}

template <int R>
__device__ __forceinline__ void load_k_tile(double* kt, const Tile& T, const double* k, const Geom& g,
                                            const OpCoef& c) {
  const int n = T.rows * T.cols;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int tr = e / T.cols, tc = e - tr * T.cols;
    kt[e] = kpad(k, g, c, T.rlo - R + tr, tc - R);
  }
}

// (A u) at global (gj, i) from the windows (same arithmetic as the launch kernels)
template <int R>
__device__ __forceinline__ cd op_point_tile(const OpCoef& c, const Geom& g, const Tile& T, const cd* ut,
                                            const double* kt, const cd* ucoef, int gj, int i) {
  const int tr = gj - T.rlo + R, tc = i + R;
  const cd* uc = ut + tr * T.cols + tc;
  if (pinned(g, c, gj, i)) return *uc;
  if (R == 1) {
    return five_point(c.s, c.mc, kt[tr * T.cols + tc], *uc, uc[-1], uc[1], uc[-T.cols], uc[T.cols]);
  }
  constexpr int N = 2 * R + 1;
  const cd* u0 = uc - R * T.cols - R;
  const double* k0 = kt + (tr - R) * T.cols + tc - R;
  cd acc = mkc(0.0, 0.0);
  if (ucoef) {  // uniform k^2 window: same rounded coefficients, formed once
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int bb = 0; bb < N; ++bb) acc = c_add(acc, c_mul(ucoef[a * N + bb], u0[a * T.cols + bb]));
    }
    return acc;
  }
#pragma unroll
  for (int a = 0; a < N; ++a) {
#pragma unroll
    for (int bb = 0; bb < N; ++bb) {
      const double kp = k0[a * T.cols + bb];
      const cd m = c.mass[a * N + bb];
      const cd coef = mkc(__dadd_rn(c.lap[a * N + bb], __dmul_rn(m.x, kp)), __dmul_rn(m.y, kp));
      acc = c_add(acc, c_mul(coef, u0[a * T.cols + bb]));
    }
  }
  return acc;
}

__device__ __forceinline__ cd warp_sum_c(cd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// block partial -> thread 0 (fixed tree)
__device__ __forceinline__ cd block_partial(cd v, RSmem& s) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum_c(v);
  if (lane == 0) s.warp[wid] = v;
  __syncthreads();
  cd t = mkc(0.0, 0.0);
  if (wid == 0) {
    t = lane < kRT / 32 ? s.warp[lane] : mkc(0.0, 0.0);
    t = warp_sum_c(t);
  }
  return t;  // valid in thread 0
}

// --- cluster reductions: push all-gather through DSMEM ----------------------
// Every CTA's thread 0 writes its block partial with st.async into slot
// [its rank] of every CTA's partial array and completes that CTA's mbarrier
// (16 bytes of transaction each); every thread then waits on its local
// mbarrier and sums the C slots in rank order.  No cluster barrier, no global
// fence: a step costs one DSMEM latency.  Buffers alternate; a buffer's
// mbarrier is re-armed right after its phase completes, which always precedes
// the next pushes into it (those need this CTA's partial of the step between).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.b32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void push_c16(uint32_t raddr, cd v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rbar) : "memory");
}

constexpr int kMaxCluster = 16;

struct ClusterSync {
  static constexpr bool kGather = true;
  static constexpr int kVecMax = kGatherCap;
  cg::cluster_group cl;
  uint32_t par[2];
  GatherBuf* gb = nullptr;  // in dynamic shared memory after RSmem
  __device__ ClusterSync() : cl(cg::this_cluster()) { par[0] = par[1] = 0; }
  __device__ int rank() const { return (int)cl.block_rank(); }
  __device__ int nranks() const { return (int)cl.num_blocks(); }
  __device__ void barrier() { cl.sync(); }
  __device__ void init(RSmem& s, void* gather_mem) {
    gb = reinterpret_cast<GatherBuf*>(gather_mem);
    if (threadIdx.x == 0) {
      mbar_init(&s.mbar[0], 1);
      mbar_init(&s.mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();  // every CTA's barriers exist before any push
  }
  // all-gather + ordered sum of the block partial vector s.pv[0..m) (written and
  // __syncthreads-visible); result in out[0..m) (smem), visible to all threads
  // on return.  Arming happens here: pushes that arrive earlier only drive the
  // transaction count negative while the local arrival is still pending.
  __device__ void gather_sum(RSmem& s, int m, cd* out, int& buf) {
    const int C = nranks(), me = rank(), b = buf;
    if (threadIdx.x == 0) mbar_arm(&s.mbar[b], 16u * (uint32_t)(C * m));
    for (int e = threadIdx.x; e < m * C; e += blockDim.x) {
      const int r = e / m, i = e % m;  // destination rank, element
      push_c16(mapa(smem_addr(&(*gb)[b][me][i]), r), s.pv[i], mapa(smem_addr(&s.mbar[b]), r));
    }
    mbar_wait(&s.mbar[b], par[b]);
    par[b] ^= 1u;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      cd q = mkc(0.0, 0.0);
      for (int r = 0; r < C; ++r) {
        q.x += (*gb)[b][r][i].x;
        q.y += (*gb)[b][r][i].y;
      }
      out[i] = q;
    }
    __syncthreads();
    buf ^= 1;
  }
  __device__ cd reduce(cd v, RSmem& s, int& buf, cd*) {
    const cd t = block_partial(v, s);
    if (threadIdx.x == 0) s.pv[0] = t;
    __syncthreads();
    gather_sum(s, 1, s.bcast, buf);
    return s.bcast[0];
  }
  __device__ void reduce_vec(RSmem& s, int m, cd* out, int& buf, cd*) { gather_sum(s, m, out, buf); }
};

constexpr int kGridRounds = 5;  // ceil(148 SMs / 32): partial loads per lane in the grid reductions
static_assert(32 * kGridRounds >= 148, "grid reductions assume <= 160 CTAs");

struct GridSync {
  static constexpr bool kGather = false;
  static constexpr int kVecMax = kVecCap;
  cg::grid_group gr;
  __device__ GridSync() : gr(cg::this_grid()) {}
  __device__ int rank() const { return (int)blockIdx.x; }
  __device__ int nranks() const { return (int)gridDim.x; }
  __device__ void barrier() { gr.sync(); }
  __device__ void init(RSmem&, void*) {}
  // s.pv[0..m) -> out[0..m), fixed rank order.  Two phases when m is large:
  // CTA i sums element i over the P partials (one column each), publishes it,
  // then every CTA reads the m sums; small m: every CTA sums everything itself.
  __device__ void reduce_vec(RSmem& s, int m, cd* out, int& buf, cd* gpart) {
    const int P = nranks();
    cd* col = gpart + (long long)buf * P * kVecCap;
    for (int i = threadIdx.x; i < m; i += blockDim.x) __stcg(&col[(long long)blockIdx.x * kVecCap + i], s.pv[i]);
    gr.sync();
    if (m <= 4) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        cd q = mkc(0.0, 0.0);
        for (int r = 0; r < P; ++r) {
          const cd z = __ldcg(&col[(long long)r * kVecCap + i]);
          q.x += z.x;
          q.y += z.y;
        }
        out[i] = q;
      }
    } else if (m <= kOnePhaseMax) {
      // one grid barrier: every CTA sums all P partials of every element itself.
      // Thread t takes element e = t % m over ranks gi, gi + G, ... (gi = t / m,
      // G = kRT / m groups), the G sub-sums are then added in group order --
      // the same fixed order in every CTA, so all CTAs hold identical sums.
      const int G = kRT / m, t = threadIdx.x, e = t % m, gi = t / m;
      cd q = mkc(0.0, 0.0);
      if (gi < G) {
        for (int r0 = gi; r0 < P; r0 += 8 * G) {  // 8 partial loads in flight, then summed in rank order
          cd z[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = r0 + u * G;
            z[u] = r < P ? __ldcg(&col[(long long)r * kVecCap + e]) : mkc(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            q.x += z[u].x;
            q.y += z[u].y;
          }
        }
      }
      s.sub[t] = q;
      __syncthreads();
      for (int i = t; i < m; i += blockDim.x) {
        cd a = mkc(0.0, 0.0);
        for (int g2 = 0; g2 < G; ++g2) {
          const cd z = s.sub[g2 * m + i];
          a.x += z.x;
          a.y += z.y;
        }
        out[i] = a;
      }
    } else {
      cd* sums = gpart + 2LL * P * kVecCap + (long long)buf * kVecCap;  // published element sums
      for (int i = blockIdx.x; i < m; i += P) {
        if (threadIdx.x < 32) {
          // all of this lane's partials in flight at once (P <= 32 * kGridRounds), then summed in rank order
          cd z[kGridRounds];
#pragma unroll
          for (int u = 0; u < kGridRounds; ++u) {
            const int r = threadIdx.x + 32 * u;
            z[u] = r < P ? __ldcg(&col[(long long)r * kVecCap + i]) : mkc(0.0, 0.0);
          }
          cd q = mkc(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < kGridRounds; ++u) {
            q.x += z[u].x;
            q.y += z[u].y;
          }
          q = warp_sum_c(q);
          if (threadIdx.x == 0) __stcg(&sums[i], q);
        }
      }
      gr.sync();
      for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = __ldcg(&sums[i]);
    }
    __syncthreads();
    buf ^= 1;
  }
  __device__ cd reduce(cd v, RSmem& s, int& buf, cd* gpart) {
    const cd t = block_partial(v, s);
    const int P = nranks();
    if (threadIdx.x == 0) __stcg(&gpart[((long long)buf * P + blockIdx.x) * kVecCap], t);
    gr.sync();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      cd z[kGridRounds];
#pragma unroll
      for (int u = 0; u < kGridRounds; ++u) {
        const int r = lane + 32 * u;
        z[u] = r < P ? __ldcg(&gpart[((long long)buf * P + r) * kVecCap]) : mkc(0.0, 0.0);
      }
      cd q = mkc(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < kGridRounds; ++u) {
        q.x += z[u].x;
        q.y += z[u].y;
      }
      q = warp_sum_c(q);
      if (lane == 0) s.bcast[buf] = q;
    }
    __syncthreads();
    const cd r = s.bcast[buf];
    buf ^= 1;
    return r;
  }
};

__device__ __forceinline__ double cabs_(cd z) { return hypot(z.x, z.y); }
__device__ __forceinline__ cd cmul_(cd a, cd b) { return mkc(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cd cdiv_(cd a, cd b) {
  if (b.y == 0.0) return mkc(a.x / b.x, a.y / b.x);
  const double d = b.x * b.x + b.y * b.y;
  return mkc((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// CGS pass: out = V[0..m)^H w (warp per basis vector over this CTA's points),
// then w -= V out.  Returns with out[] reduced cluster/grid-wide in s.hv.
// with_norm: element m of the reduction carries <w, w> of the incoming w.
// `ph(k)` marks sub-phases (telemetry): 6 after the local dots, 7 after the
// reduction, 8 after the update.
// vb: this CTA's slice of V_0 (global basis + p0, or the shared-memory copy), vs: the
// stride between consecutive basis slices
template <class Sync, class Ph>
__device__ void cgs_pass(Sync& sy, RSmem& s, cd* ws, const cd* vb, long long vs, int cnt, int m,
                         int& buf, cd* gpart, bool with_norm, Ph&& ph) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int mm = m + (with_norm ? 1 : 0);
  constexpr int NW = kRT / 32;
  // warp w takes vectors w and w + NW together (one latency round for both);
  // each dot keeps its lane-strided order and warp tree
  for (int i = wid; i < mm; i += 2 * NW) {
    const int i2 = i + NW;
    const bool two = i2 < mm;
    const cd* v1 = i < m ? vb + (long long)i * vs : ws;
    const cd* v2 = !two ? v1 : (i2 < m ? vb + (long long)i2 * vs : ws);
    cd a = mkc(0.0, 0.0), b2 = mkc(0.0, 0.0);
#pragma unroll 4
    for (int q = lane; q < cnt; q += 32) {
      const cd wq = ws[q];
      a = c_conjmul_acc(a, v1[q], wq);
      b2 = c_conjmul_acc(b2, v2[q], wq);
    }
    a = warp_sum_c(a);
    b2 = warp_sum_c(b2);
    if (lane == 0) {
      s.pv[i] = a;
      if (two) s.pv[i2] = b2;
    }
  }
  __syncthreads();
  ph(6);
  sy.reduce_vec(s, mm, s.hv, buf, gpart);
  ph(7);
  for (int q = threadIdx.x; q < cnt; q += kRT) {
    cd w = ws[q];
    const cd* vq = vb + q;
    int i = 0;
    for (; i + 8 <= m; i += 8) {  // 8 loads in flight, then the dependent updates in order
      cd v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = vq[(long long)(i + u) * vs];
#pragma unroll
      for (int u = 0; u < 8; ++u) w = c_sub(w, c_mul_np(s.hv[i + u], v[u]));
    }
    for (; i < m; ++i) w = c_sub(w, c_mul_np(s.hv[i], vq[(long long)i * vs]));
    ws[q] = w;
  }
  __syncthreads();
  ph(8);
}

// Low-synchronisation MGS (one-reduce MGS, the k_mgs_ls algorithm) on this CTA's
// slice: one reduction carries g = V^H w and the new row of L (<V_j, V_k>, k < j);
// every CTA forms the new row of T = (I + L)^{-1} (rank 0 stores it in Tg) and
// h = T g into s.hcol; then w -= h_k V_k (V_j first, then k = j-1 .. 0).  The caller
// forms ||w||^2 with one more reduction.
template <class Sync>
__device__ void ls_pass(Sync& sy, RSmem& s, cd* ws, const cd* vb, long long vs, int cnt, int j,
                        int& buf, cd* gpart, cd* Tg, int rank) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, t = threadIdx.x;
  constexpr int NW = kRT / 32;
  const cd* vj = vb + (long long)j * vs;
  for (int i = wid; i <= j; i += NW) {  // warp per basis vector: g_i and (i < j) l_i
    const cd* vi = vb + (long long)i * vs;
    cd a = mkc(0.0, 0.0), l = mkc(0.0, 0.0);
#pragma unroll 4
    for (int q = lane; q < cnt; q += 32) {
      const cd v = vi[q];
      a = c_conjmul_acc(a, v, ws[q]);
      if (i < j) l = c_conjmul_acc(l, vj[q], v);
    }
    a = warp_sum_c(a);
    l = warp_sum_c(l);
    if (lane == 0) {
      s.pv[i] = a;
      if (i < j) s.pv[j + 1 + i] = l;
    }
  }
  __syncthreads();
  sy.reduce_vec(s, 2 * j + 1, s.hv, buf, gpart);  // hv: g_0..g_j, l_0..l_{j-1}
  cd* trow = s.sub;
  const long long rj = (long long)j * (j + 1) / 2;
  for (int k = t; k < j; k += kRT) {  // t_jk = -sum_{m=k}^{j-1} l_m T_mk
    cd a = mkc(0.0, 0.0);
    for (int m0 = k; m0 < j; m0 += 8) {
      cd tm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tm[u] = m0 + u < j ? __ldcg(&Tg[(long long)(m0 + u) * (m0 + u + 1) / 2 + k]) : mkc(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (m0 + u < j) {
          const cd lm = s.hv[j + 1 + m0 + u];
          a.x = __fma_rn(lm.x, tm[u].x, a.x); a.x = __fma_rn(-lm.y, tm[u].y, a.x);
          a.y = __fma_rn(lm.x, tm[u].y, a.y); a.y = __fma_rn(lm.y, tm[u].x, a.y);
        }
      }
    }
    trow[k] = mkc(-a.x, -a.y);
    if (rank == 0) Tg[rj + k] = trow[k];
  }
  if (rank == 0 && t == 0) Tg[rj + j] = mkc(1.0, 0.0);
  __syncthreads();
  for (int i = t; i <= j; i += kRT) {  // h_i = sum_{k <= i} T_ik g_k
    cd a = mkc(0.0, 0.0);
    const long long ri = (long long)i * (i + 1) / 2;
    for (int k0 = 0; k0 <= i; k0 += 8) {
      cd tk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        tk[u] = k > i ? mkc(0.0, 0.0) : (i < j ? (k < i ? __ldcg(&Tg[ri + k]) : mkc(1.0, 0.0))
                                                : (k < j ? trow[k] : mkc(1.0, 0.0)));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (k0 + u <= i) {
          const cd gk = s.hv[k0 + u];
          a.x = __fma_rn(tk[u].x, gk.x, a.x); a.x = __fma_rn(-tk[u].y, gk.y, a.x);
          a.y = __fma_rn(tk[u].x, gk.y, a.y); a.y = __fma_rn(tk[u].y, gk.x, a.y);
        }
      }
    }
    s.hcol[i] = a;
  }
  __syncthreads();
  for (int q = t; q < cnt; q += kRT) {  // w -= h_j V_j, then h_k V_k for k = j-1 .. 0
    cd w = ws[q];
    const cd* vq = vb + q;
    int i = j;
    for (; i >= 7; i -= 8) {  // 8 loads in flight, then the dependent updates in order
      cd v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = vq[(long long)(i - u) * vs];
#pragma unroll
      for (int u = 0; u < 8; ++u) w = c_sub(w, c_mul_np(s.hcol[i - u], v[u]));
    }
    for (; i >= 0; --i) w = c_sub(w, c_mul_np(s.hcol[i], vq[(long long)i * vs]));
    ws[q] = w;
  }
  __syncthreads();
}

template <class Sync, int R, int ORTHO>
__global__ void __launch_bounds__(kRT) k_resident_gmres(ResidentArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RSmem& s = *reinterpret_cast<RSmem*>(smem_raw);
  constexpr size_t kHead = ((sizeof(RSmem) + 15) / 16) * 16 + (Sync::kGather ? sizeof(GatherBuf) : 0);
  Sync sy;
  sy.init(s, smem_raw + ((sizeof(RSmem) + 15) / 16) * 16);
  const int P = sy.nranks(), rank = sy.rank();
  const long long n = A.n;
  const long long p0 = n * rank / P, p1 = n * (rank + 1) / P;
  const int cnt = (int)(p1 - p0);
  const long long chunk_max = (n + P - 1) / P;
  cd* ws = reinterpret_cast<cd*>(smem_raw + kHead);  // this CTA's slice of w
  const Tile T = make_tile<R>(A.g, p0, p1);
  cd* ut = A.tiled ? ws + chunk_max : nullptr;                 // stencil window of the current vector
  double* kt = A.tiled ? reinterpret_cast<double*>(ut + A.tile_elems) : nullptr;  // k^2 window (constant)
  // optional shared-memory copy of this CTA's basis slices (after the windows, 16-B aligned)
  cd* sb = nullptr;
  if (A.sbasis) {
    const size_t off = ((size_t)(reinterpret_cast<unsigned char*>(kt + A.tile_elems) - smem_raw) + 15) / 16 * 16;
    sb = reinterpret_cast<cd*>(smem_raw + off);
  }
  // optional shared-memory copy of the packed R factor (after the basis slices / windows):
  // the back substitution's dependent chain then reads shared memory instead of L2
  cd* Rs = nullptr;
  if (A.rsm) {
    const unsigned char* end = sb ? reinterpret_cast<unsigned char*>(sb + (size_t)(A.cap + 1) * A.sstride)
                                  : reinterpret_cast<unsigned char*>(kt + A.tile_elems);
    Rs = reinterpret_cast<cd*>(smem_raw + ((size_t)(end - smem_raw) + 15) / 16 * 16);
  }
  if (A.tiled && cnt > 0) load_k_tile<R>(kt, T, A.ksq, A.g, A.c);
  const cd* ucoef = nullptr;
  if (A.tiled && R > 1) {
    if (threadIdx.x == 0) s.uniform = cnt > 0;
    __syncthreads();
    const int ne = T.rows * T.cols;
    const double k00 = cnt > 0 ? kt[0] : 0.0;
    for (int e = threadIdx.x; e < ne; e += kRT)
      if (kt[e] != k00) s.uniform = 0;
    __syncthreads();
    if (s.uniform) {
      constexpr int NN = (2 * R + 1) * (2 * R + 1);
      if (threadIdx.x < NN) {
        const cd m = A.c.mass[threadIdx.x];
        s.coef[threadIdx.x] = mkc(__dadd_rn(A.c.lap[threadIdx.x], __dmul_rn(m.x, k00)), __dmul_rn(m.y, k00));
      }
      ucoef = s.coef;
    }
    __syncthreads();
  }
  const int t = threadIdx.x;
  const int nx = A.g.nx;
  int buf = 0;
  auto V = [&](int i) { return A.basis + (long long)i * n; };
  const cd* vb = sb ? sb : A.basis + p0;      // this CTA's slice of V_0
  const long long vs = sb ? A.sstride : n;    // stride between basis slices
  cd* Rg = A.Rg;
  cd* yg = A.Rg + (long long)A.cap * (A.cap + 1) / 2;

  cd acc = mkc(0.0, 0.0);
  for (int q = t; q < cnt; q += kRT) { const cd v = A.b[p0 + q]; acc = c_conjmul_acc(acc, v, v); }
  const double bnorm = sqrt(fmax(sy.reduce(acc, s, buf, A.gpart).x, 0.0));
  if (bnorm == 0.0) {  // krylov.py:96-97
    for (int q = t; q < cnt; q += kRT) A.x[p0 + q] = mkc(0.0, 0.0);
    if (rank == 0 && t == 0) { *A.its_out = 0; *A.relres_out = 0.0; }
    sy.barrier();
    return;
  }
  if (!isfinite(bnorm)) {
    if (rank == 0 && t == 0) { A.flag->x = 2.0; *A.its_out = 0; }
    sy.barrier();
    return;
  }
  const double beta = bnorm;  // r0 = b (zero initial guess); rel = 1 never triggers the early exit
  {
    const double inv = 1.0 / beta;
    cd* v0 = V(0);
    for (int q = t; q < cnt; q += kRT) {
      const cd v = A.b[p0 + q];
      v0[p0 + q] = mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv));
      if (sb) sb[q] = v0[p0 + q];
    }
  }
  if (t == 0) s.g[0] = mkc(beta, 0.0);
  int its = 0;
  long long tprev_ = clock64();
  auto ph = [&](int k) { PHASE(k); };
  // ws = M V_j for this CTA's points (stencil from the shared-memory windows).
  // `givens_j` >= 0: thread 0 first applies the rotations of step givens_j,
  // overlapping that serial work with everybody else's stencil points.
  auto apply_M = [&](int jv, int givens_j, double hn_prev) {
    const cd* vj = V(jv);
    if (A.tiled) {
      if (cnt > 0) load_u_tile<R>(ut, T, vj, A.ksq, A.g, A.c);
      __syncthreads();
    }
    PHASE(9);
    if (givens_j >= 0 && t == kRT - 1) {
      // rotations (krylov.py:126-151), identical in every CTA.  Run by the LAST
      // thread: on small levels its warp owns no stencil points, so this serial
      // work overlaps the other warps' stencil instead of delaying warp 0.  The
      // rotated entry is carried in registers (no shared-memory round trip on
      // the dependency chain); same operations in the same order as before.
      const int j = givens_j;
      const double hn = hn_prev;
      cd* col = s.hcol;
      col[j + 1] = mkc(hn, 0.0);
      cd cur = col[0];
      bool finite = isfinite(cur.x) && isfinite(cur.y) && isfinite(hn);
#pragma unroll 4
      for (int i = 0; i < j; ++i) {
        const cd nxt = col[i + 1];
        const double csi = s.cs[i];
        const cd sni = s.sn[i];
        finite &= isfinite(nxt.x) && isfinite(nxt.y);
        const cd sc = cmul_(sni, nxt);
        const cd tt = mkc(csi * cur.x + sc.x, csi * cur.y + sc.y);
        const cd nb = cmul_(mkc(-sni.x, sni.y), cur);
        cur = mkc(nb.x + csi * nxt.x, nb.y + csi * nxt.y);
        col[i] = tt;
      }
      col[j] = cur;
      const cd h1 = col[j], h2 = col[j + 1];
      double c;
      cd sn;
      const double a1 = cabs_(h1), a2 = cabs_(h2);
      if (a2 == 0.0) { c = 1.0; sn = mkc(0.0, 0.0); }
      else if (a1 == 0.0) { c = 0.0; sn = mkc(1.0, 0.0); }
      else {
        const double tt = hypot(a1, a2);
        c = a1 / tt;
        const cd q = cmul_(mkc(h1.x / a1, h1.y / a1), mkc(h2.x, -h2.y));
        sn = mkc(q.x / tt, q.y / tt);
      }
      s.cs[j] = c;
      s.sn[j] = sn;
      const cd sh = cmul_(sn, h2);
      col[j] = mkc(c * h1.x + sh.x, c * h1.y + sh.y);
      if (rank == 0) {
        cd* Rc = (Rs ? Rs : Rg) + (long long)j * (j + 1) / 2;
        for (int i = 0; i <= j; ++i) Rc[i] = col[i];
      }
      const cd gj = s.g[j];
      s.g[j + 1] = cmul_(mkc(-sn.x, sn.y), gj);
      s.g[j] = mkc(c * gj.x, c * gj.y);
      const double rel = cabs_(s.g[j + 1]) / bnorm;
      s.decision = !finite ? 2 : ((hn < 1e-30 || rel <= A.tol) ? 1 : 0);
    }
    PHASE(10);
    if (jv < A.cap) {  // the stencil of step jv (skipped past the cap)
      for (int q = t; q < cnt; q += kRT) {
        const long long p = p0 + q;
        const int gj = (int)(p / nx) + A.g.row0, i = (int)(p % nx);
        ws[q] = A.tiled ? op_point_tile<R>(A.c, A.g, T, ut, kt, ucoef, gj, i)
                        : op_point<R>(A.c, A.g, vj, A.ksq, gj, i);
      }
    }
    __syncthreads();
  };
  sy.barrier();  // V_0 complete everywhere
  apply_M(0, -1, 0.0);
  PHASE(1);
  int dec = 0;
  for (int j = 0; j < A.cap; ++j) {
    if (ORTHO == 0) {
      // modified Gram-Schmidt (krylov.py:121-124): h_i = <V_i, w>; w -= h_i V_i
      for (int i = 0; i <= j; ++i) {
        const cd* vi = vb + (long long)i * vs;
        cd a = mkc(0.0, 0.0);
        for (int q = t; q < cnt; q += kRT) a = c_conjmul_acc(a, vi[q], ws[q]);
        const cd h = sy.reduce(a, s, buf, A.gpart);
        if (t == 0) s.hcol[i] = h;
        for (int q = t; q < cnt; q += kRT) ws[q] = c_sub(ws[q], c_mul_np(h, vi[q]));
      }
    } else if (ORTHO == 3) {
      __syncthreads();
      ls_pass(sy, s, ws, vb, vs, cnt, j, buf, A.gpart, Rg + (long long)A.cap * (A.cap + 1) / 2 + A.cap, rank);
    } else if (ORTHO == 1) {
      // classical Gram-Schmidt with one re-orthogonalisation (CGS2): the same
      // Hessenberg column in exact arithmetic, two reductions instead of j+1
      __syncthreads();
      cgs_pass(sy, s, ws, vb, vs, cnt, j + 1, buf, A.gpart, false, ph);
      for (int i = t; i <= j; i += kRT) s.hcol[i] = s.hv[i];
      __syncthreads();
      cgs_pass(sy, s, ws, vb, vs, cnt, j + 1, buf, A.gpart, false, ph);
      for (int i = t; i <= j; i += kRT) s.hcol[i] = c_add(s.hcol[i], s.hv[i]);
      __syncthreads();
    }
    double hn;
    if (ORTHO == 2) {
      // CGS with DGKS re-orthogonalisation: one reduction carries V^H w and
      // <w, w>; ||w'||^2 = <w, w> - sum |h_i|^2 (Pythagoras, V orthonormal).
      // Only when that drops below half of <w, w> (cancellation: w close to
      // span V) is a second pass made, whose reduction carries <w', w'> and
      // the (tiny) corrections.  Same Hessenberg column in exact arithmetic;
      // every CTA takes the same branch (identically reduced scalars).
      __syncthreads();
      cgs_pass(sy, s, ws, vb, vs, cnt, j + 1, buf, A.gpart, true, ph);
      double nw = s.hv[j + 1].x, sh = 0.0;
      for (int i = 0; i <= j; ++i) sh += s.hv[i].x * s.hv[i].x + s.hv[i].y * s.hv[i].y;
      __syncthreads();
      for (int i = t; i <= j; i += kRT) s.hcol[i] = s.hv[i];
      double est = nw - sh;
      if (!(est > 0.5 * nw)) {
        __syncthreads();
        cgs_pass(sy, s, ws, vb, vs, cnt, j + 1, buf, A.gpart, true, ph);
        nw = s.hv[j + 1].x;
        sh = 0.0;
        for (int i = 0; i <= j; ++i) sh += s.hv[i].x * s.hv[i].x + s.hv[i].y * s.hv[i].y;
        __syncthreads();
        for (int i = t; i <= j; i += kRT) s.hcol[i] = c_add(s.hcol[i], s.hv[i]);
        est = nw - sh;
      }
      __syncthreads();
      PHASE(2);
      hn = sqrt(fmax(est, 0.0));
    } else {
      PHASE(2);
      cd a = mkc(0.0, 0.0);
      for (int q = t; q < cnt; q += kRT) a = c_conjmul_acc(a, ws[q], ws[q]);
      hn = sqrt(fmax(sy.reduce(a, s, buf, A.gpart).x, 0.0));
    }
    PHASE(3);
    // V_{j+1} = w / ||w|| (harmless if step j turns out to be the last)
    const double inv = 1.0 / hn;
    cd* vn = V(j + 1) + p0;
    cd* sn1 = sb ? sb + (long long)(j + 1) * vs : nullptr;
    for (int q = t; q < cnt; q += kRT) {
      const cd v = ws[q];
      const cd u = mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv));
      vn[q] = u;
      if (sn1) sn1[q] = u;
    }
    sy.barrier();  // V_{j+1} complete everywhere
    PHASE(5);
    // Givens of step j on thread 0 while the stencil of step j+1 runs
    apply_M(j + 1, j, hn);
    PHASE(4);
    its = j + 1;
    dec = s.decision;
    if (dec != 0) break;
  }
  if (dec == 2) {
    if (rank == 0 && t == 0) { A.flag->x = 2.0; *A.its_out = its; }
    sy.barrier();
    return;
  }
  // least squares (krylov.py:161-168) on rank 0, y broadcast through global memory
  if (rank == 0 && t == 0) {
    if (Rs) {  // R and y in shared memory (s.pv is free here): same operations in the same order
      cd* ys = s.pv;
      const bool ysh = its <= kVecCap;
      for (int i = its - 1; i >= 0; --i) {
        cd accy = s.g[i];
        for (int k = i + 1; k < its; ++k) {
          const cd pr = cmul_(Rs[(long long)k * (k + 1) / 2 + i], ysh ? ys[k] : yg[k]);
          accy = mkc(accy.x - pr.x, accy.y - pr.y);
        }
        const cd yi = cdiv_(accy, Rs[(long long)i * (i + 1) / 2 + i]);
        if (ysh) ys[i] = yi;
        yg[i] = yi;
      }
    } else {
      for (int i = its - 1; i >= 0; --i) {
        cd accy = s.g[i];
        for (int k = i + 1; k < its; ++k) {
          const cd pr = cmul_(Rg[(long long)k * (k + 1) / 2 + i], yg[k]);
          accy = mkc(accy.x - pr.x, accy.y - pr.y);
        }
        yg[i] = cdiv_(accy, Rg[(long long)i * (i + 1) / 2 + i]);
      }
    }
  }
  sy.barrier();
  const bool ysm = its <= kVecCap;
  if (ysm)
    for (int i = t; i < its; i += kRT) s.hv[i] = __ldcg(&yg[i]);
  __syncthreads();
  const cd* yc = ysm ? s.hv : yg;
  for (int q = t; q < cnt; q += kRT) {
    cd xx = mkc(0.0, 0.0);
    const cd* vq = vb + q;
    int i = 0;
    for (; i + 8 <= its; i += 8) {
      cd v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = vq[(long long)(i + u) * vs];
#pragma unroll
      for (int u = 0; u < 8; ++u) xx = c_add(xx, c_mul_np(yc[i + u], v[u]));
    }
    for (; i < its; ++i) xx = c_add(xx, c_mul_np(yc[i], vq[(long long)i * vs]));
    A.x[p0 + q] = xx;
  }
  sy.barrier();  // x complete everywhere
  // explicit true residual (krylov.py:174)
  cd f = mkc(0.0, 0.0);
  if (A.tiled) {
    if (cnt > 0) load_u_tile<R>(ut, T, A.x, A.ksq, A.g, A.c);
    __syncthreads();
  }
  for (int q = t; q < cnt; q += kRT) {
    const long long p = p0 + q;
    const int gj = (int)(p / nx) + A.g.row0, i = (int)(p % nx);
    const cd ax = A.tiled ? op_point_tile<R>(A.c, A.g, T, ut, kt, ucoef, gj, i) : op_point<R>(A.c, A.g, A.x, A.ksq, gj, i);
    const cd d = c_sub(A.b[p], ax);
    f = c_conjmul_acc(f, d, d);
  }
  const double fin = sqrt(fmax(sy.reduce(f, s, buf, A.gpart).x, 0.0)) / bnorm;
  if (rank == 0 && t == 0) {
    *A.its_out = its;
    *A.relres_out = fin;
    if (!isfinite(fin)) A.flag->x = 2.0;
  }
  sy.barrier();  // no CTA leaves while a peer may still address its shared memory
}

// ------------------------------------------------------------------ launch
static size_t smem_head(bool cluster) {
  return ((sizeof(RSmem) + 15) / 16) * 16 + (cluster ? sizeof(GatherBuf) : 0);
}
static size_t smem_for(long long chunk, bool cluster) { return smem_head(cluster) + (size_t)chunk * sizeof(cd); }

// largest stencil window over the P CTAs (rows x (nx + 2R))
static int tile_elems_for(long long n, int nx, int P, int R) {
  long long best = 0;
  for (int r = 0; r < P; ++r) {
    const long long p0 = n * r / P, p1 = n * (r + 1) / P;
    if (p1 <= p0) continue;
    const long long rows = (p1 - 1) / nx - p0 / nx + 1 + 2 * R;
    best = std::max(best, rows * (nx + 2 * R));
  }
  return (int)best;
}

static size_t smem_tiled(long long chunk, int tile, bool cluster) {
  return smem_for(chunk, cluster) + (size_t)tile * (sizeof(cd) + sizeof(double));
}

// add the shared-memory basis slices ((cap + 1) x chunk points) when they fit beside the
// windows (HDB_RES_SBASIS=0 disables): the dots and updates then read shared memory
static size_t with_sbasis(ResidentArgs& a, size_t sm, long long chunk, size_t limit) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HDB_RES_SBASIS");
    on = e ? atoi(e) : 1;
  }
  a.sbasis = 0;
  a.sstride = (int)chunk;
  const size_t extra = 16 + (size_t)(a.cap + 1) * (size_t)chunk * sizeof(cd);
  if (on && sm + extra <= limit) {
    a.sbasis = 1;
    return sm + extra;
  }
  return sm;
}

// add the shared-memory R factor (cap (cap + 1) / 2 entries) when it fits (HDB_RES_RSM=0 disables)
static size_t with_rsm(ResidentArgs& a, size_t sm, size_t limit) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("HDB_RES_RSM");
    on = e ? atoi(e) : 1;
  }
  a.rsm = 0;
  const size_t extra = 16 + (size_t)a.cap * (a.cap + 1) / 2 * sizeof(cd);
  if (on && sm + extra <= limit) {
    a.rsm = 1;
    return sm + extra;
  }
  return sm;
}

static int g_cluster = 0;
static long long* g_prof = nullptr;  // set by resident_set_profile (telemetry)

void resident_set_profile(long long* dev_counters) { g_prof = dev_counters; }
static int g_grid = 0;
static size_t g_smem_optin = 0;

// device limits, read once per process (every rank thread of a process uses the
// same device model); std::call_once makes the first use thread-safe
static std::once_flag g_limits_once;
static void init_limits() {
  std::call_once(g_limits_once, [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_grid = v > 32 * kGridRounds ? 32 * kGridRounds : v;  // reductions batch <= 32 * kGridRounds partials
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    g_smem_optin = (size_t)v;
  });
}

template <class K>
static void set_attrs(K kern, size_t sm, bool cluster) {
  ensure_smem_attr((const void*)kern, sm);
  if (cluster) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

template <int R, int O>
static bool launch_cluster(const ResidentArgs& a, cudaStream_t st) {
  auto kern = k_resident_gmres<ClusterSync, R, O>;
  if (g_cluster == 0) {
    const size_t sm0 = smem_for(4096, true);
    set_attrs(kern, sm0, true);
    for (int c : {16, 8, 4}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(c); cfg.blockDim = dim3(kRT); cfg.dynamicSmemBytes = sm0; cfg.attrs = at; cfg.numAttrs = 1;
      int num = 0;
      if (cudaOccupancyMaxActiveClusters(&num, kern, &cfg) == cudaSuccess && num > 0) { g_cluster = c; break; }
      cudaGetLastError();
    }
    if (g_cluster == 0) g_cluster = -1;
  }
  if (g_cluster < 0) return false;
  const long long chunk = (a.n + g_cluster - 1) / g_cluster;
  ResidentArgs b = a;
  b.tile_elems = tile_elems_for(a.n, a.g.nx, g_cluster, R);
  size_t sm = smem_tiled(chunk, b.tile_elems, true);
  b.tiled = sm <= g_smem_optin;
  if (!b.tiled) return false;  // untiled resident solves lose to the launch path
  sm = with_sbasis(b, sm, chunk, g_smem_optin);
  sm = with_rsm(b, sm, g_smem_optin);
  set_attrs(kern, sm, true);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g_cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(g_cluster);
  cfg.blockDim = dim3(kRT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, b) == cudaSuccess;
}

// CTAs of a grid-mode resident solve: all SMs by default; HDB_RES_GRID_PTS=p caps
// the grid at one CTA per p points (fewer CTAs: cheaper barriers and reductions)
static int grid_ctas_for(long long n) {
  static long long per = -1;
  if (per < 0) {
    const char* e = getenv("HDB_RES_GRID_PTS");
    per = e ? atoll(e) : 0;
  }
  if (per <= 0) return g_grid;
  const long long p = (n + per - 1) / per;
  return (int)std::max(16LL, std::min<long long>(g_grid, p));
}

template <int R, int O>
static bool launch_grid(ResidentArgs a, cudaStream_t st) {
  auto kern = k_resident_gmres<GridSync, R, O>;
  const int P = grid_ctas_for(a.n);
  const long long chunk = (a.n + P - 1) / P;
  a.tile_elems = tile_elems_for(a.n, a.g.nx, P, R);
  size_t sm = smem_tiled(chunk, a.tile_elems, false);
  a.tiled = sm <= g_smem_optin;
  if (!a.tiled) return false;  // untiled resident solves lose to the launch path
  sm = with_sbasis(a, sm, chunk, g_smem_optin);
  sm = with_rsm(a, sm, g_smem_optin);
  set_attrs(kern, sm, false);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRT, sm) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return false;
  }
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)kern, dim3(P), dim3(kRT), args, sm, st) == cudaSuccess;
}

int resident_max_cap() { return kMaxCap; }

long long mgs_global_tier_bytes() {
  static long long v = -1;
  if (v < 0) {
    const char* e = getenv("HDB_MGS_L2_BYTES");
    v = e ? atoll(e) : 80LL << 20;  // w up to 80 MB rides in the 126 MB L2
  }
  return v;
}
int resident_vec_cap() { return kVecCap - 1; }  // gpart stride - 1
// SmallSolve::gpart size: two buffers of per-CTA partial vectors plus the published sums
long long resident_gpart_elems() { return 2LL * resident_grid_ctas() * kVecCap + 2LL * kVecCap; }

long long resident_cluster_points() {
  init_limits();
  const size_t room = g_smem_optin > smem_for(0, true) ? g_smem_optin - smem_for(0, true) : 0;
  return (long long)(room / sizeof(cd)) * 16;
}
long long resident_grid_points() {
  init_limits();
  const size_t room = g_smem_optin > smem_for(0, false) ? g_smem_optin - smem_for(0, false) : 0;
  return (long long)(room / sizeof(cd)) * g_grid;
}

// returns 0 on success, 1 if the problem does not fit a resident launch
template <int O>
static bool launch_any(int mode, const ResidentArgs& a, int radius, cudaStream_t st) {
  if (mode == 0)
    return radius == 1 ? launch_cluster<1, O>(a, st) : radius == 2 ? launch_cluster<2, O>(a, st)
                                                                    : launch_cluster<3, O>(a, st);
  return radius == 1 ? launch_grid<1, O>(a, st) : radius == 2 ? launch_grid<2, O>(a, st) : launch_grid<3, O>(a, st);
}

int launch_resident_gmres(int mode, int ortho, const OpCoef& c, const Geom& g, const double* ksq, const cd* b, cd* x,
                          cd* basis, cd* Rg, cd* gpart, long long n, double tol, int cap, int* its_out,
                          double* relres_out, cd* flag, cudaStream_t st) {
  init_limits();
  ResidentArgs a{};
  a.c = c; a.g = g; a.ksq = ksq; a.b = b; a.x = x; a.basis = basis; a.Rg = Rg; a.gpart = gpart; a.n = n;
  a.tol = tol; a.cap = cap; a.its_out = its_out; a.relres_out = relres_out; a.flag = flag; a.prof = g_prof;
  if (ortho == 4) ortho = n >= 131072 ? 3 : 2;  // auto
  if (ortho == 1 && cap + 1 > (mode == 0 ? kGatherCap : kVecCap)) ortho = 0;
  if (ortho == 3 && 2 * cap + 1 > (mode == 0 ? kGatherCap : kVecCap)) ortho = 2;
  if (ortho == 2 && cap + 2 > (mode == 0 ? kGatherCap : kVecCap)) ortho = 0;
  const bool ok = ortho == 3   ? launch_any<3>(mode, a, c.radius, st)
                  : ortho == 2 ? launch_any<2>(mode, a, c.radius, st)
                  : ortho == 1 ? launch_any<1>(mode, a, c.radius, st) : launch_any<0>(mode, a, c.radius, st);
  return ok ? 0 : 1;
}

int resident_grid_ctas() {
  init_limits();
  return g_grid;
}

}  // namespace hdb

namespace hdb {

// ---------------------------------------------------------------------------
// One Arnoldi step's modified Gram-Schmidt for large levels (the launch-driven
// engine's MGS chain in ONE cooperative launch): w (= A z, global) is held in
// shared memory across the chain; each step reads V_i once (the thread keeps
// its V_i values in registers between the dot and the update) and does one
// deterministic grid reduction.  Writes h_i to hout[i], ||w||^2 to hout[j+1].x
// and, as the launch path does after the host's stopping test, V_{j+1} =
// w * (1/||w||) into w's buffer (harmless when the step converges).
// Same arithmetic as k_mgs (krylov.py:121-124).
// Bulk L2 prefetch of [p, p + n) (TMA engine, no registers or shared memory):
// issued for V_{i+1} at the top of MGS step i, its HBM read overlaps step i's
// dot product and grid reduction.  Threads 0..k each issue one 64 KB piece.
__device__ __forceinline__ void prefetch_l2_span(const cd* p, long long n) {
  constexpr long long kPiece = 4096;  // elements (64 KB)
  const long long pieces = (n + kPiece - 1) / kPiece;
  for (long long k = threadIdx.x; k < pieces; k += blockDim.x) {
    const long long e0 = k * kPiece, ne = n - e0 < kPiece ? n - e0 : kPiece;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + e0), "r"((unsigned)(ne * sizeof(cd)))
                 : "memory");
  }
}

// w slice -> shared memory with 16 loads in flight per thread
__device__ __forceinline__ void load_slice_smem(cd* dst, const cd* src, int cnt) {
  for (int base = threadIdx.x; base < cnt; base += 16 * kRT) {
    cd r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int q = base + k * kRT;
      r[k] = q < cnt ? src[q] : mkc(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int q = base + k * kRT;
      if (q < cnt) dst[q] = r[k];
    }
  }
}

// 16-byte load with an L2 eviction-priority hint (createpolicy handle)
__device__ __forceinline__ uint64_t l2pol_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2pol_drop() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ cd ld_cd_hint(const cd* p, uint64_t pol) {
  cd v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

constexpr int kMgsPPT = 16;  // points per thread held in registers

__global__ void __launch_bounds__(kRT) k_mgs_grid(cd* w, const cd* const* V, int j, long long n, cd* gpart,
                                                  cd* hout, const int* skip) {
  if (skip && *skip) return;  // grid-uniform: every CTA reads the same flag
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RSmem& s = *reinterpret_cast<RSmem*>(smem_raw);
  cd* ws = reinterpret_cast<cd*>(smem_raw + ((sizeof(RSmem) + 15) / 16) * 16);
  GridSync sy;
  const int P = gridDim.x, rank = blockIdx.x, t = threadIdx.x;
  const long long p0 = n * rank / P, p1 = n * (rank + 1) / P;
  const int cnt = (int)(p1 - p0);
  int buf = 0;
  if (cnt > 0) prefetch_l2_span(V[0] + p0, cnt);
  load_slice_smem(ws, w + p0, cnt);
  for (int i = 0; i <= j; ++i) {
    const cd* vi = V[i] + p0;
    if (i < j && cnt > 0) prefetch_l2_span(V[i + 1] + p0, cnt);
    cd vr[kMgsPPT];
    cd a = mkc(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      vr[k] = q < cnt ? vi[q] : mkc(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      if (q < cnt) a = c_conjmul_acc(a, vr[k], ws[q]);
    }
    for (int q = t + kMgsPPT * kRT; q < cnt; q += kRT) a = c_conjmul_acc(a, vi[q], ws[q]);
    const cd h = sy.reduce(a, s, buf, gpart);
    if (rank == 0 && t == 0) hout[i] = h;
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      if (q < cnt) ws[q] = c_sub(ws[q], c_mul_np(h, vr[k]));
    }
    for (int q = t + kMgsPPT * kRT; q < cnt; q += kRT) ws[q] = c_sub(ws[q], c_mul_np(h, vi[q]));
  }
  cd a = mkc(0.0, 0.0);
  for (int q = t; q < cnt; q += kRT) a = c_conjmul_acc(a, ws[q], ws[q]);
  const cd nn = sy.reduce(a, s, buf, gpart);
  if (rank == 0 && t == 0) hout[j + 1] = nn;
  const double hn = sqrt(nn.x > 0.0 ? nn.x : 0.0);
  const double inv = 1.0 / hn;
  for (int q = t; q < cnt; q += kRT) {
    const cd v = ws[q];
    w[p0 + q] = hn > 0.0 ? mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv)) : v;
  }
}

// Larger levels: this CTA's slice of w lives partly in shared memory (slots
// k < ks of q = t + k*kRT) and partly in registers (up to kMgsReg slots), so w
// of up to ~22k points per SM (3.3M points) stays on chip for the whole chain;
// V_i is read from HBM once for the dot and re-read from L2 for the update.
constexpr int kMgsReg = 16;

struct MgsSmem {
  cd warp[kRT / 32];
  cd bcast[2];
};

__device__ __forceinline__ cd grid_reduce_small(cd v, MgsSmem& s, int& buf, cd* gpart, cg::grid_group& gr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, P = gridDim.x;
  v = warp_sum_c(v);
  if (lane == 0) s.warp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    cd t = lane < kRT / 32 ? s.warp[lane] : mkc(0.0, 0.0);
    t = warp_sum_c(t);
    if (lane == 0) __stcg(&gpart[((long long)buf * P + blockIdx.x) * kVecCap], t);
  }
  gr.sync();
  if (wid == 0) {
    cd q = mkc(0.0, 0.0);
    for (int r = lane; r < P; r += 32) {
      const cd z = __ldcg(&gpart[((long long)buf * P + r) * kVecCap]);
      q.x += z.x;
      q.y += z.y;
    }
    q = warp_sum_c(q);
    if (lane == 0) s.bcast[buf] = q;
  }
  __syncthreads();
  const cd r = s.bcast[buf];
  buf ^= 1;
  return r;
}

__global__ void __launch_bounds__(kRT) k_mgs_grid2(cd* w, const cd* const* V, int j, long long n, cd* gpart,
                                                   cd* hout, int ks, const int* skip, int hint) {
  if (skip && *skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MgsSmem& s = *reinterpret_cast<MgsSmem*>(smem_raw);
  cd* ws = reinterpret_cast<cd*>(smem_raw + ((sizeof(MgsSmem) + 15) / 16) * 16);
  cg::grid_group gr = cg::this_grid();
  const int P = gridDim.x, rank = blockIdx.x, t = threadIdx.x;
  const long long p0 = n * rank / P, p1 = n * (rank + 1) / P;
  const int cnt = (int)(p1 - p0);
  int buf = 0;
  cd wr[kMgsReg];
  const cd* wg = w + p0;
  // (no L2 prefetch of V here: it would evict the L2-resident tier of w)
  load_slice_smem(ws, wg, min(cnt, ks * kRT));  // slot k of thread t = element t + k*kRT
#pragma unroll
  for (int k = 0; k < kMgsReg; ++k) {
    const int q = t + (ks + k) * kRT;
    wr[k] = q < cnt ? wg[q] : mkc(0.0, 0.0);
  }
  const int qg = t + (ks + kMgsReg) * kRT;  // first point of the global (L2-resident) tier
  cd* wgl = w + p0;
  // Every pass batches its basis loads (kB slots per thread in flight before the dependent
  // arithmetic).  After the first dot, ONE fused pass per MGS step applies w -= h_i V_i and
  // forms the next reduction from the updated values -- <V_{i+1}, w> or, after the last
  // update, <w, w> -- so V_{i+1} streams from HBM while V_i is re-read (L2) and a step costs
  // one pass and one grid reduction.  Per thread the sums keep their slot order (shared
  // tier, register tier, global tier): bit-identical to separate dot and update passes.
  // L2 priorities (hint != 0): a basis vector is read twice, in two consecutive passes -- first
  // as V_{i+1} (kept: evict_last), then as V_i (its last use: evict_first) -- so one vector plus
  // the global tier of w stay L2-resident and each pass reads one vector from HBM.
  const uint64_t pk = l2pol_keep(), pd = l2pol_drop();
  auto ldk = [&](const cd* p) { return hint ? ld_cd_hint(p, pk) : *p; };
  auto ldd = [&](const cd* p) { return hint ? ld_cd_hint(p, pd) : *p; };
  constexpr int kB = 4;   // register-tier batch
  constexpr int kS = 4;   // shared-memory tier batch (8 measured slower: spills; profiles/r03i_bench_*.json)
  cd a = mkc(0.0, 0.0);
  {
    const cd* v0 = V[0] + p0;
    for (int k0 = 0; k0 < ks; k0 += kS) {
      cd v[kS];
#pragma unroll
      for (int u = 0; u < kS; ++u) {
        const int q = t + (k0 + u) * kRT;
        v[u] = (k0 + u < ks && q < cnt) ? ldk(v0 + q) : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kS; ++u) {
        const int q = t + (k0 + u) * kRT;
        if (k0 + u < ks && q < cnt) a = c_conjmul_acc(a, v[u], ws[(k0 + u) * kRT + t]);
      }
    }
#pragma unroll
    for (int k0 = 0; k0 < kMgsReg; k0 += kB) {
      cd v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = t + (ks + k0 + u) * kRT;
        v[u] = q < cnt ? ldk(v0 + q) : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = t + (ks + k0 + u) * kRT;
        if (q < cnt) a = c_conjmul_acc(a, v[u], wr[k0 + u]);
      }
    }
    for (int q0 = qg; q0 < cnt; q0 += kB * kRT) {
      cd v[kB], x[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = q0 + u * kRT;
        v[u] = q < cnt ? ldk(v0 + q) : mkc(0.0, 0.0);
        x[u] = q < cnt ? wgl[q] : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (q0 + u * kRT < cnt) a = c_conjmul_acc(a, v[u], x[u]);
    }
  }
  for (int i = 0; i <= j; ++i) {
    const cd h = grid_reduce_small(a, s, buf, gpart, gr);
    if (rank == 0 && t == 0) hout[i] = h;
    const cd* vi = V[i] + p0;
    const bool last = i == j;               // the next reduction is <w, w>
    const cd* vn = last ? vi : V[i + 1] + p0;  // (last: vn unused, any valid pointer)
    a = mkc(0.0, 0.0);
    for (int k0 = 0; k0 < ks; k0 += kS) {
      cd v[kS], n2[kS];
#pragma unroll
      for (int u = 0; u < kS; ++u) {
        const int q = t + (k0 + u) * kRT;
        const bool ok = k0 + u < ks && q < cnt;
        v[u] = ok ? ldd(vi + q) : mkc(0.0, 0.0);
        n2[u] = (ok && !last) ? ldk(vn + q) : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kS; ++u) {
        const int q = t + (k0 + u) * kRT;
        if (k0 + u < ks && q < cnt) {
          const cd x = c_sub(ws[(k0 + u) * kRT + t], c_mul_np(h, v[u]));
          ws[(k0 + u) * kRT + t] = x;
          a = c_conjmul_acc(a, last ? x : n2[u], x);
        }
      }
    }
#pragma unroll
    for (int k0 = 0; k0 < kMgsReg; k0 += kB) {
      cd v[kB], n2[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = t + (ks + k0 + u) * kRT;
        v[u] = q < cnt ? ldd(vi + q) : mkc(0.0, 0.0);
        n2[u] = (q < cnt && !last) ? ldk(vn + q) : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = t + (ks + k0 + u) * kRT;
        if (q < cnt) {
          wr[k0 + u] = c_sub(wr[k0 + u], c_mul_np(h, v[u]));
          a = c_conjmul_acc(a, last ? wr[k0 + u] : n2[u], wr[k0 + u]);
        }
      }
    }
    for (int q0 = qg; q0 < cnt; q0 += kB * kRT) {
      cd v[kB], n2[kB], x[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = q0 + u * kRT;
        v[u] = q < cnt ? ldd(vi + q) : mkc(0.0, 0.0);
        n2[u] = (q < cnt && !last) ? ldk(vn + q) : mkc(0.0, 0.0);
        x[u] = q < cnt ? wgl[q] : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int q = q0 + u * kRT;
        if (q < cnt) {
          const cd y = c_sub(x[u], c_mul_np(h, v[u]));
          wgl[q] = y;
          a = c_conjmul_acc(a, last ? y : n2[u], y);
        }
      }
    }
  }
  const cd nn = grid_reduce_small(a, s, buf, gpart, gr);
  if (rank == 0 && t == 0) hout[j + 1] = nn;
  const double hn = sqrt(nn.x > 0.0 ? nn.x : 0.0);
  const double inv = 1.0 / hn;
  cd* wo = w + p0;
  for (int k = 0; k < ks; ++k) {
    const int q = t + k * kRT;
    if (q < cnt) {
      const cd v = ws[k * kRT + t];
      wo[q] = hn > 0.0 ? mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv)) : v;
    }
  }
#pragma unroll
  for (int k = 0; k < kMgsReg; ++k) {
    const int q = t + (ks + k) * kRT;
    if (q < cnt) {
      const cd v = wr[k];
      wo[q] = hn > 0.0 ? mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv)) : v;
    }
  }
  if (hn > 0.0)
    for (int q = qg; q < cnt; q += kRT) {
      const cd v = wo[q];
      wo[q] = mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv));
    }
}

// TMA-fed form (levels whose w slice AND one basis-vector slice fit shared
// memory together, e.g. the 1025^2 level of config 2): V_{i+1}'s slice is
// streamed HBM -> shared memory by the bulk-copy engine (cp.async.bulk,
// mbarrier completion) while step i computes its dot, waits in the grid
// reduction and applies its update, so the basis stream overlaps the
// synchronisation instead of following it.  V_i is pulled from shared memory
// into registers (kept for the update), then the buffer is handed to the copy
// engine for V_{i+1}.  Same arithmetic and reduction tree as k_mgs_grid.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// same with an L2 eviction-priority hint (policy from createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// thread 0: arm the barrier for `bytes` and issue the slice copy in 32 KB pieces
__device__ __forceinline__ void issue_slice(cd* dst, const cd* src, int cnt, uint64_t* bar) {
  const uint32_t bytes = (uint32_t)cnt * (uint32_t)sizeof(cd);
  mbar_arm(bar, bytes);
  constexpr uint32_t kPiece = 32768;
  for (uint32_t off = 0; off < bytes; off += kPiece) {
    const uint32_t nb = bytes - off < kPiece ? bytes - off : kPiece;
    bulk_g2s(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off, nb, bar);
  }
}

struct MgsTSmem {
  MgsSmem red;
  uint64_t bar;
};

__global__ void __launch_bounds__(kRT) k_mgs_grid_t(cd* w, const cd* const* V, int j, long long n, cd* gpart,
                                                    cd* hout, const int* skip) {
  if (skip && *skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MgsTSmem& s = *reinterpret_cast<MgsTSmem*>(smem_raw);
  constexpr size_t kHead = ((sizeof(MgsTSmem) + 127) / 128) * 128;
  cg::grid_group gr = cg::this_grid();
  const int P = gridDim.x, rank = blockIdx.x, t = threadIdx.x;
  const long long p0 = n * rank / P, p1 = n * (rank + 1) / P;
  const int cnt = (int)(p1 - p0);
  const int cap = (int)((n + P - 1) / P);
  cd* ws = reinterpret_cast<cd*>(smem_raw + kHead);
  cd* vb = ws + ((cap + 7) / 8) * 8;  // 128-byte aligned
  if (t == 0) {
    mbar_init(&s.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && cnt > 0) issue_slice(vb, V[0] + p0, cnt, &s.bar);
  load_slice_smem(ws, w + p0, cnt);
  int buf = 0;
  uint32_t parity = 0;
  for (int i = 0; i <= j; ++i) {
    cd vr[kMgsPPT];
    if (cnt > 0) {
      mbar_wait(&s.bar, parity);
      parity ^= 1u;
    }
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      vr[k] = q < cnt ? vb[q] : mkc(0.0, 0.0);
    }
    cd a = mkc(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      if (q < cnt) a = c_conjmul_acc(a, vr[k], ws[q]);
    }
    // every thread has CONSUMED its V_i values (the dot above), so no shared
    // load from the buffer is still in flight: hand it to the copy engine
    __syncthreads();
    if (i < j && t == 0 && cnt > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_slice(vb, V[i + 1] + p0, cnt, &s.bar);
    }
    const cd h = grid_reduce_small(a, s.red, buf, gpart, gr);
    if (rank == 0 && t == 0) hout[i] = h;
#pragma unroll
    for (int k = 0; k < kMgsPPT; ++k) {
      const int q = t + k * kRT;
      if (q < cnt) ws[q] = c_sub(ws[q], c_mul_np(h, vr[k]));
    }
  }
  __syncthreads();
  cd a = mkc(0.0, 0.0);
  for (int q = t; q < cnt; q += kRT) a = c_conjmul_acc(a, ws[q], ws[q]);
  const cd nn = grid_reduce_small(a, s.red, buf, gpart, gr);
  if (rank == 0 && t == 0) hout[j + 1] = nn;
  const double hn = sqrt(nn.x > 0.0 ? nn.x : 0.0);
  const double inv = 1.0 / hn;
  for (int q = t; q < cnt; q += kRT) {
    const cd v = ws[q];
    w[p0 + q] = hn > 0.0 ? mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv)) : v;
  }
}

// ---------------------------------------------------------------------------
// Low-synchronisation MGS step (one-reduce MGS in the compact-WY form of
// Swirydowicz, Langou, Ananthan, Yang & Thomas, "Low synchronization
// Gram-Schmidt and GMRES algorithms", NLAA 2020).  MGS computes
//     h_i = <V_i, w - sum_{k<i} h_k V_k> = g_i - sum_{k<i} <V_i, V_k> h_k,
// i.e. h = (I + L)^{-1} g with g = V^H w and L the strictly lower part of
// V^H V.  One streaming pass over V_0..V_{j-1} yields g and the new row of L
// (<V_j, V_k>, k < j) together; ONE grid reduction combines them; the new row
// of T = (I + L)^{-1} (t_jk = -sum_{m=k}^{j-1} <V_j, V_m> T_mk, rows < j kept
// in Tg from the earlier steps) and h = T g follow redundantly in every CTA; a
// second pass subtracts h_k V_k (V_j from shared memory, then V_{j-1}..V_0,
// the recently streamed vectors first so they are still in L2); one more
// reduction gives ||w||^2.  Two grid barriers per Arnoldi step instead of
// j + 2, at the price of re-reading the basis (partly from L2).  Same
// coefficients as MGS in exact arithmetic (krylov.py:121-124); the rounding
// differs like the reference's own worker-count-dependent zdotc rounding does.
// The w slice lives in registers (14 points per thread), the V_j slice in
// shared memory, and the other basis vectors stream HBM -> shared memory
// through a TMA ring (cp.async.bulk, mbarrier full/empty pairs) that runs ahead
// across both passes -- pass B's first chunks are already in flight while the
// coefficient reduction and the small triangular work run.  Levels with <= 7168
// points per CTA (the 1025^2 level of config 2: 7099).
constexpr int kLsSlot = 14;                // w points per thread (kRT * 14 = 7168)
constexpr int kLsMaxJ = 63;                // 4 j + 2 scalars fit the staging area
constexpr int kLsStage = 16;               // reduced elements per warp-partial staging round
constexpr int kLsChunk = 2 * kRT;          // ring chunk: 1024 points (16 KB) = 2 per thread
constexpr int kLsChunks = kLsSlot / 2;     // chunks per slice (7)
constexpr int kLsRing = 6;                 // ring stages
constexpr int kLsKeep = 5;                 // last pass-A vectors kept in L2 (evict_last) for pass B
struct LsSmem {
  MgsSmem red;
  cd stage[kRT / 32][kLsStage];            // warp partials; reused for g, l, t-row and h
  uint64_t full[kLsRing], empty[kLsRing];
  const cd* vptr[kLsMaxJ + 1];             // basis pointers (the producer's chunk sources)
  cd gcol[kLsMaxJ + 3];                    // fused Givens step (device-driven GMRES): Hessenberg column,
  cd gsn[kLsMaxJ + 1];                     // earlier rotations
  double gcs[kLsMaxJ + 1];
};
// Device-driven GMRES state of the solve this step belongs to (gm_state_elems layout); st ==
// nullptr: no fused Givens (the launch-driven FGMRES reads the column on the host).
struct GmFuse {
  cd* st;
  int cap, maxit;
  double tol;
  cd* flag;
};
constexpr size_t kLsHead = ((sizeof(LsSmem) + 127) / 128) * 128;

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__global__ void __launch_bounds__(kRT, 1) k_mgs_ls(cd* w, const cd* const* V, int j, long long n, cd* gpart,
                                                   cd* hout, cd* Tg, const int* skip, GmFuse gf) {
  if (skip && *skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LsSmem& s = *reinterpret_cast<LsSmem*>(smem_raw);
  cg::grid_group gr = cg::this_grid();
  const int P = gridDim.x, rank = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const long long p0 = n * rank / P, p1 = n * (rank + 1) / P;
  const int cnt = (int)(p1 - p0);
  cd* ring = reinterpret_cast<cd*>(smem_raw + kLsHead);                 // kLsRing x kLsChunk
  cd* vj = ring + (size_t)kLsRing * kLsChunk;                           // V_j slice
  // chunk sequence: pass A streams V_0..V_{j-1}, pass B V_{j-1}..V_0, kLsChunks chunks each
  const int nchunks = 2 * j * kLsChunks;
  // L2 policy: pass A marks its last kLsKeep vectors evict_last (pass B reads them first,
  // in reverse order) and the others evict_first; pass B reads are the last use this step
  const uint64_t pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();
  auto chunk_pol = [&](int q) {
    const int v = q / kLsChunks;
    return (v < j && v >= j - kLsKeep) ? pol_keep : pol_drop;
  };
  auto chunk_src = [&](int q, int& bytes) -> const cd* {
    const int v = q / kLsChunks, c = q - v * kLsChunks;
    const int k = v < j ? v : 2 * j - 1 - v;
    const int e0 = c * kLsChunk;
    const int ne = cnt - e0 < kLsChunk ? cnt - e0 : kLsChunk;
    bytes = ne > 0 ? ne * (int)sizeof(cd) : 0;
    return s.vptr[k] + p0 + e0;
  };
  auto issue = [&](int q) {  // thread 0
    const int st = q % kLsRing;
    int bytes = 0;
    const cd* src = chunk_src(q, bytes);
    if (bytes > 0) {
      mbar_arm(&s.full[st], (uint32_t)bytes);
      bulk_g2s_hint(ring + (size_t)st * kLsChunk, src, (uint32_t)bytes, &s.full[st], chunk_pol(q));
    } else {
      mbar_arrive1(&s.full[st]);  // empty tail chunk: complete the phase without data
    }
  };
  if (t == 0) {
    for (int st = 0; st < kLsRing; ++st) {
      mbar_init(&s.full[st], 1);
      mbar_init(&s.empty[st], kRT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t <= j) s.vptr[t] = V[t];  // no global pointer load on the producer's refill path
  __syncthreads();
  if (t == 0)
    for (int q = 0; q < kLsRing && q < nchunks; ++q) issue(q);
  cd wr[kLsSlot];
#pragma unroll
  for (int m = 0; m < kLsSlot; ++m) {
    const int q = t + m * kRT;
    wr[m] = q < cnt ? w[p0 + q] : mkc(0.0, 0.0);
  }
  load_slice_smem(vj, V[j] + p0, cnt);
  __syncthreads();
  int qn = 0;  // next chunk to consume
  // consume one chunk: f(m, v) for this thread's two points (m = slot index)
  auto consume = [&](auto&& f) {
    const int st = qn % kLsRing;
    mbar_wait(&s.full[st], (uint32_t)((qn / kLsRing) & 1));
    const cd* rb = ring + (size_t)st * kLsChunk;
    f(rb);
    __syncwarp();
    if (lane == 0) mbar_arrive1(&s.empty[st]);
    // refill the stage of the PREVIOUS chunk (every warp has long released it) with the
    // chunk kLsRing ahead of it: the producer does not wait for this chunk's stragglers
    const int qp = qn - 1;
    if (t == 0 && qp >= 0 && qp + kLsRing < nchunks) {
      const int sp = qp % kLsRing;
      mbar_wait(&s.empty[sp], (uint32_t)((qp / kLsRing) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(qp + kLsRing);
    }
    ++qn;
  };
  const int ne = 2 * j + 1;  // g_0..g_j, then l_0..l_{j-1}
  cd pw[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) pw[k] = mkc(0.0, 0.0);
  auto stash = [&](int e, cd v) {
    v = warp_sum_c(v);
    v.x = __shfl_sync(0xffffffffu, v.x, 0);
    v.y = __shfl_sync(0xffffffffu, v.y, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e == 32 * k + lane) pw[k] = v;
  };
  // pass A: g_k = <V_k, w>, l_k = <V_j, V_k> for k < j
  for (int k = 0; k < j; ++k) {
    cd ag = mkc(0.0, 0.0), al = mkc(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < kLsChunks; ++c) {
      consume([&](const cd* rb) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int q = c * kLsChunk + h2 * kRT + t;
          if (q < cnt) {
            const cd v = rb[h2 * kRT + t];
            ag = c_conjmul_acc(ag, v, wr[2 * c + h2]);
            al = c_conjmul_acc(al, vj[q], v);
          }
        }
      });
    }
    stash(k, ag);
    stash(j + 1 + k, al);
  }
  {
    cd ag = mkc(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < kLsSlot; ++m) {
      const int q = t + m * kRT;
      if (q < cnt) ag = c_conjmul_acc(ag, vj[q], wr[m]);
    }
    stash(j, ag);
  }
  // block partials (16 warps in order) -> gpart region 0, one grid barrier
  for (int e0 = 0; e0 < ne; e0 += kLsStage) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = 32 * k + lane;
      if (e >= e0 && e < e0 + kLsStage && e < ne) s.stage[wid][e - e0] = pw[k];
    }
    __syncthreads();
    if (t < kLsStage && e0 + t < ne) {
      cd a = mkc(0.0, 0.0);
#pragma unroll
      for (int ww = 0; ww < kRT / 32; ++ww) {
        a.x += s.stage[ww][t].x;
        a.y += s.stage[ww][t].y;
      }
      __stcg(&gpart[(long long)rank * kVecCap + e0 + t], a);
    }
    __syncthreads();
  }
  gr.sync();
  cd* tot = &s.stage[0][0];  // [0, 2j]: g then l; [2j+1, 3j]: new T row; [3j+1, 4j+1]: h
  for (int e = wid; e < ne; e += kRT / 32) {  // rank-ordered per lane (all loads in flight), then a warp tree
    cd z[kGridRounds];
#pragma unroll
    for (int u = 0; u < kGridRounds; ++u) {
      const int r = lane + 32 * u;
      z[u] = r < P ? __ldcg(&gpart[(long long)r * kVecCap + e]) : mkc(0.0, 0.0);
    }
    cd a = mkc(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kGridRounds; ++u) {
      a.x += z[u].x;
      a.y += z[u].y;
    }
    a = warp_sum_c(a);
    if (lane == 0) tot[e] = a;
  }
  __syncthreads();
  cd* trow = tot + ne;
  cd* hs = trow + j;
  const long long rj = (long long)j * (j + 1) / 2;
  // T entries come from L2: batches of kLsTB independent loads, then the ordered FMAs
  constexpr int kLsTB = 8;
  if (t < j) {  // t_jk = -sum_{m=k}^{j-1} l_m T_mk
    cd a = mkc(0.0, 0.0);
    for (int m0 = t; m0 < j; m0 += kLsTB) {
      cd tm[kLsTB];
#pragma unroll
      for (int u = 0; u < kLsTB; ++u) {
        const int m = m0 + u;
        tm[u] = m < j ? __ldcg(&Tg[(long long)m * (m + 1) / 2 + t]) : mkc(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kLsTB; ++u) {
        const int m = m0 + u;
        if (m < j) {
          const cd lm = tot[j + 1 + m];
          a.x = __fma_rn(lm.x, tm[u].x, a.x); a.x = __fma_rn(-lm.y, tm[u].y, a.x);
          a.y = __fma_rn(lm.x, tm[u].y, a.y); a.y = __fma_rn(lm.y, tm[u].x, a.y);
        }
      }
    }
    trow[t] = mkc(-a.x, -a.y);
    if (rank == 0) Tg[rj + t] = mkc(-a.x, -a.y);
  }
  if (rank == 0 && t == 0) Tg[rj + j] = mkc(1.0, 0.0);
  __syncthreads();
  if (t <= j) {  // h_i = sum_{k <= i} T_ik g_k
    cd a = mkc(0.0, 0.0);
    const long long ri = (long long)t * (t + 1) / 2;
    for (int k0 = 0; k0 <= t; k0 += kLsTB) {
      cd tk[kLsTB];
#pragma unroll
      for (int u = 0; u < kLsTB; ++u) {
        const int k = k0 + u;
        tk[u] = k > t ? mkc(0.0, 0.0)
                      : (t < j ? (k < t ? __ldcg(&Tg[ri + k]) : mkc(1.0, 0.0)) : (k < j ? trow[k] : mkc(1.0, 0.0)));
      }
#pragma unroll
      for (int u = 0; u < kLsTB; ++u) {
        const int k = k0 + u;
        if (k <= t) {
          const cd gk = tot[k];
          a.x = __fma_rn(tk[u].x, gk.x, a.x); a.x = __fma_rn(-tk[u].y, gk.y, a.x);
          a.y = __fma_rn(tk[u].x, gk.y, a.y); a.y = __fma_rn(tk[u].y, gk.x, a.y);
        }
      }
    }
    hs[t] = a;
    if (rank == 0) hout[t] = a;
  }
  __syncthreads();
  // pass B: w -= h_j V_j (shared), then h_k V_k for k = j-1 .. 0 (ring)
  {
    const cd hj = hs[j];
#pragma unroll
    for (int m = 0; m < kLsSlot; ++m) {
      const int q = t + m * kRT;
      if (q < cnt) wr[m] = c_sub(wr[m], c_mul_np(hj, vj[q]));
    }
  }
  for (int k = j - 1; k >= 0; --k) {
    const cd hk = hs[k];
#pragma unroll
    for (int c = 0; c < kLsChunks; ++c) {
      consume([&](const cd* rb) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int q = c * kLsChunk + h2 * kRT + t;
          if (q < cnt) wr[2 * c + h2] = c_sub(wr[2 * c + h2], c_mul_np(hk, rb[h2 * kRT + t]));
        }
      });
    }
  }
  cd a = mkc(0.0, 0.0);
#pragma unroll
  for (int m = 0; m < kLsSlot; ++m) {
    const int q = t + m * kRT;
    if (q < cnt) a = c_conjmul_acc(a, wr[m], wr[m]);
  }
  int buf = 1;  // gpart region 1 (region 0 holds the coefficient partials)
  const cd nn = grid_reduce_small(a, s.red, buf, gpart, gr);
  if (rank == 0 && t == 0) hout[j + 1] = nn;
  const double hn = sqrt(nn.x > 0.0 ? nn.x : 0.0);
  const double inv = 1.0 / hn;
  // Fused Givens / stopping step of the device-driven GMRES (k_gm_givens's operations in the
  // same order: bit-identical), on warp 0 of CTA 0 while every other warp writes V_{j+1}.
  if (gf.st && rank == 0 && wid == 0) {
    cd* g_ = gf.st + 2;
    cd* sn_ = g_ + gf.cap + 1;
    cd* cs_ = sn_ + gf.cap;
    cd* R_ = cs_ + gf.cap;
    int* fl = reinterpret_cast<int*>(gf.st + 1);
    for (int i = lane; i < j; i += 32) {
      s.gsn[i] = sn_[i];
      s.gcs[i] = cs_[i].x;
    }
    for (int i = lane; i <= j; i += 32) s.gcol[i] = hs[i];
    __syncwarp();
    if (lane == 0) {
      cd* col = s.gcol;
      const double bnorm = gf.st[0].x;
      const double hg = sqrt(fmax(nn.x, 0.0));
      bool finite = isfinite(hg);
      for (int i = 0; i <= j; ++i) finite &= isfinite(col[i].x) && isfinite(col[i].y);
      for (int i = 0; i < j; ++i) {  // rotation i touches entries i, i+1 <= j
        const cd ci = col[i], cn = col[i + 1];
        const double c = s.gcs[i];
        const cd sc = cmul_(s.gsn[i], cn);
        const cd nb = cmul_(mkc(-s.gsn[i].x, s.gsn[i].y), ci);
        col[i] = mkc(c * ci.x + sc.x, c * ci.y + sc.y);
        col[i + 1] = mkc(nb.x + c * cn.x, nb.y + c * cn.y);
      }
      const cd h1 = col[j], h2 = mkc(hg, 0.0);
      double c;
      cd sn;
      const double a1 = cabs_(h1), a2 = cabs_(h2);
      if (a2 == 0.0) { c = 1.0; sn = mkc(0.0, 0.0); }
      else if (a1 == 0.0) { c = 0.0; sn = mkc(1.0, 0.0); }
      else {
        const double tt = hypot(a1, a2);
        c = a1 / tt;
        const cd q = cmul_(mkc(h1.x / a1, h1.y / a1), mkc(h2.x, -h2.y));
        sn = mkc(q.x / tt, q.y / tt);
      }
      cs_[j] = mkc(c, 0.0);
      sn_[j] = sn;
      const cd sh = cmul_(sn, h2);
      col[j] = mkc(c * h1.x + sh.x, c * h1.y + sh.y);
      const cd gj = g_[j];
      g_[j + 1] = cmul_(mkc(-sn.x, sn.y), gj);
      g_[j] = mkc(c * gj.x, c * gj.y);
      const double rel = cabs_(g_[j + 1]) / bnorm;
      fl[1] = j + 1;
      if (!finite) {
        gf.flag->x = 2.0;
        fl[2] = 2;
        fl[0] = 1;
      } else if (hg < 1e-30 || rel <= gf.tol || j + 1 >= gf.maxit) {
        fl[0] = 1;
      }
    }
    __syncwarp();
    cd* Rc = R_ + (long long)j * (j + 1) / 2;  // column j: R[0..j]
    for (int i = lane; i <= j; i += 32) Rc[i] = s.gcol[i];
  }
#pragma unroll
  for (int m = 0; m < kLsSlot; ++m) {
    const int q = t + m * kRT;
    if (q < cnt) {
      const cd v = wr[m];
      w[p0 + q] = hn > 0.0 ? mkc(__dmul_rn(v.x, inv), __dmul_rn(v.y, inv)) : v;
    }
  }
}

static size_t mgs_ls_smem(long long chunk) {
  return kLsHead + (size_t)kLsRing * kLsChunk * sizeof(cd) + (size_t)((chunk + 7) / 8) * 8 * sizeof(cd);
}

long long mgs_ls_tg_elems() { return (long long)(kLsMaxJ + 1) * (kLsMaxJ + 2) / 2; }

static int g_mgs_ls = -1;  // -1: from HDB_MGS_LS (default on)
void set_mgs_ls(int on) { g_mgs_ls = on ? 1 : 0; }
static bool mgs_ls_enabled() {
  if (g_mgs_ls < 0) {
    const char* e = getenv("HDB_MGS_LS");
    g_mgs_ls = e ? (atoi(e) != 0) : 1;
  }
  return g_mgs_ls != 0;
}

static size_t mgs_t_smem(long long chunk) {
  const size_t head = ((sizeof(MgsTSmem) + 127) / 128) * 128;
  return head + 2 * (size_t)((chunk + 7) / 8) * 8 * sizeof(cd);
}

// Launch plan of the cooperative MGS step for length n: 1 = k_mgs_grid (w in
// registers + shared memory), 2 = k_mgs_grid2 with `ks` shared-memory slots,
// 0 = does not fit (caller: launch chain).
static int mgs_grid_plan(long long n, long long& ks_out) {
  init_limits();
  const long long chunk = (n + g_grid - 1) / g_grid;
  static const bool tma = [] {
    const char* e = getenv("HDB_MGS_TMA");
    return !e || atoi(e) != 0;
  }();
  if (tma && chunk <= (long long)kMgsPPT * kRT && mgs_t_smem(chunk) <= g_smem_optin) return 3;
  const size_t sm = smem_for(chunk, false);
  if (sm <= g_smem_optin && chunk <= (long long)kMgsPPT * kRT * 2) return 1;
  // hybrid shared-memory + register slice of w; beyond those the slice stays in
  // w itself (L2-resident up to mgs_global_tier_bytes(); larger levels keep
  // the launch chain)
  const size_t head = ((sizeof(MgsSmem) + 15) / 16) * 16;
  const long long slots = (chunk + kRT - 1) / kRT;
  const long long ks_max = (long long)((g_smem_optin - head) / (sizeof(cd) * kRT));
  if (n * (long long)sizeof(cd) > mgs_global_tier_bytes() && std::max(0LL, slots - kMgsReg) > ks_max) return 0;
  ks_out = std::min(std::max(0LL, slots - kMgsReg), ks_max);
  return 2;
}

bool mgs_grid_fits(long long n) {
  long long ks = 0;
  return mgs_grid_plan(n, ks) != 0;
}

bool mgs_ls_on() { return mgs_ls_enabled(); }

bool mgs_ls_fits(long long n, int j) {
  init_limits();
  const long long chunk = (n + g_grid - 1) / g_grid;
  return mgs_ls_enabled() && j <= kLsMaxJ && chunk <= (long long)kLsSlot * kRT && mgs_ls_smem(chunk) <= g_smem_optin;
}

// returns 0 when launched, 1 when the level does not fit (caller: launch chain)
int launch_mgs_grid(cd* w, const cd* const* Vtab, int j, long long n, cd* gpart, cd* hout, cudaStream_t st,
                    const int* skip, cd* tg, const GmFuseArgs* fuse) {
  if (tg && mgs_ls_fits(n, j)) {
    const size_t sm = mgs_ls_smem((n + g_grid - 1) / g_grid);
    if (!ensure_smem_attr((const void*)k_mgs_ls, sm)) return 1;
    GmFuse gf{nullptr, 0, 0, 0.0, nullptr};
    if (fuse) gf = GmFuse{fuse->st, fuse->cap, fuse->maxit, fuse->tol, fuse->flag};
    void* args[] = {&w, (void*)&Vtab, &j, &n, &gpart, &hout, &tg, (void*)&skip, &gf};
    return cudaLaunchCooperativeKernel((void*)k_mgs_ls, dim3(g_grid), dim3(kRT), args, sm, st) == cudaSuccess ? 0 : 1;
  }
  long long ks = 0;
  const int plan = mgs_grid_plan(n, ks);
  if (plan == 0) return 1;
  if (plan == 2) {
    const size_t head = ((sizeof(MgsSmem) + 15) / 16) * 16;
    const size_t sm2 = head + (size_t)ks * kRT * sizeof(cd);
    if (!ensure_smem_attr((const void*)k_mgs_grid2, sm2)) return 1;
    int ksi = (int)ks;
    static const int hint2 = [] {  // HDB_MGS2_HINT=0: plain loads in the hybrid MGS step
      const char* e = getenv("HDB_MGS2_HINT");
      return e ? atoi(e) : 1;
    }();
    int hint = hint2;
    void* args2[] = {&w, (void*)&Vtab, &j, &n, &gpart, &hout, &ksi, (void*)&skip, &hint};
    return cudaLaunchCooperativeKernel((void*)k_mgs_grid2, dim3(g_grid), dim3(kRT), args2, sm2, st) == cudaSuccess ? 0 : 1;
  }
  if (plan == 3) {
    const size_t sm3 = mgs_t_smem((n + g_grid - 1) / g_grid);
    if (!ensure_smem_attr((const void*)k_mgs_grid_t, sm3)) return 1;
    void* args3[] = {&w, (void*)&Vtab, &j, &n, &gpart, &hout, (void*)&skip};
    return cudaLaunchCooperativeKernel((void*)k_mgs_grid_t, dim3(g_grid), dim3(kRT), args3, sm3, st) == cudaSuccess ? 0 : 1;
  }
  const size_t sm = smem_for((n + g_grid - 1) / g_grid, false);
  if (!ensure_smem_attr((const void*)k_mgs_grid, sm)) return 1;
  void* args[] = {&w, (void*)&Vtab, &j, &n, &gpart, &hout, (void*)&skip};
  return cudaLaunchCooperativeKernel((void*)k_mgs_grid, dim3(g_grid), dim3(kRT), args, sm, st) == cudaSuccess ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Device-driven GMRES control for the launch path (large levels): the host
// enqueues Arnoldi steps in batches without reading anything back; the Givens
// update, the stopping test and the least-squares solve run in single-thread
// kernels with the resident kernel's arithmetic (krylov.py:126-168), and a
// `done` flag makes every later launch of the batch return at once.
// State layout (cd units): [0] (bnorm, 1/bnorm); [1] int flags {done, its,
// status, -}; then g[cap+1], sn[cap], cs[cap] (.x), R[cap(cap+1)/2], y[cap].
namespace {
struct GmView {
  cd* hdr;
  int* fl;
  cd *g, *sn, *cs, *R, *y;
  __device__ GmView(cd* st, int cap) {
    hdr = st;
    fl = reinterpret_cast<int*>(st + 1);
    g = st + 2;
    sn = g + cap + 1;
    cs = sn + cap;
    R = cs + cap;
    y = R + (long long)cap * (cap + 1) / 2;
  }
};
}  // namespace

long long gm_state_elems(int cap) { return 2 + (cap + 1) + 2LL * cap + (long long)cap * (cap + 1) / 2 + cap; }

__global__ void k_gm_init(const cd* nn, cd* st, int cap, cd* flag) {
  GmView v(st, cap);
  const double bnorm = sqrt(fmax(nn->x, 0.0));
  v.hdr[0] = mkc(bnorm, 1.0 / bnorm);
  v.fl[1] = 0;
  v.fl[2] = 0;
  v.g[0] = mkc(bnorm, 0.0);
  if (!isfinite(bnorm)) {
    flag->x = 2.0;
    v.fl[2] = 2;
  }
  v.fl[0] = (bnorm == 0.0 || !isfinite(bnorm)) ? 1 : 0;  // krylov.py:96-97: b = 0 -> x = 0
}

// V0 = b * (1/beta)  (zero initial guess: r0 = b, beta = ||b||)
__global__ void k_gm_scale(const cd* __restrict__ b, cd* __restrict__ v0, const cd* st, long long n) {
  if (reinterpret_cast<const int*>(st + 1)[0]) return;
  const double inv = st[0].y;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const cd x = b[p];
    v0[p] = mkc(__dmul_rn(x.x, inv), __dmul_rn(x.y, inv));
  }
}

// rotations of step j (krylov.py:126-151) from the Hessenberg column the MGS
// step left in hcol[0..j] and ||w||^2 in hcol[j+1].x; stopping test.  One warp:
// the operands are staged into shared memory in parallel, thread 0 runs the
// serial rotation chain on them.
constexpr int kGmThreads = 32;
__global__ void __launch_bounds__(kGmThreads) k_gm_givens(int j, const cd* hcol, cd* st, int cap, int maxit,
                                                          double tol, cd* flag) {
  __shared__ cd col[kMaxCap + 2];
  __shared__ cd ssn[kMaxCap];
  __shared__ double scs[kMaxCap];
  GmView v(st, cap);
  if (v.fl[0]) return;
  const int t = threadIdx.x;
  for (int i = t; i <= j; i += kGmThreads) col[i] = hcol[i];
  for (int i = t; i < j; i += kGmThreads) {
    ssn[i] = v.sn[i];
    scs[i] = v.cs[i].x;
  }
  __syncthreads();
  if (t == 0) {
    const double bnorm = v.hdr[0].x;
    const double hn = sqrt(fmax(hcol[j + 1].x, 0.0));
    bool finite = isfinite(hn);
    for (int i = 0; i <= j; ++i) finite &= isfinite(col[i].x) && isfinite(col[i].y);
    for (int i = 0; i < j; ++i) {  // rotation i touches entries i, i+1 <= j
      const cd ci = col[i], cn = col[i + 1];
      const double c = scs[i];
      const cd sc = cmul_(ssn[i], cn);
      const cd nb = cmul_(mkc(-ssn[i].x, ssn[i].y), ci);
      col[i] = mkc(c * ci.x + sc.x, c * ci.y + sc.y);
      col[i + 1] = mkc(nb.x + c * cn.x, nb.y + c * cn.y);
    }
    const cd h1 = col[j], h2 = mkc(hn, 0.0);
    double c;
    cd sn;
    const double a1 = cabs_(h1), a2 = cabs_(h2);
    if (a2 == 0.0) { c = 1.0; sn = mkc(0.0, 0.0); }
    else if (a1 == 0.0) { c = 0.0; sn = mkc(1.0, 0.0); }
    else {
      const double tt = hypot(a1, a2);
      c = a1 / tt;
      const cd q = cmul_(mkc(h1.x / a1, h1.y / a1), mkc(h2.x, -h2.y));
      sn = mkc(q.x / tt, q.y / tt);
    }
    v.cs[j] = mkc(c, 0.0);
    v.sn[j] = sn;
    const cd sh = cmul_(sn, h2);
    col[j] = mkc(c * h1.x + sh.x, c * h1.y + sh.y);
    const cd gj = v.g[j];
    v.g[j + 1] = cmul_(mkc(-sn.x, sn.y), gj);
    v.g[j] = mkc(c * gj.x, c * gj.y);
    const double rel = cabs_(v.g[j + 1]) / bnorm;
    v.fl[1] = j + 1;
    if (!finite) {
      flag->x = 2.0;
      v.fl[2] = 2;
      v.fl[0] = 1;
    } else if (hn < 1e-30 || rel <= tol || j + 1 >= maxit) {
      v.fl[0] = 1;
    }
  }
  __syncthreads();
  cd* Rc = v.R + (long long)j * (j + 1) / 2;  // column j: R[0..j]
  for (int i = t; i <= j; i += kGmThreads) Rc[i] = col[i];
}

// least squares R y = g (krylov.py:161-168), its = flags[1]; R staged in shared
// memory when it fits (its <= 63), serial substitution on thread 0
constexpr int kGmRStage = 2048;
__global__ void __launch_bounds__(kGmThreads) k_gm_solve(cd* st, int cap) {
  __shared__ cd sR[kGmRStage];
  __shared__ cd sg[64];
  __shared__ cd ys[64];
  GmView v(st, cap);
  const int its = v.fl[1];
  const long long nr = (long long)its * (its + 1) / 2;
  const bool staged = nr <= kGmRStage && its <= 64;
  if (staged) {
    for (int i = threadIdx.x; i < nr; i += kGmThreads) sR[i] = v.R[i];
    for (int i = threadIdx.x; i < its; i += kGmThreads) sg[i] = v.g[i];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const cd* R = staged ? sR : v.R;
  const cd* g = staged ? sg : v.g;
  for (int i = its - 1; i >= 0; --i) {
    cd accy = g[i];
    for (int k = i + 1; k < its; ++k) {
      const cd pr = cmul_(R[(long long)k * (k + 1) / 2 + i], staged ? ys[k] : v.y[k]);
      accy = mkc(accy.x - pr.x, accy.y - pr.y);
    }
    const cd yi = cdiv_(accy, R[(long long)i * (i + 1) / 2 + i]);
    if (staged) ys[i] = yi;
    v.y[i] = yi;
  }
}

// explicit true residual norm (krylov.py:174) -> the solve's count / relres slots
__global__ void k_gm_final(const cd* nn, const cd* st, int cap, int* its_out, double* rel_out, cd* flag) {
  const int* fl = reinterpret_cast<const int*>(st + 1);
  const double bnorm = st[0].x;
  const double fin = bnorm > 0.0 ? sqrt(fmax(nn->x, 0.0)) / bnorm : 0.0;
  if (its_out) *its_out = fl[1];
  if (rel_out) *rel_out = fin;
  if (!isfinite(fin)) flag->x = 2.0;
  (void)cap;
}

void launch_gm_init(const cd* nn, cd* st, int cap, cd* flag, cudaStream_t s) { k_gm_init<<<1, 1, 0, s>>>(nn, st, cap, flag); }
void launch_gm_scale(const cd* b, cd* v0, const cd* st, long long n, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4 * 148);
  k_gm_scale<<<blocks, 256, 0, s>>>(b, v0, st, n);
}
void launch_gm_givens(int j, const cd* hcol, cd* st, int cap, int maxit, double tol, cd* flag, cudaStream_t s) {
  k_gm_givens<<<1, kGmThreads, 0, s>>>(j, hcol, st, cap, maxit, tol, flag);
}
void launch_gm_solve(cd* st, int cap, cudaStream_t s) { k_gm_solve<<<1, kGmThreads, 0, s>>>(st, cap); }
void launch_gm_final(const cd* nn, const cd* st, int cap, int* its_out, double* rel_out, cd* flag, cudaStream_t s) {
  k_gm_final<<<1, 1, 0, s>>>(nn, st, cap, its_out, rel_out, flag);
}
const int* gm_flags(const cd* st) { return reinterpret_cast<const int*>(st + 1); }
cd* gm_y(cd* st, int cap) { return st + 2 + (cap + 1) + 2LL * cap + (long long)cap * (cap + 1) / 2; }

}  // namespace hdb
