#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "comm.h"
#include "engine.h"

namespace hdb {

// ----------------------------------------------------------------- NCCL
// Minimal NCCL ABI (nccl.h of NCCL 2.x), resolved at run time so single-GPU
// use has no NCCL dependency.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { ncclSuccess = 0 };
enum { ncclInt8 = 0, ncclFloat64 = 8 };
enum { ncclSum = 0 };
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(ncclUniqueId*);
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  int (*CommDestroy)(ncclComm_t);
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  const char* (*GetErrorString)(int);
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char* env = getenv("HDB_NCCL_LIB");
  const char* cands[] = {env ? env : "", "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c || !*c) continue;
    api.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) throw Error(E_CUDA, "cannot dlopen libnccl.so.2 (import torch first or set HDB_NCCL_LIB)");
  auto sym = [&](const char* n) {
    void* p = dlsym(api.h, n);
    if (!p) throw Error(E_CUDA, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = (int (*)(ncclUniqueId*))sym("ncclGetUniqueId");
  api.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))sym("ncclCommInitRank");
  api.CommDestroy = (int (*)(ncclComm_t))sym("ncclCommDestroy");
  api.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclAllReduce");
  api.Send = (int (*)(const void*, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclSend");
  api.Recv = (int (*)(void*, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclRecv");
  api.GroupStart = (int (*)())sym("ncclGroupStart");
  api.GroupEnd = (int (*)())sym("ncclGroupEnd");
  api.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
  return api;
}

#define NCCL_CHECK(x)                                                                          \
  do {                                                                                         \
    int r_ = (x);                                                                              \
    if (r_ != ncclSuccess) throw Error(E_CUDA, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  NcclComm(const char* id, int n, int r) {
    rank = r;
    size = n;
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    NCCL_CHECK(nccl().CommInitRank(&c, n, u, r));
  }
  ~NcclComm() override {
    if (c) nccl().CommDestroy(c);
  }
  void allreduce(double* dev, int count, cudaStream_t st) override {
    NCCL_CHECK(nccl().AllReduce(dev, dev, (size_t)count, ncclFloat64, ncclSum, c, st));
  }
  void exchange(const void* su, void* ru, size_t bu, const void* sd, void* rd, size_t bd, cudaStream_t st) override {
    NCCL_CHECK(nccl().GroupStart());
    if (rank > 0) {
      NCCL_CHECK(nccl().Send(su, bu, ncclInt8, rank - 1, c, st));
      NCCL_CHECK(nccl().Recv(ru, bu, ncclInt8, rank - 1, c, st));
    }
    if (rank < size - 1) {
      NCCL_CHECK(nccl().Send(sd, bd, ncclInt8, rank + 1, c, st));
      NCCL_CHECK(nccl().Recv(rd, bd, ncclInt8, rank + 1, c, st));
    }
    NCCL_CHECK(nccl().GroupEnd());
  }
  void allgatherv(const void* local, void* full, const std::vector<size_t>& off, const std::vector<size_t>& bytes,
                  cudaStream_t st) override {
    HDB_CUDA(cudaMemcpyAsync((char*)full + off[rank], local, bytes[rank], cudaMemcpyDeviceToDevice, st));
    NCCL_CHECK(nccl().GroupStart());
    for (int r = 0; r < size; ++r) {
      if (r == rank) continue;
      NCCL_CHECK(nccl().Send(local, bytes[rank], ncclInt8, r, c, st));
      NCCL_CHECK(nccl().Recv((char*)full + off[r], bytes[r], ncclInt8, r, c, st));
    }
    NCCL_CHECK(nccl().GroupEnd());
  }
};

Comm* make_nccl_comm(const char* id, int n, int r) { return new NcclComm(id, n, r); }

void nccl_unique_id(char* out) {
  ncclUniqueId u;
  NCCL_CHECK(nccl().GetUniqueId(&u));
  std::memcpy(out, u.internal, 128);
}

// ---------------------------------------------------------------- threads
struct ThreadGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> p0, p1;    // published device pointers
  std::vector<std::vector<double>> vals;
  std::vector<long long> tag;          // per-rank (kind, size) of the collective being entered
  std::vector<int> dev;                // CUDA device of every rank (one GPU per rank thread: P2P halos)
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

static std::mutex g_groups_m;
static std::map<long long, ThreadGroup*> g_groups;

struct ThreadComm : Comm {
  ThreadGroup* g;
  ThreadComm(long long group, int n, int r) {
    rank = r;
    size = n;
    std::lock_guard<std::mutex> lk(g_groups_m);
    auto it = g_groups.find(group);
    if (it == g_groups.end()) {
      g = new ThreadGroup();
      g->n = n;
      g->p0.assign(n, nullptr);
      g->p1.assign(n, nullptr);
      g->vals.assign(n, {});
      g->tag.assign(n, 0);
      g->dev.assign(n, -1);
      g_groups[group] = g;
    } else {
      g = it->second;
    }
    cudaGetDevice(&g->dev[r]);
  }
  // Rank threads that own different GPUs of one node exchange halos with direct
  // peer-to-peer copies over NVLink (cudaMemcpyAsync between peer allocations): enable
  // peer access to the neighbours' devices once, after every rank has published its device.
  bool peers_ready = false;
  void enable_peers() {
    if (peers_ready) return;
    peers_ready = true;
    for (int nb : {rank - 1, rank + 1}) {
      if (nb < 0 || nb >= size || g->dev[nb] < 0 || g->dev[nb] == g->dev[rank]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, g->dev[rank], g->dev[nb]) == cudaSuccess && can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[nb], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          throw Error(E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
      }
    }
  }
  // every rank must enter the same collective: publish (kind, size), check after the barrier
  void enter(long long kind, long long size) {
    g->tag[rank] = kind * (1LL << 40) + size;
    g->barrier();
    for (int r = 0; r < this->size; ++r)
      if (g->tag[r] != g->tag[rank])
        throw Error(E_CUDA, "thread transport: ranks entered different collectives (kind/size " +
                                std::to_string(g->tag[rank]) + " vs " + std::to_string(g->tag[r]) + ")");
  }
  void allreduce(double* dev, int count, cudaStream_t st) override {
    std::vector<double>& mine = g->vals[rank];
    mine.resize(count);
    HDB_CUDA(cudaMemcpyAsync(mine.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    HDB_CUDA(cudaStreamSynchronize(st));
    enter(1, count);
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < size; ++r)
      for (int i = 0; i < count; ++i) sum[i] += g->vals[r][i];  // rank order: identical everywhere
    g->barrier();
    HDB_CUDA(cudaMemcpyAsync(dev, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
    HDB_CUDA(cudaStreamSynchronize(st));
  }
  void exchange(const void* su, void* ru, size_t bu, const void* sd, void* rd, size_t bd, cudaStream_t st) override {
    HDB_CUDA(cudaStreamSynchronize(st));
    g->p0[rank] = su;  // my first rows (for rank-1)
    g->p1[rank] = sd;  // my last rows (for rank+1)
    enter(2, (long long)bu);
    enable_peers();
    if (rank > 0) HDB_CUDA(cudaMemcpyAsync(ru, g->p1[rank - 1], bu, cudaMemcpyDeviceToDevice, st));
    if (rank < size - 1) HDB_CUDA(cudaMemcpyAsync(rd, g->p0[rank + 1], bd, cudaMemcpyDeviceToDevice, st));
    HDB_CUDA(cudaStreamSynchronize(st));
    g->barrier();
  }
  void allgatherv(const void* local, void* full, const std::vector<size_t>& off, const std::vector<size_t>& bytes,
                  cudaStream_t st) override {
    HDB_CUDA(cudaStreamSynchronize(st));
    g->p0[rank] = local;
    enter(3, (long long)off.size());
    for (int r = 0; r < size; ++r)
      HDB_CUDA(cudaMemcpyAsync((char*)full + off[r], g->p0[r], bytes[r], cudaMemcpyDeviceToDevice, st));
    HDB_CUDA(cudaStreamSynchronize(st));
    g->barrier();
  }
};

Comm* make_thread_comm(long long group, int n, int r) { return new ThreadComm(group, n, r); }

// One-rank NCCL round trip on the calling engine's device and stream: resolves the
// library, creates a communicator, runs the three collectives the slab path uses and
// checks their results (a single GPU can exercise the binding, not the transport).
void nccl_selftest(cudaStream_t st) {
  char id[128];
  nccl_unique_id(id);
  std::unique_ptr<Comm> c(make_nccl_comm(id, 1, 0));
  const int n = 6;
  double h[n] = {1.5, -2.25, 3.0, 0.0, 1e300, -7.0}, back[2 * n];
  double *d = nullptr, *full = nullptr;
  HDB_CUDA(cudaMalloc(&d, sizeof(double) * n));
  HDB_CUDA(cudaMalloc(&full, sizeof(double) * n));
  HDB_CUDA(cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  c->allreduce(d, n, st);                                            // sum over one rank: unchanged
  c->exchange(d, d, 16, d + 2, d + 2, 16, st);                       // no neighbours: nothing moves
  c->allgatherv(d, full, {0}, {sizeof(double) * n}, st);             // one slab: a copy
  HDB_CUDA(cudaMemcpyAsync(back, d, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  HDB_CUDA(cudaMemcpyAsync(back + n, full, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  HDB_CUDA(cudaStreamSynchronize(st));
  cudaFree(d);
  cudaFree(full);
  for (int i = 0; i < n; ++i)
    if (back[i] != h[i] || back[n + i] != h[i]) throw Error(E_CUDA, "NCCL self-test: collective changed the data");
}

}  // namespace hdb
