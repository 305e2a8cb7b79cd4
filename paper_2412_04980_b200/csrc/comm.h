// Inter-rank communication for the row-slab decomposition.
//
// NcclComm    one process per GPU; NCCL (dlopen'd from the torch-bundled
//             libnccl.so.2) all-reduce for dots, grouped send/recv for halos,
//             grouped send/recv all-gather for replicated coarse levels.
// ThreadComm  ranks are host threads of one process (own stream and engine
//             each, e.g. several slabs on one GPU for testing): host barrier +
//             device-to-device copies; kernels never wait on each other.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace hdb {

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() {}
  // in-place sum of `count` doubles in device memory, identical result on every rank
  virtual void allreduce(double* dev, int count, cudaStream_t st) = 0;
  // rows exchange with the neighbours: up = rank-1, down = rank+1 (absent at the ends)
  virtual void exchange(const void* send_up, void* recv_up, size_t bytes_up, const void* send_down,
                        void* recv_down, size_t bytes_down, cudaStream_t st) = 0;
  // all-gather of row-contiguous slabs into a full vector (byte offsets/sizes per rank)
  virtual void allgatherv(const void* local, void* full, const std::vector<size_t>& off,
                          const std::vector<size_t>& bytes, cudaStream_t st) = 0;
};

Comm* make_nccl_comm(const char* unique_id128, int nranks, int rank);  // throws on failure
void nccl_unique_id(char* out128);
Comm* make_thread_comm(long long group, int nranks, int rank);
void nccl_selftest(cudaStream_t st);  // one-rank round trip through the NCCL binding (throws on failure)

}  // namespace hdb
