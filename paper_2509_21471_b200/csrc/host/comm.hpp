// NCCL for the multi-GPU evaluation (one process per GPU): the halo
// exchange of outgoing expansions and the assembly of u run on the
// context's own stream.  libnccl.so.2 is opened at first use (the process
// usually has torch's copy loaded already), so single-GPU users and the CPU
// test container never need it.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace sdmkb {

constexpr int kNcclIdBytes = 128;

class Comm {
 public:
  // rank 0 creates the id; every rank passes the same bytes to init
  static void unique_id(unsigned char out[kNcclIdBytes]);
  Comm(int rank, int nranks, const unsigned char id[kNcclIdBytes], int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }
  // one NCCL group: send[q] doubles to rank q, recv[q] doubles from rank q
  void exchange(const double* send, const std::vector<int64_t>& send_off, double* recv,
                const std::vector<int64_t>& recv_off, cudaStream_t st);
  void allreduce_sum(double* buf, size_t count, cudaStream_t st);
  // recv[r * count + i] = rank r's send[i]
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st);

 private:
  void* comm_ = nullptr;
  int rank_ = 0, nranks_ = 1;
};

}  // namespace sdmkb
