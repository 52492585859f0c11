// NCCL through dlopen (types from nccl.h, symbols resolved at first use).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "setup.hpp"

namespace sdmkb {

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL: cannot open libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) err = std::string("NCCL: missing symbol ") + name;
      return f;
    };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
    n.Send = (decltype(n.Send))sym("ncclSend");
    n.Recv = (decltype(n.Recv))sym("ncclRecv");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
  });
  if (!err.empty()) throw RuntimeError(err);
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw RuntimeError(std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void Comm::unique_id(unsigned char out[kNcclIdBytes]) {
  ncclUniqueId id;
  check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == kNcclIdBytes, "ncclUniqueId size");
  std::memcpy(out, &id, kNcclIdBytes);
}

Comm::Comm(int rank, int nranks, const unsigned char id[kNcclIdBytes], int device) : rank_(rank), nranks_(nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("comm init: need 0 <= rank < nranks");
  if (cudaSetDevice(device) != cudaSuccess) throw RuntimeError("comm init: cudaSetDevice failed");
  ncclUniqueId uid;
  std::memcpy(&uid, id, kNcclIdBytes);
  ncclComm_t c = nullptr;
  check(nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  comm_ = c;
}

Comm::~Comm() {
  if (comm_) nccl().CommDestroy((ncclComm_t)comm_);
}

void Comm::exchange(const double* send, const std::vector<int64_t>& so, double* recv, const std::vector<int64_t>& ro,
                    cudaStream_t st) {
  const Nccl& n = nccl();
  check(n.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < nranks_; ++q) {
    if (q == rank_) continue;
    const int64_t ns = so[q + 1] - so[q], nr = ro[q + 1] - ro[q];
    if (ns > 0) check(n.Send(send + so[q], (size_t)ns, ncclFloat64, q, (ncclComm_t)comm_, st), "ncclSend");
    if (nr > 0) check(n.Recv(recv + ro[q], (size_t)nr, ncclFloat64, q, (ncclComm_t)comm_, st), "ncclRecv");
  }
  check(n.GroupEnd(), "ncclGroupEnd");
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t st) {
  check(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm_, st), "ncclAllReduce");
}

void Comm::allgather(const double* send, double* recv, size_t count, cudaStream_t st) {
  check(nccl().AllGather(send, recv, count, ncclFloat64, (ncclComm_t)comm_, st), "ncclAllGather");
}

}  // namespace sdmkb
