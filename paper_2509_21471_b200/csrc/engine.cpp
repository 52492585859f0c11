// B200 DMK engine: host orchestration of the sm_100a passes.
// Citations are to the reference passes each stage reproduces.
#include "engine.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <malloc.h>


namespace sdmkb {

namespace {

constexpr double PI = 3.14159265358979323846;

// Chebyshev proxy machinery on the host (dmk.cpp:25-66): nodes, barycentric
// weights, Lagrange basis with the exact-hit rule, child matrices.
struct Cheb1 {
  int p;
  std::vector<double> x, w;
  explicit Cheb1(int p_) : p(p_), x(p_), w(p_) {
    for (int i = 0; i < p; ++i) {
      double a = (2.0 * i + 1.0) * PI / (2.0 * p);
      x[i] = std::cos(a);
      w[i] = (i % 2 ? -1.0 : 1.0) * std::sin(a);
    }
  }
  void basis(double t, double* out) const {
    for (int i = 0; i < p; ++i)
      if (t == x[i]) {
        for (int j = 0; j < p; ++j) out[j] = j == i ? 1.0 : 0.0;
        return;
      }
    double s = 0.0;
    for (int i = 0; i < p; ++i) {
      out[i] = w[i] / (t - x[i]);
      s += out[i];
    }
    double inv = 1.0 / s;
    for (int i = 0; i < p; ++i) out[i] *= inv;
  }
  // row i: parent basis at child node i of the lower (bit 0) / upper half
  std::vector<double> child(int bit) const {
    std::vector<double> M((size_t)p * p);
    double off = bit ? 1.0 : -1.0;
    for (int i = 0; i < p; ++i) basis((x[i] + off) * 0.5, M.data() + (size_t)i * p);
    return M;
  }
};

std::vector<double> transpose(const std::vector<double>& M, int p) {
  std::vector<double> T((size_t)p * p);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) T[(size_t)j * p + i] = M[(size_t)i * p + j];
  return T;
}

bool timing_on() {
  static const bool on = std::getenv("SDMK_TIMING") != nullptr;
  return on;
}

// band limit in mode-index units, squared (dmk.cpp:472-477)
double band_r2(const Plan& P, int M, double spacing) {
  if (P.window != kProlate) return 3.0 * double(M) * M + 1.0;
  double b = P.c / spacing;
  return b * b * (1.0 + 1e-12);
}

// Packs host vectors into one pinned blob for a single H2D copy.
struct Packer {
  struct Item {
    size_t off, bytes;
    const void* src;
  };
  std::vector<Item> items;
  size_t total = 0;
  template <class T>
  size_t add(const std::vector<T>& v) {
    total = (total + 127) & ~size_t(127);
    size_t off = total;
    items.push_back({off, v.size() * sizeof(T), v.data()});
    total += v.size() * sizeof(T);
    return off;
  }
  // all items into one (pinned) staging buffer, in 1 MB pieces over the host threads
  void copy_to(char* dst) const {
    constexpr size_t kPiece = size_t(1) << 20;
    std::vector<std::array<size_t, 3>> pieces;  // (dst offset, src item, src offset)
    for (size_t i = 0; i < items.size(); ++i)
      for (size_t o = 0; o < items[i].bytes; o += kPiece) pieces.push_back({items[i].off + o, i, o});
#pragma omp parallel for schedule(dynamic, 1) if (pieces.size() > 4)
    for (size_t k = 0; k < pieces.size(); ++k) {
      const Item& it = items[pieces[k][1]];
      const size_t o = pieces[k][2];
      std::memcpy(dst + pieces[k][0], static_cast<const char*>(it.src) + o, std::min(kPiece, it.bytes - o));
    }
  }
};

}  // namespace

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw OomError(std::string(what) + ": out of device memory");
  }
  throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

Arena::~Arena() {
  for (auto& kv : bufs_) cudaFree(kv.second.base);
}

void* Arena::get(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  auto it = bufs_.find(name);
  if (it != bufs_.end() && it->second.req >= bytes) return static_cast<char*>(it->second.base) + (guard_ ? kGuard : 0);
  if (it != bufs_.end()) {
    cudaFree(it->second.base);
    bufs_.erase(it);
  }
  const size_t alloc = guard_ ? bytes + 2 * kGuard : bytes + bytes / 16 + 256;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, alloc);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw OomError("device allocation of " + std::to_string(alloc) + " bytes for '" + name + "' failed");
  }
  if (guard_) {
    char* c = static_cast<char*>(p);
    cuda_check(cudaMemset(c, 0xA5, kGuard), "guard memset");
    cuda_check(cudaMemset(c + kGuard, 0xFF, bytes), "poison memset");
    cuda_check(cudaMemset(c + kGuard + bytes, 0xA5, kGuard), "guard memset");
    cuda_check(cudaDeviceSynchronize(), "guard memset");
  }
  bufs_[name] = {p, alloc, guard_ ? bytes : alloc};
  return static_cast<char*>(p) + (guard_ ? kGuard : 0);
}

void Arena::set_guard(bool on) {
  if (on == guard_) return;
  cudaDeviceSynchronize();
  for (auto& kv : bufs_) cudaFree(kv.second.base);
  bufs_.clear();
  guard_ = on;
}

std::vector<std::string> Arena::check() const {
  std::vector<std::string> bad;
  if (!guard_) return bad;
  cuda_check(cudaDeviceSynchronize(), "guard check");
  std::vector<unsigned char> h(kGuard);
  for (auto& kv : bufs_) {
    const char* c = static_cast<const char*>(kv.second.base);
    bool ok = true;
    for (const char* g : {c, c + kGuard + kv.second.req}) {
      cuda_check(cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost), "guard check");
      for (unsigned char v : h) ok = ok && v == 0xA5;
    }
    if (!ok) bad.push_back(kv.first);
  }
  return bad;
}

bool Arena::selftest() {
  if (!guard_) return false;
  bool caught = true;
  for (int side = 0; side < 2; ++side) {
    const std::string name = "guard_selftest";
    char* p = static_cast<char*>(get(name, 1000));
    cuda_check(cudaMemset(side ? p - 1 : p + 1000, 0, 1), "guard selftest");
    const std::vector<std::string> bad = check();
    caught = caught && bad.size() == 1 && bad[0] == name;
    cudaFree(bufs_[name].base);
    bufs_.erase(name);
  }
  return caught && check().empty();
}

size_t Arena::bytes() const {
  size_t s = 0;
  for (auto& kv : bufs_) s += kv.second.alloc;
  return s;
}

Pinned::~Pinned() {
  for (auto& kv : bufs_) cudaFreeHost(kv.second.first);
}

void* Pinned::get(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  auto it = bufs_.find(name);
  if (it != bufs_.end() && it->second.second >= bytes) return it->second.first;
  if (it != bufs_.end()) {
    cudaFreeHost(it->second.first);
    bufs_.erase(it);
  }
  size_t alloc = bytes + bytes / 8 + 256;
  void* p = nullptr;
  cuda_check(cudaMallocHost(&p, alloc), "cudaMallocHost");
  bufs_[name] = {p, alloc};
  return p;
}

// The host passes rebuild tree, neighbour and work lists (tens of MB of
// std::vectors) on every evaluation.  With glibc's default thresholds those
// blocks are mmapped and returned on free, so every call page-faults them in
// again (~1 ms per 4 MB); keeping them in the heap makes the host critical
// path between the sort and the upward pass ~20 % shorter.  Process-wide;
// SDMK_NO_MALLOPT=1 leaves the allocator alone.
static void tune_host_allocator() {
  static bool done = false;
  if (done) return;
  done = true;
  mallopt(M_MMAP_THRESHOLD, 512 << 20);
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
}

Context::Context(int device) : device_(device) {
  tune_host_allocator();
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&str_ev_, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&x_ev_, cudaEventDisableTiming), "cudaEventCreate");
}

Context::~Context() {
  cudaSetDevice(device_);
  if (st_) cudaStreamSynchronize(st_);
  for (auto& e : ev_) cudaEventDestroy(e);
  for (auto& e : pw_ev_) cudaEventDestroy(e);
  for (auto& e : stage_ev_) cudaEventDestroy(e);
  if (st2_) cudaStreamSynchronize(st2_);
  if (str_ev_) cudaEventDestroy(str_ev_);
  if (x_ev_) cudaEventDestroy(x_ev_);
  if (st2_) cudaStreamDestroy(st2_);
  if (st_) cudaStreamDestroy(st_);
}

void Context::sync() { cuda_check(cudaStreamSynchronize(st_), "stream synchronize"); }

// Host <-> device copies of the caller's arrays.  Pinned (or device) memory
// goes straight to the copy engine; pageable memory is staged through a ring
// of pinned chunks, the chunk copies on the host threads overlapping the DMA
// of the previous chunk (a pageable cudaMemcpy runs at a fraction of the
// link rate).
namespace {
bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t blk = size_t(1) << 20;
  const int64_t nblk = (int64_t)((bytes + blk - 1) / blk);
#pragma omp parallel for schedule(static) if (nblk > 1)
  for (int64_t i = 0; i < nblk; ++i) {
    const size_t o = (size_t)i * blk, n = std::min(blk, bytes - o);
    std::memcpy((char*)dst + o, (const char*)src + o, n);
  }
}
constexpr size_t kStageBytes = size_t(32) << 20;     // largest ring chunk
constexpr size_t kStageMin = size_t(1) << 20;        // pageable copies above this are staged
// chunk of a staged copy: about an eighth of it (so the host copies and the
// DMA overlap even for a few tens of MB), between 4 and 32 MB
size_t stage_chunk(size_t bytes) { return std::min(kStageBytes, std::max(size_t(4) << 20, (bytes / 8 + 4095) & ~size_t(4095))); }
constexpr size_t kSideStreamMin = size_t(32) << 20;  // pinned strengths above this go on the side stream
constexpr int kStages = 4;
}  // namespace

void Context::stage_events() {
  if (!stage_ev_.empty()) return;
  for (int i = 0; i < kStages; ++i) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    stage_ev_.push_back(e);
  }
}

void Context::copy_in(void* dst, const void* src, size_t bytes, bool device_ptrs) {
  if (bytes == 0) return;
  if (device_ptrs || !is_pageable(src) || bytes <= kStageMin) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_),
               "copy in");
    return;
  }
  stage_events();
  char* ring = (char*)pinned_.get("stage", kStages * kStageBytes);
  const size_t ck = stage_chunk(bytes);
  int k = 0;
  for (size_t o = 0; o < bytes; o += ck, k = (k + 1) % kStages) {
    const size_t n = std::min(ck, bytes - o);
    cuda_check(cudaEventSynchronize(stage_ev_[k]), "stage wait");  // the chunk's previous DMA is done
    par_memcpy(ring + k * kStageBytes, (const char*)src + o, n);
    cuda_check(cudaMemcpyAsync((char*)dst + o, ring + k * kStageBytes, n, cudaMemcpyHostToDevice, st_), "copy in");
    cudaEventRecord(stage_ev_[k], st_);
  }
}

void Context::copy_out(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (!is_pageable(dst) || bytes <= kStageMin) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st_), "copy out");
    return;
  }
  stage_events();
  char* ring = (char*)pinned_.get("stage", kStages * kStageBytes);
  const size_t ck = stage_chunk(bytes);
  const size_t nch = (bytes + ck - 1) / ck;
  auto issue = [&](size_t c) {
    const size_t o = c * ck, n = std::min(ck, bytes - o);
    cuda_check(cudaMemcpyAsync(ring + (c % kStages) * kStageBytes, (const char*)src + o, n, cudaMemcpyDeviceToHost, st_),
               "copy out");
    cudaEventRecord(stage_ev_[c % kStages], st_);
  };
  for (size_t c = 0; c < std::min<size_t>(nch, kStages - 1); ++c) issue(c);
  for (size_t c = 0; c < nch; ++c) {
    if (c + kStages - 1 < nch) issue(c + kStages - 1);  // keep the copy engine busy
    cuda_check(cudaEventSynchronize(stage_ev_[c % kStages]), "stage wait");
    const size_t o = c * ck, n = std::min(ck, bytes - o);
    par_memcpy((char*)dst + o, ring + (c % kStages) * kStageBytes, n);
  }
}

void Context::set_shard(int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("set_shard: need 0 <= rank < nranks");
  if (comm_ && (rank != comm_->rank() || nranks != comm_->nranks()))
    throw InvalidArgument("set_shard: the context's communicator fixes rank and nranks");
  rank_ = rank;
  nranks_ = nranks;
  prob_.ready = false;  // lists depend on the shard
}

void Context::comm_init(int rank, int nranks, const unsigned char* id) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  comm_.reset();
  comm_ = std::make_unique<Comm>(rank, nranks, id, device_);
  rank_ = rank;
  nranks_ = nranks;
  prob_.ready = false;
}

void Context::set_manual_exchange(bool on) {
  manual_x_ = on;
  prob_.ready = false;
}

void Context::halo_slab(int peer, bool recv, double** ptr, int64_t* count) {
  const Problem& pr = prob_;
  if (!begun_ || !pr.halo) throw InvalidArgument("halo_slab: no evaluation between evaluate_begin and evaluate_end");
  if (peer < 0 || peer >= nranks_) throw InvalidArgument("halo_slab: bad peer");
  const std::vector<int64_t>& off = recv ? pr.recv_off : pr.send_off;
  double* base = arena_.as<double>(recv ? "halo_recv" : "halo_send", 1);
  *ptr = base + off[peer];
  *count = off[peer + 1] - off[peer];
}

double Context::ev_ms(int a, int b) {
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, ev_[a], ev_[b]);
  return ms;
}

void Context::load_tables(const std::string& path) {
  Tables t = sdmkb::load_tables(path);
  char key[256];
  double wpar = t.win.kind == kProlate ? t.win.c : t.win.sigma;
  std::snprintf(key, sizeof key, "%d/%d/%d/%.17g/%.17g", t.kernel, t.dim, t.win.kind, wpar, t.table_tol);
  auto it = tables_.find(key);
  if (it != tables_.end())  // replaced in place: drop the residual fits made from the old tables
    for (auto c = pw_cache_.begin(); c != pw_cache_.end();)
      c = c->first.first == &it->second ? pw_cache_.erase(c) : std::next(c);
  tables_[key] = t;
}

const Tables& Context::tables_for(const Plan& P) {
  double tt = P.table_tol > 0.0 ? P.table_tol : std::max(0.03 * P.tol, P.dim == 2 ? 1e-12 : 1e-14);
  double wpar = P.window == kProlate ? P.c : P.sigma;
  char key[256];
  std::snprintf(key, sizeof key, "%d/%d/%d/%.17g/%.17g", P.kernel, P.dim, P.window, wpar, tt);
  auto it = tables_.find(key);
  if (it == tables_.end()) it = tables_.emplace(key, tables_for_plan(P)).first;
  return it->second;
}

void Context::check_inputs(const Plan& P, int dim, int64_t ns, int64_t nt, int mode) {
  if (P.dim != dim) throw InvalidArgument("evaluate: plan and system dimensions differ");
  if (P.kernel != kStokeslet && P.kernel != kStresslet && P.kernel != kRotlet)
    throw InvalidArgument("particle sums support the Stokeslet, stresslet, and rotlet kernels");
  if (dim != 2 && dim != 3) throw InvalidArgument("ParticleSystem: dim must be 2 or 3");
  if (ns < 1) throw InvalidArgument("ParticleSystem: bad source array length");
  if (nt < 0) throw InvalidArgument("ParticleSystem: bad target array length");
  if (ns > (int64_t(1) << 31) - 1 || nt > (int64_t(1) << 31) - 1)
    throw InvalidArgument("evaluate: more than 2^31-1 points");
  if (mode != 0 && mode != 1) throw InvalidArgument("evaluate: bad EwaldMode");
  if (mode == 1 && P.kernel == kStresslet && dim == 2)
    throw InvalidArgument("evaluate: the periodic 2D stresslet sum is not absolutely convergent");
  if (P.n_s < 1) throw InvalidArgument("build_tree: n_s must be >= 1");
  if (P.p < 1) throw InvalidArgument("build_tree: proxy order must be >= 1");
  if (P.p > 64) throw InvalidArgument("evaluate: proxy order above the GPU path limit (64)");
  if (P.N1 < 1 || P.N1 > 127 || P.N_per < 1 || P.N_per > 127)
    throw InvalidArgument("evaluate: Fourier grid size outside [1, 127]");
  if (P.window == kProlate && !(P.c > 0.0)) throw InvalidArgument("build_prolate: c must be positive");
  if (P.window == kGaussian && !(P.sigma > 0.0)) throw InvalidArgument("build_gaussian: sigma must be positive");
}

GridDev& Context::grid(GridDev& gd, const std::string& name, int dim, int p, int N, double theta, double br2) {
  if (gd.key_N == N && gd.key_p == p && gd.key_dim == dim && gd.key_theta == theta && gd.key_band == br2) return gd;
  const int M = (N - 1) / 2, Nz = dim == 3 ? N : 1, Mz = dim == 3 ? M : 0, pz = dim == 3 ? p : 1;
  Cheb1 cb(p);
  // E[m+M][i] = exp(-i theta m s_i)  (dmk.cpp:137-147)
  std::vector<double2> E((size_t)N * p), Ez((size_t)Nz * pz);
  for (int m = -M; m <= M; ++m)
    for (int i = 0; i < p; ++i) {
      double a = -theta * m * cb.x[i];
      E[(size_t)(m + M) * p + i] = make_double2(std::cos(a), std::sin(a));
    }
  if (dim == 3) Ez = E;
  else Ez[0] = make_double2(1.0, 0.0);
  // row limits (dmk.cpp:323-333)
  auto lim = [&](int mz, int my) {
    double rem = br2 - double(mz) * mz - double(my) * my;
    return rem >= 0.0 ? std::min(M, (int)std::floor(std::sqrt(rem))) : -1;
  };
  struct Col {
    int my, m0, lz;
  };
  std::vector<Col> cols;
  for (int m0 = 0; m0 <= M; ++m0)
    for (int my = -M; my <= M; ++my) {
      int lz = -1;
      for (int mz = -Mz; mz <= Mz; ++mz)
        if (lim(mz, my) >= m0) lz = std::max(lz, std::abs(mz));
      if (lz < 0) continue;
      for (int mz = -lz; mz <= lz; ++mz)
        if (lim(mz, my) < m0) throw RuntimeError("plane-wave band is not z-convex");
      cols.push_back({my, m0, lz});
    }
  std::stable_sort(cols.begin(), cols.end(), [](const Col& a, const Col& b) {
    if (a.lz != b.lz) return a.lz > b.lz;
    int ra = a.my * a.my + a.m0 * a.m0, rb = b.my * b.my + b.m0 * b.m0;
    if (ra != rb) return ra < rb;
    if (a.m0 != b.m0) return a.m0 < b.m0;
    return a.my < b.my;
  });
  const int ncol = (int)cols.size();
  std::vector<int> col_my(ncol), col_m0(ncol), col_lz(ncol), slab_ncol(Nz), slab_off(Nz + 1, 0), m0_start(M + 2, 0),
      m0_cols;
  for (int c = 0; c < ncol; ++c) {
    col_my[c] = cols[c].my;
    col_m0[c] = cols[c].m0;
    col_lz[c] = cols[c].lz;
  }
  for (int s = 0; s < Nz; ++s) {
    int mz = s - Mz, cnt = 0;
    for (int c = 0; c < ncol; ++c) cnt += col_lz[c] >= std::abs(mz);
    slab_ncol[s] = cnt;
    slab_off[s + 1] = slab_off[s] + cnt;
  }
  const int nhalf = slab_off[Nz];
  std::vector<int> mode_code(nhalf);
  for (int s = 0; s < Nz; ++s)
    for (int c = 0; c < slab_ncol[s]; ++c) mode_code[slab_off[s] + c] = (s << 16) | c;
  for (int m0 = 0; m0 <= M; ++m0) {
    for (int c = 0; c < ncol; ++c)
      if (col_m0[c] == m0) m0_cols.push_back(c);
    m0_start[m0 + 1] = (int)m0_cols.size();
  }
  Packer pk;
  size_t oE = pk.add(E), oEz = pk.add(Ez), omy = pk.add(col_my), om0 = pk.add(col_m0), olz = pk.add(col_lz),
         oso = pk.add(slab_off), osn = pk.add(slab_ncol), oms = pk.add(m0_start), omc = pk.add(m0_cols),
         omd = pk.add(mode_code);
  char* h = (char*)pinned_.get(name, pk.total);
  for (auto& it : pk.items) std::memcpy(h + it.off, it.src, it.bytes);
  char* d = (char*)arena_.get(name, pk.total);
  cuda_check(cudaMemcpyAsync(d, h, pk.total, cudaMemcpyHostToDevice, st_), "grid upload");
  sync();
  PWGrid& g = gd.g;
  g.N = N;
  g.M = M;
  g.Nz = Nz;
  g.Mz = Mz;
  g.p = p;
  g.pz = pz;
  g.dim = dim;
  g.ncol = ncol;
  g.nhalf = nhalf;
  g.E = (const double2*)(d + oE);
  g.Ez = (const double2*)(d + oEz);
  g.col_my = (const int*)(d + omy);
  g.col_m0 = (const int*)(d + om0);
  g.col_lz = (const int*)(d + olz);
  g.slab_off = (const int*)(d + oso);
  g.slab_ncol = (const int*)(d + osn);
  g.m0_start = (const int*)(d + oms);
  g.m0_cols = (const int*)(d + omc);
  g.mode_code = (const int*)(d + omd);
  gd.key_N = N;
  gd.key_p = p;
  gd.key_dim = dim;
  gd.key_theta = theta;
  gd.key_band = br2;
  gd.col_lz_host = col_lz;
  return gd;
}

// ------------------------------------------------------------ problem ----
void Context::build_problem(const Plan& P, int dim, int ns, int nt, int mode, bool defer_lists) {
  Problem& pr = prob_;
  pr.ready = false;
  pr.plan = P;
  pr.dim = dim;
  pr.periodic = mode == 1;
  pr.nch = channels_out(P.kernel, dim);
  pr.sc = strength_width(P.kernel, dim);
  pr.ns = ns;
  pr.alias = nt == 0;
  pr.nt = pr.alias ? ns : nt;
  const int d = dim;
  double* src = arena_.as<double>("src_in", (size_t)ns * d);
  double* tgt = pr.alias ? nullptr : arena_.as<double>("tgt_in", (size_t)nt * d);
  double* str = arena_.as<double>("str_in", (size_t)ns * pr.sc);
  int* flags = arena_.as<int>("flags", 8);
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  // validate_system (oracle.cpp:103-131) then wrap_into_box (oracle.cpp:133-141)
  // (build_tree itself wraps nothing and accepts only points inside the box, tree.cpp:240-244)
  const int range_free = pr.periodic && !tree_only_;
  launch_validate(src, (int64_t)ns * d, range_free, flags, 0, st_);
  if (tgt) launch_validate(tgt, (int64_t)nt * d, range_free, flags, 0, st_);
  if (!str_pending_) launch_validate(str, (int64_t)ns * pr.sc, 1, flags, 2, st_);
  if (pr.periodic && !tree_only_) {
    launch_wrap(src, (int64_t)ns * d, st_);
    if (tgt) launch_wrap(tgt, (int64_t)nt * d, st_);
  }
  launches_ += 3 + (pr.periodic ? 2 : 0);
  // Morton sort (tree.cpp:258-281)
  // 3D: one 64-bit radix sort on the top 64 of the 90 key bits; exact unless
  // two keys tie there (points within 2^-21 on every axis), which the flags
  // round trip below detects, and then the set is re-sorted on all 90 bits
  auto sort_set = [&](const double* pts, int n, const std::string& tag, int*& perm, double*& soa, int32_t*& q,
                      int tie_flag, bool full) {
    uint64_t* klo = arena_.as<uint64_t>("klo", n);
    uint64_t* khi = arena_.as<uint64_t>("khi", n);
    uint64_t* klo2 = arena_.as<uint64_t>("klo2", n);
    uint64_t* khi2 = arena_.as<uint64_t>("khi2", n);
    int* idx = arena_.as<int>("idx", n);
    int* idx2 = arena_.as<int>("idx2", n);
    perm = arena_.as<int>(tag + "perm", n);
    size_t tb = sort_temp_bytes(n);
    void* tmp = arena_.get("sort_tmp", tb);
    uint64_t* ktop = d == 3 ? arena_.as<uint64_t>("ktop", n) : nullptr;
    launch_morton(pts, n, d, klo, khi, ktop, idx, st_);
    if (d == 3 && !full) {
      sort_morton_top(n, ktop, arena_.as<uint64_t>("ktop2", n), idx, perm, tmp, tb, flags + tie_flag, st_);
      ++launches_;
    } else {
      sort_morton(n, d, klo, khi, idx, klo2, khi2, idx2, perm, tmp, tb, st_);
    }
    soa = arena_.as<double>(tag + "pts", (size_t)n * d);
    q = arena_.as<int32_t>(tag + "q", (size_t)n * d);
    launch_gather_points(pts, perm, n, d, soa, q, st_);
    launches_ += 3;
  };
  int32_t *sq = nullptr, *tq = nullptr;
  sort_set(src, ns, "s", pr.sperm, pr.spts, sq, 4, false);
  pr.sstr = arena_.as<double>("sstr", (size_t)ns * pr.sc);
  // strengths still in flight on the side stream: validated and gathered
  // once the topology is built (finish_strengths)
  auto finish_strengths = [&]() {
    if (str_pending_) {
      cuda_check(cudaStreamWaitEvent(st_, str_ev_, 0), "stream wait");
      cuda_check(cudaMemsetAsync(flags + 2, 0, sizeof(int), st_), "memset");
      launch_validate(str, (int64_t)ns * pr.sc, 1, flags, 2, st_);
      ++launches_;
    }
    launch_gather_strengths(str, pr.sperm, ns, pr.sc, pr.sstr, st_);
    ++launches_;
  };
  if (!str_pending_) finish_strengths();
  if (!pr.alias) {
    sort_set(tgt, nt, "t", pr.tperm, pr.tpts, tq, 5, false);
    pr.tpts_caller = tgt;
  } else {
    pr.tperm = pr.sperm;
    pr.tpts = pr.spts;
    pr.tpts_caller = src;
  }
  // The box topology is built on the host from the GPU-sorted points, which
  // stay on the device: the refine asks the GPU for child boundaries one level
  // at a time; the quantized coordinates come to the host only if the 2:1
  // repair must subdivide a leaf.
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  const auto w0 = std::chrono::steady_clock::now();
  sync();
  const auto w1 = std::chrono::steady_clock::now();
  auto check_strengths = [&]() {  // after finish_strengths: one more flags round trip
    cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
    sync();
    str_pending_ = false;
    if (hflags[2]) throw InvalidArgument("ParticleSystem: non-finite strength");
  };
  if (str_pending_ && (hflags[0] || hflags[1])) {  // the reference checks strengths first (oracle.cpp:116-118)
    finish_strengths();
    check_strengths();
  }
  if (tree_only_ && (hflags[0] || hflags[1])) throw InvalidArgument("build_tree: point outside the unit box");
  if (hflags[2]) throw InvalidArgument("ParticleSystem: non-finite strength");
  if (hflags[0]) throw InvalidArgument("ParticleSystem: non-finite coordinate");
  if (hflags[1]) throw InvalidArgument("ParticleSystem: coordinate outside the unit box");
  if (hflags[4] || hflags[5]) {  // ties in the top 64 key bits: re-sort on all 90
    if (hflags[4]) {
      sort_set(src, ns, "s", pr.sperm, pr.spts, sq, 4, true);
      if (!str_pending_) finish_strengths();  // gathered with the first permutation
    }
    if (!pr.alias && hflags[5]) sort_set(tgt, nt, "t", pr.tperm, pr.tpts, tq, 5, true);
    if (pr.alias) {
      pr.tperm = pr.sperm;
      pr.tpts = pr.spts;
    }
  }
  pr.sq = sq;
  pr.tq = tq;
  hq_ = nullptr;
  PointAccess pa;
  pa.split = [&](int n, const int* lvl, const int* srng, const int* trng, int* sbnd, int* tbnd) {
    const size_t in_bytes = sizeof(int) * (size_t)n * 5, out_bytes = sizeof(int) * (size_t)n * 18;
    int* h = (int*)pinned_.get("split", in_bytes + out_bytes + 256);
    std::memcpy(h, lvl, sizeof(int) * n);
    std::memcpy(h + n, srng, sizeof(int) * 2 * n);
    std::memcpy(h + 3 * n, trng, sizeof(int) * 2 * n);
    int* dvb = (int*)arena_.get("split", in_bytes + out_bytes + 256);
    cuda_check(cudaMemcpyAsync(dvb, h, in_bytes, cudaMemcpyHostToDevice, st_), "split upload");
    int* dout = dvb + 5 * n;
    launch_split_ranges(n, dvb, dvb + n, sq, ns, d, dout, st_);
    if (!pr.alias) launch_split_ranges(n, dvb, dvb + 3 * n, tq, nt, d, dout + 9 * n, st_);
    launches_ += pr.alias ? 1 : 2;
    int* hout = h + 5 * n;
    cuda_check(cudaMemcpyAsync(hout, dout, sizeof(int) * (size_t)n * (pr.alias ? 9 : 18), cudaMemcpyDeviceToHost, st_),
               "split download");
    sync();
    std::memcpy(sbnd, hout, sizeof(int) * (size_t)n * 9);
    if (!pr.alias) std::memcpy(tbnd, hout + 9 * n, sizeof(int) * (size_t)n * 9);
  };
  pa.host_q = [&](const int32_t** qs_out, const int32_t** qt_out) {
    int32_t* hq = (int32_t*)pinned_.get("hq", sizeof(int32_t) * ((size_t)ns + (pr.alias ? 0 : nt)) * d + 64);
    cuda_check(cudaMemcpyAsync(hq, sq, sizeof(int32_t) * (size_t)ns * d, cudaMemcpyDeviceToHost, st_), "D2H q");
    if (!pr.alias)
      cuda_check(
          cudaMemcpyAsync(hq + (size_t)ns * d, tq, sizeof(int32_t) * (size_t)nt * d, cudaMemcpyDeviceToHost, st_),
          "D2H q");
    sync();
    hq_ = hq;
    *qs_out = hq;
    *qt_out = pr.alias ? nullptr : hq + (size_t)ns * d;
  };
  // refine_to_capacity in one cooperative launch; the boxes come back in the
  // reference's id order (the host keeps the 2:1 repair and the lists)
  static_assert(sizeof(RefBox) == sizeof(Box) && offsetof(RefBox, leaf) == offsetof(Box, leaf) &&
                    offsetof(RefBox, anchor) == offsetof(Box, anchor) && offsetof(RefBox, sb) == offsetof(Box, sb) &&
                    offsetof(RefBox, te) == offsetof(Box, te),
                "RefBox mirrors host/tree.hpp Box");
  static const bool host_refine = std::getenv("SDMK_HOST_REFINE") != nullptr;  // A/B and fallback tests
  if (!host_refine)
    pa.refine = [&](std::vector<Box>& boxes, int& max_level, bool& capped) {
      const int nchild = 1 << d;
      const int64_t want = 8 * (int64_t)nchild * ((int64_t)ns / std::max(1, P.n_s) + 1) + 4096;
      static const char* cap_env = std::getenv("SDMK_REFINE_CAP");  // test hook: force the fallback
      const int cap = cap_env ? std::max(16, std::atoi(cap_env)) : (int)std::min<int64_t>(want, int64_t(1) << 26);
      void* nodes = arena_.get("refine_nodes", (size_t)cap * refine_node_bytes());
      RefBox* out = (RefBox*)arena_.get("refine_out", (size_t)cap * sizeof(RefBox));
      int* hdr = arena_.as<int>("refine_hdr", 64);
      if (!launch_refine(sq, ns, pr.alias ? nullptr : tq, pr.alias ? 0 : nt, pr.alias ? 1 : 0, d, P.n_s, cap, nodes,
                         hdr, out, st_))
        return false;
      ++launches_;
      int* hh = (int*)pinned_.get("refine_hdr", 64 * sizeof(int));
      cuda_check(cudaMemcpyAsync(hh, hdr, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H refine header");
      sync();
      if (hh[3]) return false;  // more boxes than slots: the host refines
      const int nb = hh[0];
      Box* hb = (Box*)pinned_.get("refine_out", (size_t)nb * sizeof(Box));
      cuda_check(cudaMemcpyAsync(hb, out, (size_t)nb * sizeof(Box), cudaMemcpyDeviceToHost, st_), "D2H boxes");
      sync();
      boxes.reserve((size_t)nb + nb / 4 + 64);  // room for the 2:1 repair's boxes
      boxes.resize(nb);
      std::memcpy((void*)boxes.data(), hb, (size_t)nb * sizeof(Box));
      max_level = hh[1] - 1;
      capped = hh[2] != 0;
      return true;
    };
  if (!host_refine)
    pa.repair_scan = [&](int nb, uint32_t* cand) {
      uint32_t* dc = arena_.as<uint32_t>("repair_cand", (size_t)nb);
      launch_repair_scan((const RefBox*)arena_.get("refine_out", 1), nb, d, pr.periodic ? 1 : 0, dc, st_);
      ++launches_;
      uint32_t* hc = (uint32_t*)pinned_.get("repair_cand", (size_t)nb * sizeof(uint32_t));
      cuda_check(cudaMemcpyAsync(hc, dc, (size_t)nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_),
                 "D2H repair candidates");
      sync();
      std::memcpy(cand, hc, (size_t)nb * sizeof(uint32_t));
    };
  pr.tree = build_topology(d, pr.periodic, P.n_s, P.p, ns, pr.alias ? 0 : nt, pa, /*with_neighbours=*/false);
  if (str_pending_) {
    finish_strengths();
    check_strengths();
  }
  const auto w2 = std::chrono::steady_clock::now();
  pr.lists_b = false;
  upload_tree_lists_a();
  if (!defer_lists) upload_tree_lists_b();
  const auto w3 = std::chrono::steady_clock::now();
  if (timing_on()) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[sdmk timing] sort+D2H wait %.2f ms, host topology %.2f ms, lists+upload %.2f ms (%d boxes)\n",
                 ms(w0, w1), ms(w1, w2), ms(w2, w3), pr.tree.num_boxes());
  }
  pr.ready = true;
}

// Sibling groups for k_acc_group: consecutive plane-wave targets with one
// parent.  Each colleague entry (slot, tau) of child c sits at the
// parent-relative position c + tau in {-1..2}^d; the group kernel sums every
// position inside child c's 3^d window, so the level is grouped only when
// those windows reproduce each target's entry list exactly (one slot per
// position, no repeats, the leaf's own position the only one skipped).
// Otherwise the lists are left empty and the level stays per-target.
static void build_groups(const HostTree& t, int lev, const std::vector<int>& tbx, const std::vector<int>& es,
                         const std::vector<int>& eslot, const std::vector<int>& etau, std::vector<int>& gstart,
                         std::vector<int>& gslot, std::vector<int>& tmeta) {
  const int d = t.dim, ntg = (int)tbx.size();
  if (ntg == 0) return;
  const int64_t side_int = int64_t(1) << (30 - lev);
  for (int i = 0; i < ntg; ++i)
    if (i == 0 || t.boxes[tbx[i]].parent != t.boxes[tbx[i - 1]].parent) gstart.push_back(i);
  gstart.push_back(ntg);
  const int ng = (int)gstart.size() - 1;
  gslot.assign((size_t)ng * 64, -1);
  tmeta.assign(ntg, 0);
  auto pcode = [&](int x, int y, int z) { return (x + 1) + 4 * (y + 1) + 16 * (d == 3 ? z + 1 : 1); };
  uint64_t window[8];
  for (int c = 0; c < (1 << d); ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = d == 3 ? (c >> 2) & 1 : 0;
    uint64_t m = 0;
    for (int z = (d == 3 ? -1 : 0); z <= (d == 3 ? 1 : 0); ++z)
      for (int y = -1; y <= 1; ++y)
        for (int x = -1; x <= 1; ++x) m |= uint64_t(1) << pcode(cx + x, cy + y, cz + z);
    window[c] = m;
  }
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(min : ok)
  for (int gi = 0; gi < ng; ++gi) {
    const int i0 = gstart[gi], i1 = gstart[gi + 1];
    const Box& P = t.boxes[t.boxes[tbx[i0]].parent];
    int* slot = gslot.data() + (size_t)gi * 64;
    uint64_t emask[8], umask = 0;
    int cc[8];
    bool good = i1 - i0 <= (1 << d);
    for (int i = i0; i < i1 && good; ++i) {
      const Box& B = t.boxes[tbx[i]];
      int c = 0;
      for (int ax = 0; ax < d; ++ax) {
        const int64_t diff = int64_t(B.anchor[ax]) - int64_t(P.anchor[ax]);
        if (diff != 0 && diff != side_int) good = false;
        c |= (diff == side_int) << ax;
      }
      const int k = i - i0;
      cc[k] = c;
      emask[k] = 0;
      for (int e = es[i]; e < es[i + 1]; ++e) {
        const int code = etau[e];
        const int pc = pcode((c & 1) + code % 3 - 1, ((c >> 1) & 1) + (code / 3) % 3 - 1,
                             ((c >> 2) & 1) + code / 9 - 1);
        if ((emask[k] >> pc) & 1) good = false;
        emask[k] |= uint64_t(1) << pc;
        if (slot[pc] == -1) slot[pc] = eslot[e];
        else if (slot[pc] != eslot[e]) good = false;
      }
      umask |= emask[k];
    }
    for (int i = i0; i < i1 && good; ++i) {
      const int k = i - i0, c = cc[k];
      const uint64_t self = uint64_t(1) << pcode(c & 1, (c >> 1) & 1, (c >> 2) & 1);
      uint64_t expect = window[c] & umask;
      const bool sub = t.boxes[tbx[i]].leaf && (umask & self);
      if (sub) expect &= ~self;
      if (expect != emask[k]) good = false;
      tmeta[i] = c | (sub ? 8 : 0);
    }
    if (!good) ok = 0;
  }
  if (!ok) {
    gstart.clear();
    gslot.clear();
    tmeta.clear();
  }
}

// Phase A: what the upward pass needs (box records, anterpolation leaves,
// merge lists, Chebyshev matrices).  Phase B: everything the downward,
// far-field and residual passes need; evaluate() builds it on the host while
// the GPU runs the upward pass.
void Context::upload_tree_lists_a() {
  Problem& pr = prob_;
  const HostTree& t = pr.tree;
  const int nb = t.num_boxes(), d = pr.dim, nchild = 1 << d;
  std::vector<dev::DBox> boxes(nb);
#pragma omp parallel for schedule(static)
  for (int b = 0; b < nb; ++b) {
    const Box& x = t.boxes[b];
    dev::DBox& o = boxes[b];
    o.sb = x.sb;
    o.se = x.se;
    o.tb = x.tb;
    o.te = x.te;
    o.level = x.level;
    o.parent = x.parent;
    o.first_child = x.first_child;
    o.leaf = x.leaf;
    auto c = t.center(b);
    o.c[0] = c[0];
    o.c[1] = c[1];
    o.c[2] = c[2];
    o.side = t.side(b);
    o.half = 0.5 * o.side;
  }
  // halo mode: this rank anterpolates and merges its own cut subtrees; the
  // boxes above the cut are merged after the exchange (top lists)
  pr.halo = halo_run_;
  if (pr.halo) pr.hp = halo_owners(t, nranks_);
  else pr.hp = HaloPlan{};
  auto mine = [&](int b) { return !pr.halo || pr.hp.owner[b] == rank_; };
  std::vector<int> ant;
  for (int b = 0; b < nb; ++b)
    if (t.boxes[b].leaf && t.nsrc(b) > 0 && mine(b)) ant.push_back(b);
  const int L = t.max_level + 1;
  std::vector<std::vector<int>> m_out(L), m_in(L), m_ci(L), u_out(L), u_in(L), u_ci(L);
  for (int lev = 0; lev < L; ++lev)
    for (int b : t.level_boxes[lev]) {
      const Box& x = t.boxes[b];
      if (!x.leaf && t.nsrc(b) > 0 && (mine(b) || pr.hp.owner[b] == -1)) {  // upward merge (dmk.cpp:638-651)
        const bool top = !mine(b);
        (top ? u_out : m_out)[lev].push_back(b);
        for (int ci = 0; ci < nchild; ++ci) {
          int c = x.first_child + ci;
          (top ? u_in : m_in)[lev].push_back(t.nsrc(c) > 0 ? c : -1);
          (top ? u_ci : m_ci)[lev].push_back(ci);
        }
      }
    }
  // Chebyshev nodes/weights and the child matrices (dmk.cpp:25-66, 626-629)
  const int p = pr.plan.p;
  Cheb1 cb(p);
  std::vector<double> m0 = cb.child(0), m1 = cb.child(1), t0 = transpose(m0, p), t1 = transpose(m1, p);
  std::vector<double> blob;
  blob.insert(blob.end(), cb.x.begin(), cb.x.end());
  blob.insert(blob.end(), cb.w.begin(), cb.w.end());
  blob.insert(blob.end(), t0.begin(), t0.end());  // upward: transposed child matrices
  blob.insert(blob.end(), t1.begin(), t1.end());
  blob.insert(blob.end(), m0.begin(), m0.end());  // downward: child matrices
  blob.insert(blob.end(), m1.begin(), m1.end());
  Packer pk;
  const size_t o_blob = pk.add(blob), o_boxes = pk.add(boxes), o_ant = pk.add(ant);
  std::vector<std::array<size_t, 6>> off(L);
  for (int lev = 0; lev < L; ++lev)
    off[lev] = {pk.add(m_out[lev]), pk.add(m_in[lev]), pk.add(m_ci[lev]),
                pk.add(u_out[lev]), pk.add(u_in[lev]), pk.add(u_ci[lev])};
  char* h = (char*)pinned_.get("treeA", pk.total + 64);
  pk.copy_to(h);
  char* dv = (char*)arena_.get("treeA", pk.total + 64);
  cuda_check(cudaMemcpyAsync(dv, h, pk.total, cudaMemcpyHostToDevice, st_), "tree upload");
  const double* db = (const double*)(dv + o_blob);
  cheb_nodes_ = db;
  cheb_wts_ = db + p;
  mats_up_ = db + 2 * p;
  mats_down_ = db + 2 * p + 2 * p * p;
  pr.boxes = (dev::DBox*)(dv + o_boxes);
  pr.ant_leaves = (int*)(dv + o_ant);
  pr.n_ant = (int)ant.size();
  pr.levels.assign(L, {});
  for (int lev = 0; lev < L; ++lev) {
    Problem::LevelLists& X = pr.levels[lev];
    X.n_merge = (int)m_out[lev].size();
    X.merge_out = (int*)(dv + off[lev][0]);
    X.merge_in = (int*)(dv + off[lev][1]);
    X.merge_ci = (int*)(dv + off[lev][2]);
    X.n_top = (int)u_out[lev].size();
    X.top_out = (int*)(dv + off[lev][3]);
    X.top_in = (int*)(dv + off[lev][4]);
    X.top_ci = (int*)(dv + off[lev][5]);
  }
}

void Context::upload_tree_lists_b() {
  Problem& pr = prob_;
  const auto hb0 = std::chrono::steady_clock::now();
  finish_topology(pr.tree);  // neighbour lists (tree.cpp:167-212), while the GPU runs the upward pass
  const auto hb1 = std::chrono::steady_clock::now();
  const HostTree& t = pr.tree;
  const int nb = t.num_boxes(), d = pr.dim, nchild = 1 << d;
  // target ownership (one rank owns everything unless set_shard was called):
  // the downward, far-field and residual work is restricted to the owned
  // target leaves and their ancestors
  ShardCosts costs;
  if (nranks_ > 1) costs = shard_costs(t);
  ShardPlan sp = shard_plan(t, rank_, nranks_, nranks_ > 1 ? &costs : nullptr);
  const std::vector<int>& itp = sp.leaves;
  const std::vector<char>& need = sp.need;
  // halo mode: what this rank reads, and the exchange lists
  std::vector<int> send_ids, recv_ids;
  if (pr.halo) {
    halo_reads(t, pr.hp, &costs);
    const int64_t elems = (int64_t)pr.nch * (d == 3 ? pr.plan.p : 1) * pr.plan.p * pr.plan.p;
    pr.send_off.assign(nranks_ + 1, 0);
    pr.recv_off.assign(nranks_ + 1, 0);
    // one pass over the boxes (= halo_boxes(rank, q) and halo_boxes(q, rank)
    // for every peer q, each in increasing box order)
    std::vector<std::vector<int>> sv(nranks_), rv(nranks_);
    const uint64_t me = uint64_t(1) << rank_, all = nranks_ >= 64 ? ~uint64_t(0) : (uint64_t(1) << nranks_) - 1;
    for (int b = 0; b < nb; ++b) {
      const int o = pr.hp.owner[b];
      if (o < 0) continue;
      const uint64_t rd = pr.hp.cut[b] ? all : pr.hp.readmask[b];
      if (o == rank_) {
        for (uint64_t m = rd & ~me; m; m &= m - 1) sv[__builtin_ctzll(m)].push_back(b);
      } else if (rd & me) {
        rv[o].push_back(b);
      }
    }
    for (int q = 0; q < nranks_; ++q) {
      send_ids.insert(send_ids.end(), sv[q].begin(), sv[q].end());
      recv_ids.insert(recv_ids.end(), rv[q].begin(), rv[q].end());
      pr.send_off[q + 1] = (int64_t)send_ids.size() * elems;
      pr.recv_off[q + 1] = (int64_t)recv_ids.size() * elems;
    }
  }
  auto reads = [&](int b) { return !pr.halo || ((pr.hp.readmask[b] >> rank_) & 1); };
  const auto hb2 = std::chrono::steady_clock::now();
  pr.t_own0 = sp.t0;
  pr.t_own1 = sp.t1;
  pr.t_bounds.clear();
  if (nranks_ > 1 && comm_) {
    pr.t_bounds = shard_bounds(t, nranks_, costs);
    if (pr.t_bounds[rank_] != sp.t0 || pr.t_bounds[rank_ + 1] != sp.t1)
      throw RuntimeError("shard bounds disagree with the shard plan");
    int64_t* hb = (int64_t*)pinned_.get("t_bounds", sizeof(int64_t) * (nranks_ + 1));
    std::copy(pr.t_bounds.begin(), pr.t_bounds.end(), hb);
    pr.d_bounds = arena_.as<int64_t>("t_bounds", nranks_ + 1);
    cuda_check(cudaMemcpyAsync(pr.d_bounds, hb, sizeof(int64_t) * (nranks_ + 1), cudaMemcpyHostToDevice, st_),
               "bounds upload");
  }
  // near ranges per target leaf (dmk.cpp:966-990); two-pass CSR, parallel over leaves
  auto scode = [](const int8_t* s) { return (s[0] + 1) + 3 * (s[1] + 1) + 9 * (s[2] + 1); };
  auto ranges = [&](int b, int* obox, int* oinfo) {
    int n = 0;
    auto add = [&](int sbx, const int8_t* sh, bool fine_scale, bool self) {
      if (t.nsrc(sbx) == 0) return;
      if (obox) {
        obox[n] = sbx;
        oinfo[n] = scode(sh) | (fine_scale ? 32 : 0) | (self ? 64 : 0);
      }
      ++n;
    };
    const int8_t zero[3] = {0, 0, 0};
    add(b, zero, false, true);
    for (const Nbr& e : t.col[b]) {
      if (e.box == b && !e.shift[0] && !e.shift[1] && !e.shift[2]) continue;
      if (!t.boxes[e.box].leaf) continue;
      add(e.box, e.shift, true, false);
    }
    for (const Nbr& e : t.crs[b]) add(e.box, e.shift, false, false);
    for (const Nbr& e : t.fin[b]) add(e.box, e.shift, true, false);
    return n;
  };
  const int nitp = (int)itp.size();
  std::vector<int> rs(nitp + 1, 0);
  int max_ranges = 0;
#pragma omp parallel for schedule(static) reduction(max : max_ranges)
  for (int i = 0; i < nitp; ++i) {
    rs[i + 1] = ranges(itp[i], nullptr, nullptr);
    max_ranges = std::max(max_ranges, rs[i + 1]);
  }
  if (max_ranges > 160) throw RuntimeError("residual pass: more than 160 near ranges for one leaf");
  for (int i = 0; i < nitp; ++i) rs[i + 1] += rs[i];
  std::vector<int> rbox(rs[nitp]), rinfo(rs[nitp]);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nitp; ++i) ranges(itp[i], rbox.data() + rs[i], rinfo.data() + rs[i]);
  const auto hb3 = std::chrono::steady_clock::now();
  double t_groups = 0.0, t_entries = 0.0;
  // per-level lists
  const int L = t.max_level + 1;
  struct LV {
    std::vector<int> i_in, i_out, i_ci, i_seg, sbx, tbx, es, eslot, etau, gstart, gslot, tmeta;
  };
  std::vector<LV> lv(L);
  std::vector<int> gslot(nb, -1);
  bool bad_tau = false;
  for (int lev = 0; lev < L; ++lev) {
    LV& V = lv[lev];
    for (int b : t.level_boxes[lev]) {
      const Box& x = t.boxes[b];
      if (!x.leaf && t.ntgt(b) > 0) {  // downward interpolation (dmk.cpp:840-853)
        const int first = (int)V.i_in.size();
        for (int ci = 0; ci < nchild; ++ci) {
          int c = x.first_child + ci;
          if (t.ntgt(c) == 0 || !need[c]) continue;
          V.i_in.push_back(b);
          V.i_out.push_back(c);
          V.i_ci.push_back(ci);
        }
        if ((int)V.i_in.size() > first) V.i_seg.push_back(first);  // this parent's pairs
      }
      if (t.nsrc(b) > 0 && reads(b)) {  // forward transforms of the boxes this rank reads
        gslot[b] = (int)V.sbx.size();
        V.sbx.push_back(b);
      }
    }
    // plane-wave targets and their colleague entries (dmk.cpp:760-797); two-pass, parallel
    const int64_t side_int = int64_t(1) << (30 - lev);
    const std::vector<int>& ids = t.level_boxes[lev];
    const int nl = (int)ids.size();
    // a plane-wave target is kept with all its siblings (need of the parent), so
    // the sibling groups -- and every target's sums -- match the unsharded run
    auto entries = [&](int b, int* oslot, int* otau) {
      const int par = t.boxes[b].parent;
      if (t.ntgt(b) == 0 || !need[par >= 0 ? par : b]) return 0;
      int cnt = 0;
      for (const Nbr& ce : t.col[b]) {
        if (t.boxes[b].leaf && ce.box == b && !ce.shift[0] && !ce.shift[1] && !ce.shift[2]) continue;
        if (t.nsrc(ce.box) == 0) continue;
        if (oslot) {
          int tau[3] = {0, 0, 0};
          for (int ax = 0; ax < d; ++ax) {
            int64_t diff = int64_t(t.boxes[ce.box].anchor[ax]) + (int64_t(ce.shift[ax]) << 30) -
                           int64_t(t.boxes[b].anchor[ax]);
            tau[ax] = int(diff / side_int);
            if (tau[ax] < -1 || tau[ax] > 1) bad_tau = true;
          }
          oslot[cnt] = gslot[ce.box];
          otau[cnt] = (tau[0] + 1) + 3 * (tau[1] + 1) + 9 * (tau[2] + 1);
        }
        ++cnt;
      }
      return cnt;
    };
    const auto he0 = std::chrono::steady_clock::now();
    std::vector<int> cnt(nl);
    int max_e = 0;
#pragma omp parallel for schedule(static) reduction(max : max_e)
    for (int i = 0; i < nl; ++i) {
      cnt[i] = entries(ids[i], nullptr, nullptr);
      max_e = std::max(max_e, cnt[i]);
    }
    if (max_e > 64) throw RuntimeError("plane-wave pass: more than 64 colleague entries");
    std::vector<int> eoff(nl + 1, 0);
    V.es.push_back(0);
    for (int i = 0; i < nl; ++i) {
      eoff[i + 1] = eoff[i] + cnt[i];
      if (cnt[i] > 0) {
        V.tbx.push_back(ids[i]);
        V.es.push_back(eoff[i + 1]);
      }
    }
    V.eslot.resize(eoff[nl]);
    V.etau.resize(eoff[nl]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < nl; ++i)
      if (cnt[i] > 0) entries(ids[i], V.eslot.data() + eoff[i], V.etau.data() + eoff[i]);
    const auto he1 = std::chrono::steady_clock::now();
    if (lev > 0) build_groups(t, lev, V.tbx, V.es, V.eslot, V.etau, V.gstart, V.gslot, V.tmeta);
    const auto he2 = std::chrono::steady_clock::now();
    t_entries += std::chrono::duration<double, std::milli>(he1 - he0).count();
    t_groups += std::chrono::duration<double, std::milli>(he2 - he1).count();
  }
  const auto hb4 = std::chrono::steady_clock::now();
  if (bad_tau) throw RuntimeError("colleague offset outside {-1,0,1}");
  // root lists: box 0 with one zero-offset entry
  std::vector<int> root_ids = {0}, root_es = {0, 1}, root_slot = {0}, root_tau = {13};
  // residual work items: 32-target chunks of each target leaf, in leaf order
  std::vector<int> coff(nitp + 1, 0);
  for (int i = 0; i < nitp; ++i) coff[i + 1] = coff[i] + (t.ntgt(itp[i]) + 31) / 32;
  std::vector<int> chunks(2 * (size_t)coff[nitp]);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nitp; ++i) {
    const Box& x = t.boxes[itp[i]];
    int* o = chunks.data() + 2 * (size_t)coff[i];
    for (int t0 = x.tb; t0 < x.te; t0 += 32, o += 2) {
      o[0] = i;
      o[1] = t0;
    }
  }
  Packer pk;
  size_t o_chunks = pk.add(chunks), o_send = pk.add(send_ids), o_recv = pk.add(recv_ids);
  size_t o_itp = pk.add(itp), o_rs = pk.add(rs), o_rbox = pk.add(rbox), o_rinfo = pk.add(rinfo),
         o_rid = pk.add(root_ids), o_res = pk.add(root_es), o_rsl = pk.add(root_slot), o_rta = pk.add(root_tau);
  struct Off {
    size_t i_in, i_out, i_ci, i_seg, sbx, tbx, es, eslot, etau, gstart, gslot, tmeta;
  };
  std::vector<Off> off(L);
  for (int lev = 0; lev < L; ++lev) {
    LV& V = lv[lev];
    V.i_seg.push_back((int)V.i_in.size());
    off[lev] = {pk.add(V.i_in),  pk.add(V.i_out),  pk.add(V.i_ci),   pk.add(V.i_seg),
                pk.add(V.sbx),   pk.add(V.tbx),    pk.add(V.es),     pk.add(V.eslot),
                pk.add(V.etau),  pk.add(V.gstart), pk.add(V.gslot),  pk.add(V.tmeta)};
  }
  const auto hb5 = std::chrono::steady_clock::now();
  char* h = (char*)pinned_.get("treeB", pk.total + 64);
  pk.copy_to(h);
  const auto hb6 = std::chrono::steady_clock::now();
  char* dv = (char*)arena_.get("treeB", pk.total + 64);
  // inside an evaluation the upward pass is running on st_: the upload and the
  // sub-cell kernel go to the second stream (ordered after the tree build) and
  // st_ picks them up by an event, so they do not queue behind the upward pass
  cudaStream_t su = lists_side_ ? st2_ : st_;
  if (lists_side_) cuda_check(cudaStreamWaitEvent(st2_, ev_[2], 0), "stream wait");
  cuda_check(cudaMemcpyAsync(dv, h, pk.total, cudaMemcpyHostToDevice, su), "tree upload");
  pr.send_ids = (int*)(dv + o_send);
  pr.recv_ids = (int*)(dv + o_recv);
  pr.n_send = (int)send_ids.size();
  pr.n_recv = (int)recv_ids.size();
  pr.int_leaves = (int*)(dv + o_itp);
  pr.n_int = (int)itp.size();
  pr.rng_start = (int*)(dv + o_rs);
  pr.rng_box = (int*)(dv + o_rbox);
  pr.rng_info = (int*)(dv + o_rinfo);
  // source sub-cells for the residual cull, from the device-resident points
  pr.subrange = arena_.as<int>("subrange", (size_t)nb * 9);
  launch_leaf_subranges(pr.boxes, nb, pr.sq, pr.ns, d, pr.subrange, su);
  ++launches_;
  if (lists_side_) {
    cuda_check(cudaEventRecord(x_ev_, st2_), "event record");
    cuda_check(cudaStreamWaitEvent(st_, x_ev_, 0), "stream wait");
  }
  pr.res_chunks = (int*)(dv + o_chunks);
  pr.n_chunks = (int)(chunks.size() / 2);
  for (int lev = 0; lev < L; ++lev) {
    Problem::LevelLists& X = pr.levels[lev];
    LV& V = lv[lev];
    X.n_interp = (int)V.i_out.size();
    X.n_src = (int)V.sbx.size();
    X.n_tgt = (int)V.tbx.size();
    X.interp_in = (int*)(dv + off[lev].i_in);
    X.interp_out = (int*)(dv + off[lev].i_out);
    X.interp_ci = (int*)(dv + off[lev].i_ci);
    X.interp_seg = (int*)(dv + off[lev].i_seg);
    X.n_interp_seg = (int)V.i_seg.size() - 1;
    X.src_boxes = (int*)(dv + off[lev].sbx);
    X.tgt_boxes = (int*)(dv + off[lev].tbx);
    X.ent_start = (int*)(dv + off[lev].es);
    X.ent_slot = (int*)(dv + off[lev].eslot);
    X.ent_tau = (int*)(dv + off[lev].etau);
    X.grp_start_h = V.gstart;
    X.grp_tstart = (int*)(dv + off[lev].gstart);
    X.grp_slot = (int*)(dv + off[lev].gslot);
    X.t_meta = (int*)(dv + off[lev].tmeta);
  }
  root_dev_ids_ = (int*)(dv + o_rid);
  root_dev_es_ = (int*)(dv + o_res);
  root_dev_slot_ = (int*)(dv + o_rsl);
  root_dev_tau_ = (int*)(dv + o_rta);
  pr.lists_b = true;
  if (timing_on()) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[sdmk timing] lists B (host, overlaps the upward pass): neighbours %.2f ms, shard+halo plan %.2f ms, lists+upload %.2f ms\n",
                 ms(hb0, hb1), ms(hb1, hb2), ms(hb2, std::chrono::steady_clock::now()));
    std::fprintf(stderr, "[sdmk timing]   ranges %.2f, level lists %.2f (entries %.2f, groups %.2f), chunks+pack %.2f, copy to pinned %.2f (%.1f MB), rest %.2f ms\n",
                 ms(hb2, hb3), ms(hb3, hb4), t_entries, t_groups, ms(hb4, hb5), ms(hb5, hb6), pk.total / 1e6,
                 ms(hb6, std::chrono::steady_clock::now()));
  }
}

// ---------------------------------------------------------------- passes --
void Context::run_upward() {  // dmk.cpp:555-655
  Problem& pr = prob_;
  const int d = pr.dim, p = pr.plan.p, pz = d == 3 ? p : 1;
  const size_t nodes = (size_t)pz * p * p;
  const int nb = pr.tree.num_boxes();
  double* og = arena_.as<double>("outgoing", (size_t)nb * pr.nch * nodes);
  // outgoing of a box without sources is never read (forward transforms and
  // merges skip them), so evaluate() skips the 10 GB-scale memset; the
  // pass-level API returns whole arrays and keeps the reference's zeros
  if (zero_all_) cuda_check(cudaMemsetAsync(og, 0, sizeof(double) * nb * pr.nch * nodes, st_), "memset outgoing");
  ChebDev cb{p, pz, d, cheb_nodes_, cheb_wts_};
  if (mma_anterp_supported(p)) {
    double* basis = arena_.as<double>("basis_s", (size_t)3 * pr.ns * p);
    launch_basis(cb, pr.boxes, pr.ant_leaves, pr.n_ant, pr.spts, pr.ns, 0, basis, st_);
    cudaEventRecord(ev_[18], st_);
    launch_anterp_mma(pr.plan.kernel, cb, pr.boxes, pr.ant_leaves, pr.n_ant, basis, pr.sstr, pr.ns, og, pr.nch, st_);
    cudaEventRecord(ev_[19], st_);
    anterp_timed_ = true;
    launches_ += 2;
  } else {
    launch_anterp(pr.plan.kernel, cb, pr.boxes, pr.ant_leaves, pr.n_ant, pr.spts, pr.ns, pr.sstr, og, pr.nch, st_);
    ++launches_;
  }
  for (int lev = pr.tree.max_level - 1; lev >= 0; --lev) {
    const Problem::LevelLists& X = pr.levels[lev];
    if (X.n_merge == 0) continue;
    if (tensor_mma_supported(p, d))
      launch_tensor_mma(p, mats_up_, X.merge_in, X.merge_out, X.merge_ci, X.n_merge, pr.nch, og, og, 2, d, st_);
    else
      launch_tensor_apply(p, pz, d, mats_up_, X.merge_in, X.merge_out, X.merge_ci, X.n_merge, pr.nch, og, og, 2, st_);
    ++launches_;
  }
  cuda_check(cudaPeekAtLastError(), "kernel launch");
}

// Halo mode: the boxes above the cut, from the gathered cut boxes (the same
// per-parent merge as run_upward, so every rank forms them bit for bit alike).
void Context::run_upward_top() {
  Problem& pr = prob_;
  const int d = pr.dim, p = pr.plan.p, pz = d == 3 ? p : 1;
  double* og = arena_.as<double>("outgoing", 1);
  for (int lev = pr.tree.max_level - 1; lev >= 0; --lev) {
    const Problem::LevelLists& X = pr.levels[lev];
    if (X.n_top == 0) continue;
    if (tensor_mma_supported(p, d))
      launch_tensor_mma(p, mats_up_, X.top_in, X.top_out, X.top_ci, X.n_top, pr.nch, og, og, 2, d, st_);
    else
      launch_tensor_apply(p, pz, d, mats_up_, X.top_in, X.top_out, X.top_ci, X.n_top, pr.nch, og, og, 2, st_);
    ++launches_;
  }
  cuda_check(cudaPeekAtLastError(), "kernel launch");
}

void Context::run_root() {  // dmk.cpp:657-701
  Problem& pr = prob_;
  const Plan& P = pr.plan;
  const int d = pr.dim, p = P.p, pz = d == 3 ? p : 1;
  const size_t nodes = (size_t)pz * p * p;
  const int nb = pr.tree.num_boxes();
  double* in = arena_.as<double>("incoming", (size_t)nb * d * nodes);
  // every non-root box with targets is first written by its parent's
  // interpolation (DMMA path, write mode), so only the root needs zeros
  // unless whole arrays are returned or the FFMA fallback accumulates
  if (zero_all_ || !tensor_mma_supported(p, d))
    cuda_check(cudaMemsetAsync(in, 0, sizeof(double) * nb * d * nodes, st_), "memset incoming");
  else
    cuda_check(cudaMemsetAsync(in, 0, sizeof(double) * d * nodes, st_), "memset incoming");
  const int N = pr.periodic ? P.N_per : P.N1;
  const double h = pr.periodic ? 2.0 * PI : PI / 3.0;
  const int M = (N - 1) / 2;
  GridDev& gd = grid(grid_root_, "grid_root", d, p, N, 0.5 * h, band_r2(P, M, h));
  const PWGrid& g = gd.g;
  std::vector<double> A = symbol_table(*tab_, h, 3 * M * M, pr.periodic ? kRootPeriodic : kRootFree, 1.0, 1.0);
  double* hA = (double*)pinned_.get("symroot", A.size() * sizeof(double));
  std::memcpy(hA, A.data(), A.size() * sizeof(double));
  double* dA = arena_.as<double>("symroot", A.size());
  cuda_check(cudaMemcpyAsync(dA, hA, A.size() * sizeof(double), cudaMemcpyHostToDevice, st_), "symbol upload");
  const double pf = pr.periodic ? 1.0 : std::pow(1.0 / 6.0, d);
  double2* B = arena_.as<double2>("pw_B_root", (size_t)pr.nch * g.pz * g.ncol);
  double2* G = arena_.as<double2>("pw_G_root", (size_t)pr.nch * g.nhalf);
  double2* F = arena_.as<double2>("pw_F_root", (size_t)d * g.nhalf);
  double2* C = arena_.as<double2>("pw_C_root", (size_t)d * g.pz * g.ncol);
  launch_forward(g, root_dev_ids_, 1, pr.nch, arena_.as<double>("outgoing", 1), B, G, st_);
  launch_accumulate_symbol(g, P.kernel, 1, root_dev_es_, root_dev_slot_, root_dev_tau_, G, pr.nch, dA, h, F, st_);
  launch_inverse(g, root_dev_ids_, 1, d, F, C, pf, in, st_);
  launches_ += 5;
}

void Context::run_downward() {  // dmk.cpp:705-857
  Problem& pr = prob_;
  const Plan& P = pr.plan;
  const int d = pr.dim, p = P.p, pz = d == 3 ? p : 1;
  const double* og = arena_.as<double>("outgoing", 1);
  double* in = arena_.as<double>("incoming", 1);
  const int M = (P.N1 - 1) / 2;
  GridDev& gd = grid(grid_lev_, "grid_lev", d, p, P.N1, PI / 3.0, band_r2(P, M, PI / 3.0));
  const PWGrid& g = gd.g;
  const bool use_mma = pw_mma_supported(g);
  const int L = pr.tree.max_level + 1;
  const int S = 3 * M * M + 1;
  // per-level symbol tables (dmk.cpp:741-746), one upload
  std::vector<double> Aall((size_t)L * S);
  for (int lev = 0; lev < L; ++lev) {
    double r_c = std::ldexp(1.0, -lev), r_f = 0.5 * r_c, h = PI / (3.0 * r_f);
    std::vector<double> A = symbol_table(*tab_, h, 3 * M * M, kLevelDiff, r_c, r_f);
    std::copy(A.begin(), A.end(), Aall.begin() + (size_t)lev * S);
  }
  double* hA = (double*)pinned_.get("symlev", Aall.size() * sizeof(double));
  std::memcpy(hA, Aall.data(), Aall.size() * sizeof(double));
  double* dA = arena_.as<double>("symlev", Aall.size());
  cuda_check(cudaMemcpyAsync(dA, hA, Aall.size() * sizeof(double), cudaMemcpyHostToDevice, st_), "symbol upload");
  const size_t bytes_B = sizeof(double2) * pr.nch * g.pz * g.ncol;
  const size_t bytes_FC = sizeof(double2) * d * ((size_t)g.nhalf + (size_t)g.pz * g.ncol);
#ifndef SDMK_PW_BUDGET_MB
#define SDMK_PW_BUDGET_MB 2048
#endif
  constexpr size_t budget = size_t(SDMK_PW_BUDGET_MB) << 20;  // scratch per B / F+C chunk
  const int chunk_src = (int)std::max<size_t>(1, budget / bytes_B);
  const int chunk_tgt = (int)std::max<size_t>(1, budget / bytes_FC);
  // plane-wave timing: one event pair per level, read after the evaluation's
  // final synchronisation (no host round trip between levels)
  while ((int)pw_ev_.size() < 2 * L) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    pw_ev_.push_back(e);
  }
  pw_used_ = 0;
  for (int lev = 0; lev < L; ++lev) {
    const Problem::LevelLists& X = pr.levels[lev];
    if (X.n_src > 0 && X.n_tgt > 0) {
      double r_c = std::ldexp(1.0, -lev), r_f = 0.5 * r_c, h = PI / (3.0 * r_f);
      double pf = std::pow(1.0 / (6.0 * r_f), d);
      double2* G = arena_.as<double2>("pw_G", (size_t)X.n_src * pr.nch * g.nhalf);
      cudaEvent_t e0 = pw_ev_[2 * pw_used_], e1 = pw_ev_[2 * pw_used_ + 1];
      ++pw_used_;
      cudaEventRecord(e0, st_);
      for (int s0 = 0; s0 < X.n_src; s0 += chunk_src) {
        int n = std::min(chunk_src, X.n_src - s0);
        double2* B = arena_.as<double2>("pw_B", (size_t)n * pr.nch * g.pz * g.ncol);
        if (use_mma)
          launch_forward_mma(g, X.src_boxes + s0, n, pr.nch, og, B, G + (size_t)s0 * pr.nch * g.nhalf, st_);
        else
          launch_forward(g, X.src_boxes + s0, n, pr.nch, og, B, G + (size_t)s0 * pr.nch * g.nhalf, st_);
        launches_ += 2;
      }
      const std::vector<int>& gs = X.grp_start_h;
      const int ng = gs.empty() ? 0 : (int)gs.size() - 1;
      for (int t0 = 0, g0 = 0; t0 < X.n_tgt;) {
        int n = std::min(chunk_tgt, X.n_tgt - t0), g1 = g0;
        if (ng > 0) {  // chunk boundaries on group boundaries
          while (g1 < ng && gs[g1 + 1] - t0 <= chunk_tgt) ++g1;
          if (g1 == g0) g1 = g0 + 1;
          n = gs[g1] - t0;
        }
        double2* F = arena_.as<double2>("pw_F", (size_t)n * d * g.nhalf);
        double2* C = arena_.as<double2>("pw_C", (size_t)n * d * g.pz * g.ncol);
        if (ng > 0)
          launch_accumulate_group(g, P.kernel, g1 - g0, X.grp_tstart + g0, X.grp_slot + (size_t)g0 * 64, X.t_meta,
                                  t0, G, dA + (size_t)lev * S, h, F, st_);
        else
          launch_accumulate_symbol(g, P.kernel, n, X.ent_start + t0, X.ent_slot, X.ent_tau, G, pr.nch,
                                   dA + (size_t)lev * S, h, F, st_);
        if (use_mma)
          launch_inverse_mma(g, X.tgt_boxes + t0, n, d, F, C, pf, in, st_);
        else
          launch_inverse(g, X.tgt_boxes + t0, n, d, F, C, pf, in, st_);
        launches_ += 3;
        t0 += n;
        g0 = g1;
      }
      cudaEventRecord(e1, st_);
    }
    if (X.n_interp > 0) {
      if (accumulate_down_)  // children += interp(parent) (dmk.cpp:835-855 on caller-held incoming)
        launch_tensor_apply(p, pz, d, mats_down_, X.interp_in, X.interp_out, X.interp_ci, X.n_interp, d, in, in, 1,
                            st_);
      else if (tensor_mma_supported(p, d))
        if (tensor_seg_supported(p, d))
          launch_tensor_mma_seg(p, mats_down_, X.interp_in, X.interp_out, X.interp_ci, X.interp_seg, X.n_interp_seg,
                                d, in, in, st_);
        else
          launch_tensor_mma(p, mats_down_, X.interp_in, X.interp_out, X.interp_ci, X.n_interp, d, in, in, 3, d, st_);
      else
        launch_tensor_apply(p, pz, d, mats_down_, X.interp_in, X.interp_out, X.interp_ci, X.n_interp, d, in, in, 1,
                            st_);
      ++launches_;
    }
  }
  cuda_check(cudaPeekAtLastError(), "kernel launch");
}

double Context::planewave_ms() {  // after a synchronisation
  double t = 0.0;
  for (int i = 0; i < pw_used_; ++i) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, pw_ev_[2 * i], pw_ev_[2 * i + 1]);
    t += ms;
  }
  return t;
}

void Context::run_target_far(double* ufar) {  // dmk.cpp:861-915
  Problem& pr = prob_;
  const int p = pr.plan.p, pz = pr.dim == 3 ? p : 1;
  ChebDev cb{p, pz, pr.dim, cheb_nodes_, cheb_wts_};
  const double* incoming = arena_.as<double>("incoming", 1);
  if (mma_anterp_supported(p)) {
    // alias targets reuse the source bases computed by the upward pass
    const double* tb = nullptr;
    if (pr.alias && !pr.halo && !force_tbasis_) {  // (halo mode: this rank's source leaves are not its target leaves)
      tb = arena_.as<double>("basis_s", (size_t)3 * pr.ns * p);
    } else {
      double* b = arena_.as<double>("basis_t", (size_t)3 * pr.nt * p);
      launch_basis(cb, pr.boxes, pr.int_leaves, pr.n_int, pr.tpts, pr.nt, 1, b, st_);
      ++launches_;
      tb = b;
    }
    cudaEventRecord(ev_[16], st_);
    launch_interp_mma(cb, pr.boxes, pr.int_leaves, pr.n_int, tb, pr.nt, pr.tperm, incoming, ufar, st_);
    cudaEventRecord(ev_[17], st_);
    interp_timed_ = true;
  } else {
    launch_interp_targets(cb, pr.boxes, pr.int_leaves, pr.n_int, pr.tpts, pr.nt, pr.tperm, incoming, ufar, st_);
  }
  ++launches_;
  cuda_check(cudaPeekAtLastError(), "far-field kernel launch");
}

void Context::run_residual(double* ures, bool stats, int reserve_sms) {  // dmk.cpp:919-1032
  Problem& pr = prob_;
  const Tables& T = *tab_;
  const ResidTables rt = residual_tables(pr.plan.kernel, pr.dim);
  int* flags = arena_.as<int>("flags", 8);
  unsigned long long* st = arena_.as<unsigned long long>("stats", 4);
  if (stats) cuda_check(cudaMemsetAsync(st, 0, 4 * sizeof(unsigned long long), st_), "memset");
  cudaEventRecord(ev_[13], st_);
  launch_residual(rt, pr.boxes, pr.int_leaves, pr.n_int, pr.res_chunks, pr.n_chunks, pr.rng_start, pr.rng_box, pr.rng_info, pr.subrange, pr.spts, pr.ns,
                  pr.sstr, arena_.as<double>("srec", (size_t)pr.ns * ((pr.dim + pr.sc + 1) / 2 * 2)),
                  pr.periodic ? 1 : 0, pr.tpts, pr.nt, pr.tperm, pr.alias ? 1 : 0, reserve_sms, T.self_const, ures, flags + 3,
                  stats ? st : nullptr, arena_.get("res_scratch", residual_scratch_bytes()), st_);
  ++launches_;  // source record packing
  cudaEventRecord(ev_[12], st_);
  ++launches_;
}

// The residual kernel's radial tables for the current tables tab_ (uploaded
// to the arena): piecewise re-expansions and the reference's coefficients.
ResidTables Context::residual_tables(int kernel, int dim) {
  const Tables& T = *tab_;
  const Cheb* cd = nullptr;
  const Cheb* co = nullptr;
  if (kernel == kStokeslet) {
    cd = &T.s_diag;
    co = &T.s_offd;
  } else if (kernel == kStresslet) {
    cd = &T.t_diag;
    co = &T.t_offd;
  } else {
    co = &T.w_offd;
  }
  if (cd && (cd->lo != co->lo || cd->hi != co->hi)) throw RuntimeError("residual tables on different intervals");
  // piecewise re-expansion of the radial tables (setup.hpp): the kernel reads
  // deg + 1 coefficient pairs per pair evaluation.  Candidates in order of
  // cost (degree), each on the finest interval grid its shared table holds;
  // the first whose values stay within 2e-15 of the reference's Clenshaw
  // values is taken (else the most accurate).  The bar is absolute because
  // the residual kernels carry 1/r^2 .. 1/r^5 factors: an absolute table
  // error at small s is amplified by close pairs (points on surfaces), and
  // degree 5 on 128 intervals (1e-13 for the 3D stresslet) left 6e-9
  // scaled differences at BASELINE cfg3; degree 6 is below 1e-15.
  constexpr double kPwTol = 2e-15;
  auto& cached = pw_cache_[{&T, kernel}];  // fitted once per table set and kernel
  PiecewisePoly& po = cached.first;
  PiecewisePoly& pd = cached.second;
  if (po.c.empty()) {
    PiecewisePoly best_o, best_d;
    double best = 1e300;
    for (int deg : {5, 6, 8, 10, 12}) {
      const int ni = std::min(128, residual_max_pw() / (deg + 1));
      po = piecewise_from_cheb(*co, ni, deg, 1.0);  // rel_tol 1: exactly this degree
      double err = po.max_err;
      if (cd) {
        pd = piecewise_from_cheb(*cd, ni, deg, 1.0);
        err = std::max(err, pd.max_err);
      }
      if (err < best) {
        best = err;
        best_o = po;
        best_d = pd;
      }
      if (err <= kPwTol) break;
    }
    po = best_o;
    pd = best_d;
  }
  const int npw = po.ni * (po.deg + 1);
  if (npw > residual_max_pw()) throw RuntimeError("residual table re-expansion too large");
  const int nd = cd ? (int)cd->a.size() : 0, no = (int)co->a.size();
  if (nd > kResidMaxCheb || no > kResidMaxCheb) throw RuntimeError("residual table longer than the GPU limit (80)");
  const size_t nall = 2 * (size_t)npw + 2 * kResidMaxCheb;
  double* hc = (double*)pinned_.get("rtab", nall * sizeof(double));
  // the kernel's constant factors folded into the tables (residual_apply,
  // split.cpp:258-317): 1/(8 pi) for the 3D Stokeslet, 1/(8 pi) and -3/(4 pi)
  // for the stresslet, 1/(8 pi) (3D) or 1/(4 pi) (2D) for the rotlet; the 2D
  // Stokeslet's diagonal enters as -2 s log s - table, so it stays unscaled
  const double k8 = 1.0 / (8.0 * PI), k4 = 1.0 / (4.0 * PI);
  double sd = 1.0, so = 1.0;
  if (kernel == kStokeslet) sd = so = dim == 3 ? k8 : 1.0;
  else if (kernel == kStresslet) sd = k8, so = -3.0 * k4;
  else so = dim == 3 ? k8 : k4;
  // the kernel drops pairs past the last interval (s >= hi), where the
  // reference's residual is zero (s >= support, split.cpp:147-179)
  if (co->lo != 0.0 || co->hi != T.support) throw RuntimeError("residual table domain is not [0, support]");
  for (int i = 0; i < npw; ++i) hc[npw + i] = so * po.c[i];
  if (cd) for (int i = 0; i < npw; ++i) hc[i] = sd * pd.c[i];
  else std::fill(hc, hc + npw, 0.0);
  double* hcheb = hc + 2 * npw;
  std::fill(hcheb, hcheb + 2 * kResidMaxCheb, 0.0);
  if (cd) std::copy(cd->a.begin(), cd->a.end(), hcheb);
  std::copy(co->a.begin(), co->a.end(), hcheb + kResidMaxCheb);
  double* dc = arena_.as<double>("rtab", nall);
  cuda_check(cudaMemcpyAsync(dc, hc, nall * sizeof(double), cudaMemcpyHostToDevice, st_), "table upload");
  // the first piecewise interval takes the reference's own recurrence (see ResidTables)
  const double s_exact = co->lo + (co->hi - co->lo) / po.ni;
  return ResidTables{po.ni, po.deg, co->lo, co->hi, T.support, kernel, dim, dc, dc + npw,
                     dc + 2 * npw, dc + 2 * npw + kResidMaxCheb, nd, no, s_exact, sd, so};
}

// ------------------------------------------------------------- entries --
void Context::evaluate(const Plan& P, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                       const double* str, int mode, double* u, sdmk_report* rep, bool device_ptrs) {
  if (manual_x_ && nranks_ > 1) throw InvalidArgument("evaluate: manual exchange mode needs evaluate_begin/end");
  evaluate_begin(P, dim, ns, src, nt, tgt, str, mode, device_ptrs);
  if (prob_.halo) {  // NCCL exchange of the packed halo slabs on the side stream; evaluate_end
                     // runs the residual (which needs no halo) while it is in flight
    cuda_check(cudaStreamWaitEvent(st2_, ev_[10], 0), "stream wait");
    cudaEventRecord(ev_[14], st2_);
    comm_->exchange(arena_.as<double>("halo_send", 1), prob_.send_off, arena_.as<double>("halo_recv", 1),
                    prob_.recv_off, st2_);
    cudaEventRecord(ev_[15], st2_);
    cuda_check(cudaEventRecord(x_ev_, st2_), "event record");
    x_pending_ = true;
  }
  try {
    evaluate_end(u, rep);
  } catch (...) {
    x_pending_ = false;
    throw;
  }
}

void Context::evaluate_begin(const Plan& P, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                             const double* str, int mode, bool device_ptrs) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  begun_ = false;
  lists_side_ = false;
  check_inputs(P, dim, ns, nt, mode);
  tab_ = tab_override_ ? tab_override_ : &tables_for(P);
  if (tab_->kernel != P.kernel || tab_->dim != P.dim || tab_->win.kind != P.window)
    throw InvalidArgument("evaluate: supplied split tables do not match the plan");
  launches_ = 0;
  const int sc = strength_width(P.kernel, dim);
  const bool alias = nt == 0;
  const int ntt = alias ? (int)ns : (int)nt;
  call_ = Call{dim, sc, ntt, ns, nt, alias, device_ptrs};
  halo_run_ = nranks_ > 1 && (comm_ || manual_x_);
  interp_timed_ = anterp_timed_ = false;
  cudaEventRecord(ev_[0], st_);
  copy_in(arena_.as<double>("src_in", (size_t)ns * dim), src, sizeof(double) * ns * dim, device_ptrs);
  if (!alias) copy_in(arena_.as<double>("tgt_in", (size_t)nt * dim), tgt, sizeof(double) * nt * dim, device_ptrs);
  // pinned strengths travel on a second stream while the tree is built (they
  // are first needed by the upward pass); pageable / device ones as before
  str_pending_ = !device_ptrs && !is_pageable(str) && ns * sc * sizeof(double) > kSideStreamMin;
  if (str_pending_) {
    cuda_check(cudaStreamWaitEvent(st2_, ev_[0], 0), "stream wait");
    cuda_check(cudaMemcpyAsync(arena_.as<double>("str_in", (size_t)ns * sc), str, sizeof(double) * ns * sc,
                               cudaMemcpyHostToDevice, st2_),
               "copy in");
    cuda_check(cudaEventRecord(str_ev_, st2_), "event record");
  } else {
    copy_in(arena_.as<double>("str_in", (size_t)ns * sc), str, sizeof(double) * ns * sc, device_ptrs);
  }
  cudaEventRecord(ev_[1], st_);
  zero_all_ = false;  // only the evaluated outputs are returned
  try {
    build_problem(P, dim, (int)ns, (int)nt, mode, true);
    cudaEventRecord(ev_[2], st_);
    run_upward();
    cudaEventRecord(ev_[3], st_);
    lists_side_ = true;
    upload_tree_lists_b();  // host work overlaps the upward pass on the GPU
    lists_side_ = false;
    cudaEventRecord(ev_[8], st_);
    if (prob_.halo) {
      const Problem& pr = prob_;
      const int64_t elems = (int64_t)pr.nch * (dim == 3 ? P.p : 1) * P.p * P.p;
      double* snd = arena_.as<double>("halo_send", (size_t)pr.send_off[nranks_]);
      arena_.as<double>("halo_recv", (size_t)pr.recv_off[nranks_]);
      launch_copy_boxes(pr.n_send, pr.send_ids, arena_.as<double>("outgoing", 1), nullptr, snd, elems, st_);
      ++launches_;
    }
    cudaEventRecord(ev_[10], st_);
  } catch (...) {
    lists_side_ = false;
    zero_all_ = true;
    throw;
  }
  begun_ = true;
}

void Context::evaluate_end(double* u, sdmk_report* rep) {
  if (!begun_) throw InvalidArgument("evaluate_end: no evaluate_begin in flight");
  begun_ = false;
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  struct Restore {
    bool& f;
    ~Restore() { f = true; }
  } restore{zero_all_};
  const Plan& P = prob_.plan;
  const int dim = call_.dim, ntt = call_.ntt;
  const bool device_ptrs = call_.device_ptrs;
  cudaEventRecord(ev_[11], st_);
  double* ufar = arena_.as<double>("ufar", (size_t)ntt * dim);
  double* ures = arena_.as<double>("ures", (size_t)ntt * dim);
  unsigned char* own = nullptr;
  if (nranks_ > 1) {  // only the owned targets are written by the passes below
    cuda_check(cudaMemsetAsync(ufar, 0, sizeof(double) * ntt * dim, st_), "memset ufar");
    cuda_check(cudaMemsetAsync(ures, 0, sizeof(double) * ntt * dim, st_), "memset ures");
    own = arena_.as<unsigned char>("own", (size_t)ntt);
    launch_own_mask(ntt, prob_.tperm, prob_.t_own0, prob_.t_own1, own, st_);
    ++launches_;
  }
  // halo mode: the near field first -- it needs no halo, so with NCCL it runs
  // beside the exchange (a few SMs left free); the manual-exchange tests take
  // the same order
  const bool overlap = prob_.halo;
  if (overlap) {
    run_residual(ures, rep != nullptr, x_pending_ ? 8 : 0);
    if (x_pending_) cuda_check(cudaStreamWaitEvent(st_, x_ev_, 0), "stream wait");
    x_pending_ = false;
  }
  if (prob_.halo) {
    const Problem& pr = prob_;
    const int64_t elems = (int64_t)pr.nch * (dim == 3 ? P.p : 1) * P.p * P.p;
    launch_copy_boxes(pr.n_recv, nullptr, arena_.as<double>("halo_recv", 1), pr.recv_ids,
                      arena_.as<double>("outgoing", 1), elems, st_);
    ++launches_;
  }
  cudaEventRecord(ev_[9], st_);
  if (prob_.halo) run_upward_top();
  run_root();
  cudaEventRecord(ev_[4], st_);
  run_downward();
  run_target_far(ufar);
  cudaEventRecord(ev_[5], st_);
  if (!overlap) run_residual(ures, rep != nullptr);
  // global terms (dmk.cpp:1086-1102)
  Problem& pr = prob_;
  double* sums = arena_.as<double>("sums", 16);
  double* scratch = arena_.as<double>("sum_scratch", 256 * 8);
  double corr_scale = 0.0;
  const double* corr = nullptr;
  const double* zm = nullptr;
  if (P.kernel == kStokeslet && !pr.periodic && tab_->corr_const != 0.0) {
    launch_column_sums(pr.sstr, pr.ns, dim, sums, scratch, st_);
    corr = sums;
    corr_scale = tab_->corr_const;
    launches_ += 2;
  }
  if (P.kernel == kStresslet && pr.periodic) {
    launch_zero_mode_moments(pr.spts, pr.sstr, pr.ns, dim, sums + 8, scratch, st_);
    zm = sums + 8;
    launches_ += 2;
  }
  double* du = device_ptrs ? u : arena_.as<double>("u", (size_t)ntt * dim);
  launch_combine(ntt, dim, ufar, ures, corr, corr_scale, zm, pr.tpts_caller, own, du, st_);
  ++launches_;
  // with a communicator every rank returns the assembled u: each rank's owned
  // Morton range of targets is packed in sorted order, all-gathered (padded
  // to the longest range), and scattered to caller order on every rank --
  // (R-1)/R of u moved per rank instead of the ~2x of an all-reduce
  if (comm_ && nranks_ > 1) {
    const std::vector<int64_t>& b = pr.t_bounds;
    int64_t maxc = 1;
    for (int r = 0; r < nranks_; ++r) maxc = std::max<int64_t>(maxc, b[r + 1] - b[r]);
    double* snd = arena_.as<double>("ag_send", (size_t)maxc * dim);
    double* rcv = arena_.as<double>("ag_recv", (size_t)nranks_ * maxc * dim);
    launch_pack_owned(pr.t_own0, pr.t_own1 - pr.t_own0, dim, pr.tperm, du, snd, st_);
    comm_->allgather(snd, rcv, (size_t)maxc * dim, st_);
    launch_scatter_ranges(ntt, dim, pr.d_bounds, nranks_, maxc * dim, pr.tperm, rcv, du, st_);
    launches_ += 2;
  }
  cudaEventRecord(ev_[6], st_);
  if (!device_ptrs) copy_out(u, du, sizeof(double) * ntt * dim);
  cudaEventRecord(ev_[7], st_);
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(hflags, arena_.as<int>("flags", 8), 8 * sizeof(int), cudaMemcpyDeviceToHost, st_),
             "D2H flags");
  unsigned long long* hst = (unsigned long long*)pinned_.get("hstats", 64);
  if (rep)
    cuda_check(cudaMemcpyAsync(hst, arena_.as<unsigned long long>("stats", 4), 4 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, st_),
               "D2H stats");
  sync();
  cuda_check(cudaGetLastError(), "kernel launch");
  if (hflags[3]) throw DomainError("residual_pass: coincident points");
  if (rep) {
    // between evaluate_begin and evaluate_end: the exchange (NCCL) or the
    // caller's transfers (manual mode, excluded from t_total)
    // (halo mode runs the residual between evaluate_end's start and the
    // unpack: the unpack is timed from the residual's end)
    const double gap = ev_ms(10, 11), xfer = ev_ms(8, 10) + (pr.halo ? ev_ms(12, 9) : ev_ms(11, 9));
    const bool manual = !comm_;
    rep->num_boxes = pr.tree.num_boxes();
    rep->max_level = pr.tree.max_level;
    rep->num_sources = (int)call_.ns;
    rep->num_targets = ntt;
    rep->t_h2d = ev_ms(0, 1) * 1e-3;
    rep->t_tree = ev_ms(1, 2) * 1e-3;
    rep->t_upward = ev_ms(2, 3) * 1e-3;
    rep->t_root = (ev_ms(3, 4) - ev_ms(8, 9)) * 1e-3;
    rep->t_downward = ev_ms(4, 5) * 1e-3;
    rep->t_residual = (overlap ? ev_ms(13, 12) : ev_ms(5, 6)) * 1e-3;
    rep->t_d2h = ev_ms(6, 7) * 1e-3;
    rep->t_total = (ev_ms(0, 7) - (manual ? gap : 0.0)) * 1e-3;
    rep->t_residual_kernel = ev_ms(13, 12) * 1e-3;
    rep->t_interp_kernel = interp_timed_ ? ev_ms(16, 17) * 1e-3 : 0.0;
    rep->t_anterp_kernel = anterp_timed_ ? ev_ms(18, 19) * 1e-3 : 0.0;
    rep->t_planewave = planewave_ms() * 1e-3;
    rep->p2p_candidates = (int64_t)hst[0];
    rep->p2p_in_support = (int64_t)hst[1];
    rep->kernel_launches = launches_;
    // NCCL: pack + unpack on the stream plus the exchange on the side stream
    // (which overlaps the residual pass)
    rep->t_exchange = pr.halo ? (manual ? xfer : ev_ms(8, 10) + ev_ms(14, 15)) * 1e-3 : 0.0;
    rep->halo_bytes_sent = pr.halo ? pr.send_off[nranks_] * (int64_t)sizeof(double) : 0;
    rep->halo_bytes_recv = pr.halo ? pr.recv_off[nranks_] * (int64_t)sizeof(double) : 0;
  }
}

void Context::setup(const Plan& P, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                    const double* str, int mode) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  prob_.ready = false;
  begun_ = false;
  halo_run_ = false;  // the pass-level API keeps the replicated upward pass
  check_inputs(P, dim, ns, nt, mode);
  tab_ = &tables_for(P);
  const int sc = strength_width(P.kernel, dim);
  cuda_check(cudaMemcpyAsync(arena_.as<double>("src_in", (size_t)ns * dim), src, sizeof(double) * ns * dim,
                             cudaMemcpyHostToDevice, st_),
             "copy sources");
  if (nt > 0)
    cuda_check(cudaMemcpyAsync(arena_.as<double>("tgt_in", (size_t)nt * dim), tgt, sizeof(double) * nt * dim,
                               cudaMemcpyHostToDevice, st_),
               "copy targets");
  cuda_check(cudaMemcpyAsync(arena_.as<double>("str_in", (size_t)ns * sc), str, sizeof(double) * ns * sc,
                             cudaMemcpyHostToDevice, st_),
             "copy strengths");
  str_pending_ = false;
  build_problem(P, dim, (int)ns, (int)nt, mode);
}

static void need(const Problem& p) {
  if (!p.ready) throw InvalidArgument("no problem set up in this context (call sdmk_setup first)");
}

void Context::upward(double* out) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  run_upward();
  const int p = prob_.plan.p, pz = prob_.dim == 3 ? p : 1;
  size_t n = (size_t)prob_.tree.num_boxes() * prob_.nch * pz * p * p;
  cuda_check(cudaMemcpyAsync(out, arena_.as<double>("outgoing", 1), n * sizeof(double), cudaMemcpyDeviceToHost, st_),
             "D2H outgoing");
  sync();
}

void Context::incoming(int stage, double* out) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  run_upward();
  run_root();
  if (stage >= 1) run_downward();
  const int p = prob_.plan.p, pz = prob_.dim == 3 ? p : 1;
  size_t n = (size_t)prob_.tree.num_boxes() * prob_.dim * pz * p * p;
  cuda_check(cudaMemcpyAsync(out, arena_.as<double>("incoming", 1), n * sizeof(double), cudaMemcpyDeviceToHost, st_),
             "D2H incoming");
  sync();
}

void Context::target_far(double* out) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  run_upward();
  run_root();
  run_downward();
  double* uf = arena_.as<double>("ufar", (size_t)prob_.nt * prob_.dim);
  run_target_far(uf);
  cuda_check(cudaMemcpyAsync(out, uf, sizeof(double) * prob_.nt * prob_.dim, cudaMemcpyDeviceToHost, st_), "D2H u");
  sync();
}

void Context::residual(double* out) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  int* flags = arena_.as<int>("flags", 8);
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  double* ur = arena_.as<double>("ures", (size_t)prob_.nt * prob_.dim);
  run_residual(ur, false);
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(out, ur, sizeof(double) * prob_.nt * prob_.dim, cudaMemcpyDeviceToHost, st_), "D2H u");
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  cuda_check(cudaGetLastError(), "kernel launch");
  if (hflags[3]) throw DomainError("residual_pass: coincident points");
}

void Context::direct(int kernel, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                     const double* str, const Tables* tab, double cutoff, bool periodic, double* u, bool device_ptrs) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const char* who = tab ? "direct_residual_sum" : "direct_sum";
  if (tab) {  // oracle.cpp:184-191
    if (!(cutoff > 0.0)) throw InvalidArgument("direct_residual_sum: cutoff must be positive");
    if (periodic && cutoff > 1.0) throw InvalidArgument("direct_residual_sum: periodic image sums require cutoff <= 1");
    if (dim != tab->dim) throw InvalidArgument("direct_residual_sum: dimension mismatch");
    kernel = tab->kernel;
  }
  // validate_system (oracle.cpp:103-131)
  if (kernel != kStokeslet && kernel != kStresslet && kernel != kRotlet)
    throw InvalidArgument("particle sums support the Stokeslet, stresslet, and rotlet kernels");
  if (dim != 2 && dim != 3) throw InvalidArgument("ParticleSystem: dim must be 2 or 3");
  if (ns < 1) throw InvalidArgument("ParticleSystem: bad source array length");
  if (nt < 0) throw InvalidArgument("ParticleSystem: bad target array length");
  if (ns > (int64_t(1) << 31) - 1 || nt > (int64_t(1) << 31) - 1)
    throw InvalidArgument(std::string(who) + ": more than 2^31-1 points");
  const int sc = strength_width(kernel, dim);
  const bool alias = nt == 0;
  const int ntt = alias ? (int)ns : (int)nt;
  double* dsrc = arena_.as<double>("dir_src", (size_t)ns * dim);
  double* dtgt = alias ? dsrc : arena_.as<double>("dir_tgt", (size_t)nt * dim);
  double* dstr = arena_.as<double>("dir_str", (size_t)ns * sc);
  double* du = device_ptrs ? u : arena_.as<double>("dir_u", (size_t)ntt * dim);
  copy_in(dsrc, src, sizeof(double) * ns * dim, device_ptrs);
  if (!alias) copy_in(dtgt, tgt, sizeof(double) * nt * dim, device_ptrs);
  copy_in(dstr, str, sizeof(double) * ns * sc, device_ptrs);
  int* flags = arena_.as<int>("flags", 8);
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  const bool per = tab && periodic;
  launch_validate(dstr, (int64_t)ns * sc, 1, flags, 2, st_);
  launch_validate(dsrc, (int64_t)ns * dim, per, flags, 0, st_);
  if (!alias) launch_validate(dtgt, (int64_t)nt * dim, per, flags, 0, st_);
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  if (tree_only_ && (hflags[0] || hflags[1])) throw InvalidArgument("build_tree: point outside the unit box");
  if (hflags[2]) throw InvalidArgument("ParticleSystem: non-finite strength");
  if (hflags[0]) throw InvalidArgument("ParticleSystem: non-finite coordinate");
  if (hflags[1]) throw InvalidArgument("ParticleSystem: coordinate outside the unit box");
  if (per) {  // wrap_into_box (oracle.cpp:133-141)
    launch_wrap(dsrc, (int64_t)ns * dim, st_);
    if (!alias) launch_wrap(dtgt, (int64_t)nt * dim, st_);
  }
  DirectTables T;
  if (tab) {
    const Cheb* cd = nullptr;
    const Cheb* co = nullptr;
    if (kernel == kStokeslet) cd = &tab->s_diag, co = &tab->s_offd;
    else if (kernel == kStresslet) cd = &tab->t_diag, co = &tab->t_offd;
    else co = &tab->w_offd;
    if ((cd && cd->a.size() > (size_t)kDirectMaxCheb) || co->a.size() > (size_t)kDirectMaxCheb)
      throw InvalidArgument("direct_residual_sum: table longer than the GPU limit");
    double* hc = (double*)pinned_.get("dir_cheb", sizeof(double) * 2 * kDirectMaxCheb);
    double* dc = arena_.as<double>("dir_cheb", 2 * kDirectMaxCheb);
    if (cd) std::copy(cd->a.begin(), cd->a.end(), hc);
    std::copy(co->a.begin(), co->a.end(), hc + kDirectMaxCheb);
    cuda_check(cudaMemcpyAsync(dc, hc, sizeof(double) * 2 * kDirectMaxCheb, cudaMemcpyHostToDevice, st_), "H2D cheb");
    T.cutoff = cutoff;
    T.support = tab->support;
    T.periodic = periodic ? 1 : 0;
    T.cd = dc;
    T.co = dc + kDirectMaxCheb;
    T.nd = cd ? (int)cd->a.size() : 0;
    T.no = (int)co->a.size();
    if (cd) T.dlo = cd->lo, T.dhi = cd->hi;
    T.olo = co->lo;
    T.ohi = co->hi;
  }
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  launch_direct(kernel, dim, dsrc, (int)ns, dtgt, ntt, dstr, alias ? 1 : 0, T, tab != nullptr, du, flags, st_);
  cuda_check(cudaPeekAtLastError(), "direct kernel launch");
  if (!device_ptrs) copy_out(u, du, sizeof(double) * ntt * dim);
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  cuda_check(cudaGetLastError(), "kernel launch");
  if (hflags[0]) throw DomainError(std::string(who) + ": coincident points");
}

// ---------------------------------------------- tree-first pass-level API --
// The reference's build_tree / upward_pass / root_far_field / downward_pass /
// target_far_fields / residual_pass (tree.hpp:90-92, dmk.hpp:84-131) with
// every input and output a caller-held host array, so the C++ drop-in can
// hand ProxyData between passes exactly as the reference's callers do.
void Context::tree_build(int dim, bool periodic, int n_s, int p, int64_t ns, const double* src, int64_t nt,
                         const double* tgt) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  prob_.ready = false;
  begun_ = false;
  halo_run_ = false;
  // tree.cpp:233-244, in the reference's order
  if (dim != 2 && dim != 3) throw InvalidArgument("build_tree: dim must be 2 or 3");
  if (n_s < 1) throw InvalidArgument("build_tree: n_s must be >= 1");
  if (p < 1) throw InvalidArgument("build_tree: proxy order must be >= 1");
  if (ns < 1 || nt < 0) throw InvalidArgument("build_tree: bad point array length");
  if (ns > (int64_t(1) << 31) - 1 || nt > (int64_t(1) << 31) - 1)
    throw InvalidArgument("build_tree: more than 2^31-1 points");
  if (p > 64) throw InvalidArgument("build_tree: proxy order above the GPU path limit (64)");
  Plan P;  // the tree depends on dim, periodic, n_s and p only; passes bind their own plan
  P.kernel = kStokeslet;
  P.dim = dim;
  P.n_s = n_s;
  P.p = p;
  P.c = 1.0;
  P.N1 = P.N_per = 1;
  cuda_check(cudaMemcpyAsync(arena_.as<double>("src_in", (size_t)ns * dim), src, sizeof(double) * ns * dim,
                             cudaMemcpyHostToDevice, st_),
             "copy sources");
  if (nt > 0)
    cuda_check(cudaMemcpyAsync(arena_.as<double>("tgt_in", (size_t)nt * dim), tgt, sizeof(double) * nt * dim,
                               cudaMemcpyHostToDevice, st_),
               "copy targets");
  cuda_check(cudaMemsetAsync(arena_.as<double>("str_in", (size_t)ns * dim), 0, sizeof(double) * ns * dim, st_),
             "memset strengths");
  str_pending_ = false;
  tree_only_ = true;
  struct Reset {
    bool& f;
    ~Reset() { f = false; }
  } reset{tree_only_};
  build_problem(P, dim, (int)ns, (int)nt, periodic ? 1 : 0);
}

void Context::tree_neighbors(int64_t* counts, int32_t* entries) {
  need(prob_);
  HostTree& t = prob_.tree;
  finish_topology(t, true);
  size_t at = 0;
  for (int b = 0; b < t.num_boxes(); ++b) {
    const NbrSpan lists[3] = {t.col[b], t.crs[b], t.fin[b]};
    for (int k = 0; k < 3; ++k) {
      counts[3 * (size_t)b + k] = lists[k].size();
      if (entries)
        for (const Nbr& e : lists[k]) {
          int32_t* o = entries + 4 * at++;
          o[0] = e.box;
          o[1] = e.shift[0];
          o[2] = e.shift[1];
          o[3] = e.shift[2];
        }
    }
  }
}

void Context::tree_sorted(double* src_pts, double* tgt_pts, int32_t* src_q, int32_t* tgt_q) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  const Problem& pr = prob_;
  const int d = pr.dim;
  // device copies are SoA (axis-major); the reference's are point-major
  auto fetch = [&](const double* dp, const int32_t* dq, int n, double* hp, int32_t* hq) {
    std::vector<double> x((size_t)n * d);
    std::vector<int32_t> q((size_t)n * d);
    cuda_check(cudaMemcpyAsync(x.data(), dp, sizeof(double) * n * d, cudaMemcpyDeviceToHost, st_), "D2H points");
    cuda_check(cudaMemcpyAsync(q.data(), dq, sizeof(int32_t) * n * d, cudaMemcpyDeviceToHost, st_), "D2H q");
    sync();
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        if (hp && a < d) hp[(size_t)i * d + a] = x[(size_t)a * n + i];
        if (hq) hq[(size_t)i * 3 + a] = a < d ? q[(size_t)a * n + i] : 0;
      }
  };
  fetch(pr.spts, pr.sq, pr.ns, src_pts, src_q);
  if (!pr.alias) fetch(pr.tpts, pr.tq, pr.nt, tgt_pts, tgt_q);
}

void Context::tree_perm(int32_t* src_perm, int32_t* tgt_perm) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  const Problem& p = prob_;
  // on the context stream: ordered after the (possibly re-sorting) tree build
  cuda_check(cudaMemcpyAsync(src_perm, p.sperm, sizeof(int) * p.ns, cudaMemcpyDeviceToHost, st_), "D2H perm");
  if (tgt_perm && !p.alias)
    cuda_check(cudaMemcpyAsync(tgt_perm, p.tperm, sizeof(int) * p.nt, cudaMemcpyDeviceToHost, st_), "D2H perm");
  sync();
}

// check_plan (dmk.cpp:534-539) plus what this pass needs of the plan
void Context::bind_plan(const Plan& P, const Tables* tab, const char* who) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  need(prob_);
  begun_ = false;
  halo_run_ = false;
  Problem& pr = prob_;
  if (P.dim != pr.dim) throw InvalidArgument("dmk: tree and plan dimensions differ");
  if (P.p != pr.tree.p) throw InvalidArgument("dmk: tree proxy order does not match plan");
  if (P.kernel != kStokeslet && P.kernel != kStresslet && P.kernel != kRotlet)
    throw InvalidArgument(std::string(who) + ": the Stokeslet, stresslet, and rotlet kernels only");
  if (P.N1 < 1 || P.N1 > 127 || P.N_per < 1 || P.N_per > 127)
    throw InvalidArgument(std::string(who) + ": Fourier grid size outside [1, 127]");
  if (tab && (tab->kernel != P.kernel || tab->dim != P.dim))
    throw InvalidArgument(std::string(who) + ": split tables do not match the plan's kernel and dimension");
  const int n_s = pr.plan.n_s;
  pr.plan = P;
  pr.plan.n_s = n_s;  // the tree's capacity, as built
  pr.nch = channels_out(P.kernel, pr.dim);
  pr.sc = strength_width(P.kernel, pr.dim);
  tab_ = tab ? tab : &tables_for(P);
  zero_all_ = true;
}

void Context::load_strengths(int64_t nstr, const double* str, const char* who) {
  Problem& pr = prob_;
  if (nstr != (int64_t)pr.ns * pr.sc) throw InvalidArgument(std::string(who) + ": strength array size mismatch");
  double* d = arena_.as<double>("str_in", (size_t)pr.ns * pr.sc);
  cuda_check(cudaMemcpyAsync(d, str, sizeof(double) * nstr, cudaMemcpyHostToDevice, st_), "copy strengths");
  pr.sstr = arena_.as<double>("sstr", (size_t)pr.ns * pr.sc);
  launch_gather_strengths(d, pr.sperm, pr.ns, pr.sc, pr.sstr, st_);
}

static size_t proxy_count(const Problem& pr, int channels) {
  const int p = pr.tree.p, pz = pr.dim == 3 ? p : 1;
  return (size_t)pr.tree.num_boxes() * channels * pz * p * p;
}

void Context::pass_upward(const Plan& P, int64_t nstr, const double* str, double* out) {
  bind_plan(P, nullptr, "upward_pass");
  load_strengths(nstr, str, "upward_pass");
  run_upward();
  cuda_check(cudaMemcpyAsync(out, arena_.as<double>("outgoing", 1), proxy_count(prob_, prob_.nch) * sizeof(double),
                             cudaMemcpyDeviceToHost, st_),
             "D2H outgoing");
  sync();
}

void Context::pass_root(const Plan& P, const Tables* tab, int64_t nog, const double* og, bool periodic, int64_t nin,
                        double* in) {
  bind_plan(P, tab, "root_far_field");
  Problem& pr = prob_;
  const size_t no = proxy_count(pr, pr.nch), ni = proxy_count(pr, pr.dim);
  if ((size_t)nog != no) throw InvalidArgument("root_far_field: outgoing proxies do not match the tree and plan");
  if ((size_t)nin != ni) throw InvalidArgument("root_far_field: incoming proxies do not match the tree and plan");
  cuda_check(cudaMemcpyAsync(arena_.as<double>("outgoing", no), og, no * sizeof(double), cudaMemcpyHostToDevice, st_),
             "H2D outgoing");
  arena_.as<double>("incoming", ni);
  const bool tree_periodic = pr.periodic;
  pr.periodic = periodic;  // the lattice sum follows the argument (dmk.cpp:678-681)
  struct Restore {
    bool& f;
    bool v;
    ~Restore() { f = v; }
  } restore{pr.periodic, tree_periodic};
  zero_all_ = false;  // only box 0 is written and read back
  run_root();
  zero_all_ = true;
  const size_t nb0 = ni / pr.tree.num_boxes();
  std::vector<double> box0(nb0);
  cuda_check(cudaMemcpyAsync(box0.data(), arena_.as<double>("incoming", 1), nb0 * sizeof(double),
                             cudaMemcpyDeviceToHost, st_),
             "D2H incoming");
  sync();
  for (size_t i = 0; i < nb0; ++i) in[i] += box0[i];  // inverse_grid_add into the caller's root box
}

void Context::pass_downward(const Plan& P, const Tables* tab, int64_t nog, const double* og, bool periodic,
                            int64_t nin, double* in) {
  (void)periodic;  // periodic images enter through the colleague shifts (dmk.cpp:708)
  bind_plan(P, tab, "downward_pass");
  Problem& pr = prob_;
  const size_t no = proxy_count(pr, pr.nch), ni = proxy_count(pr, pr.dim);
  if ((size_t)nog != no) throw InvalidArgument("downward_pass: outgoing proxies do not match the tree and plan");
  if ((size_t)nin != ni) throw InvalidArgument("downward_pass: incoming proxies do not match the tree and plan");
  cuda_check(cudaMemcpyAsync(arena_.as<double>("outgoing", no), og, no * sizeof(double), cudaMemcpyHostToDevice, st_),
             "H2D outgoing");
  double* din = arena_.as<double>("incoming", ni);
  cuda_check(cudaMemcpyAsync(din, in, ni * sizeof(double), cudaMemcpyHostToDevice, st_), "H2D incoming");
  accumulate_down_ = true;
  struct Reset {
    bool& f;
    ~Reset() { f = false; }
  } reset{accumulate_down_};
  run_downward();
  cuda_check(cudaMemcpyAsync(in, din, ni * sizeof(double), cudaMemcpyDeviceToHost, st_), "D2H incoming");
  sync();
}

void Context::pass_target_far(const Plan& P, int64_t nin, const double* in, double* u) {
  bind_plan(P, nullptr, "target_far_fields");
  Problem& pr = prob_;
  const size_t ni = proxy_count(pr, pr.dim);
  if ((size_t)nin != ni) throw InvalidArgument("target_far_fields: incoming proxies do not match the tree and plan");
  cuda_check(cudaMemcpyAsync(arena_.as<double>("incoming", ni), in, ni * sizeof(double), cudaMemcpyHostToDevice, st_),
             "H2D incoming");
  double* uf = arena_.as<double>("ufar", (size_t)pr.nt * pr.dim);
  force_tbasis_ = true;
  struct Reset {
    bool& f;
    ~Reset() { f = false; }
  } reset{force_tbasis_};
  run_target_far(uf);
  cuda_check(cudaMemcpyAsync(u, uf, sizeof(double) * pr.nt * pr.dim, cudaMemcpyDeviceToHost, st_), "D2H u");
  sync();
  cuda_check(cudaGetLastError(), "kernel launch");
}

void Context::pass_residual(const Plan& P, const Tables* tab, int64_t nstr, const double* str, bool periodic,
                            double* u) {
  (void)periodic;  // images enter through the neighbour shifts (dmk.cpp:923)
  bind_plan(P, tab, "residual_pass");
  load_strengths(nstr, str, "residual_pass");
  Problem& pr = prob_;
  int* flags = arena_.as<int>("flags", 8);
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  double* ur = arena_.as<double>("ures", (size_t)pr.nt * pr.dim);
  run_residual(ur, false);
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(u, ur, sizeof(double) * pr.nt * pr.dim, cudaMemcpyDeviceToHost, st_), "D2H u");
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  cuda_check(cudaGetLastError(), "kernel launch");
  if (hflags[3]) throw DomainError("residual_pass: coincident points");
}

const Tables& Context::tables_image(const void* bytes, size_t n) {
  std::string key(static_cast<const char*>(bytes), n);
  auto it = image_tables_.find(key);
  if (it == image_tables_.end()) it = image_tables_.emplace(key, parse_tables(bytes, n)).first;
  return it->second;
}

// ------------------------------------------------------------- FFT Ewald --
namespace {
// piecewise monomials of f on [0, 1): ni intervals, degree deg (Chebyshev
// interpolation per interval, converted to monomials in u in [-1, 1])
std::vector<double> fit_pieces(const std::function<double(double)>& f, int ni, int deg) {
  const int n = deg + 1;
  std::vector<double> out((size_t)ni * n, 0.0);
  for (int i = 0; i < ni; ++i) {
    const double a = double(i) / ni, b = double(i + 1) / ni;
    std::vector<double> fv(n), ch(n, 0.0);
    for (int j = 0; j < n; ++j) fv[j] = f(0.5 * (a + b) + 0.5 * (b - a) * std::cos(PI * (2 * j + 1) / (2.0 * n)));
    for (int k = 0; k < n; ++k) {
      double sum = 0.0;
      for (int j = 0; j < n; ++j) sum += fv[j] * std::cos(k * PI * (2 * j + 1) / (2.0 * n));
      ch[k] = sum * (k ? 2.0 : 1.0) / n;
    }
    std::vector<double> T0(n, 0.0), T1(n, 0.0), T2(n, 0.0);
    double* mono = out.data() + (size_t)i * n;
    T0[0] = 1.0;
    for (int j = 0; j < n; ++j) mono[j] += ch[0] * T0[j];
    if (n > 1) {
      T1[1] = 1.0;
      for (int j = 0; j < n; ++j) mono[j] += ch[1] * T1[j];
    }
    for (int k = 2; k < n; ++k) {
      for (int j = 0; j < n; ++j) T2[j] = (j ? 2.0 * T1[j - 1] : 0.0) - T0[j];
      for (int j = 0; j < n; ++j) mono[j] += ch[k] * T2[j];
      T0 = T1;
      T1 = T2;
    }
  }
  return out;
}

int fft_size(int want) {  // smallest 2^a 3^b 5^c 7^d >= want, even
  for (int m = std::max(want, 2);; ++m) {
    if (m & 1) continue;
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}
}  // namespace

void Context::ewald(const Plan& P, int64_t ns, const double* src, int64_t nt, const double* tgt, const double* str,
                    double* u, int level, bool device_ptrs, double* info) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  prob_.ready = false;
  begun_ = false;
  if (P.kernel != kStokeslet || P.dim != 3)
    throw InvalidArgument("ewald: the FFT Ewald path covers the 3D Stokeslet");
  check_inputs(P, 3, ns, nt, 1);
  tab_ = tab_override_ ? tab_override_ : &tables_for(P);
  if (tab_->win.kind != kProlate) throw InvalidArgument("ewald: needs a prolate split window");
  const int d = 3, sc = 3;
  const bool alias = nt == 0;
  const int n = (int)ns, m = alias ? (int)ns : (int)nt;
  cudaEventRecord(ev_[0], st_);
  double* sin = arena_.as<double>("src_in", (size_t)ns * d);
  double* tin = alias ? sin : arena_.as<double>("tgt_in", (size_t)nt * d);
  double* fin = arena_.as<double>("str_in", (size_t)ns * sc);
  copy_in(sin, src, sizeof(double) * ns * d, device_ptrs);
  if (!alias) copy_in(tin, tgt, sizeof(double) * nt * d, device_ptrs);
  copy_in(fin, str, sizeof(double) * ns * sc, device_ptrs);
  int* flags = arena_.as<int>("flags", 8);
  cuda_check(cudaMemsetAsync(flags, 0, 8 * sizeof(int), st_), "memset");
  launch_validate(fin, (int64_t)ns * sc, 1, flags, 2, st_);
  launch_validate(sin, (int64_t)ns * d, 1, flags, 0, st_);
  if (!alias) launch_validate(tin, (int64_t)nt * d, 1, flags, 0, st_);
  launch_wrap(sin, (int64_t)ns * d, st_);  // wrap_into_box (oracle.cpp:133-141)
  if (!alias) launch_wrap(tin, (int64_t)nt * d, st_);
  // Morton sort of sources (and targets) as in build_problem
  auto sort_set = [&](const double* pts, int cnt, const std::string& tag, int*& perm, double*& soa, int32_t*& q) {
    uint64_t* klo = arena_.as<uint64_t>("klo", cnt);
    uint64_t* khi = arena_.as<uint64_t>("khi", cnt);
    uint64_t* klo2 = arena_.as<uint64_t>("klo2", cnt);
    uint64_t* khi2 = arena_.as<uint64_t>("khi2", cnt);
    int* idx = arena_.as<int>("idx", cnt);
    int* idx2 = arena_.as<int>("idx2", cnt);
    perm = arena_.as<int>(tag + "perm", cnt);
    size_t tb = sort_temp_bytes(cnt);
    void* tmp = arena_.get("sort_tmp", tb);
    launch_morton(pts, cnt, d, klo, khi, nullptr, idx, st_);
    sort_morton(cnt, d, klo, khi, idx, klo2, khi2, idx2, perm, tmp, tb, st_);
    soa = arena_.as<double>(tag + "pts", (size_t)cnt * d);
    q = arena_.as<int32_t>(tag + "q", (size_t)cnt * d);
    launch_gather_points(pts, perm, cnt, d, soa, q, st_);
  };
  int *sperm = nullptr, *tperm = nullptr;
  double *spts = nullptr, *tpts = nullptr;
  int32_t *sq = nullptr, *tq = nullptr;
  sort_set(sin, n, "s", sperm, spts, sq);
  double* sstr = arena_.as<double>("sstr", (size_t)ns * sc);
  launch_gather_strengths(fin, sperm, n, sc, sstr, st_);
  if (alias) {
    tperm = sperm;
    tpts = spts;
    tq = sq;
  } else {
    sort_set(tin, m, "t", tperm, tpts, tq);
  }
  // cells at level L: about 200 sources per cell
  int L = level;
  if (L < 0) {
    L = 0;
    while (L < 7 && (double)ns / std::pow(8.0, L + 1) >= 100.0) ++L;
  }
  if (L > 7) throw InvalidArgument("ewald: cell level above 7");
  const int side = 1 << L, ncell = 1 << (3 * L);
  int* sb = arena_.as<int>("ew_sbnd", (size_t)ncell + 1);
  int* tbd = alias ? sb : arena_.as<int>("ew_tbnd", (size_t)ncell + 1);
  launch_cell_bounds(n, sq, L, sb, st_);
  if (!alias) launch_cell_bounds(m, tq, L, tbd, st_);
  int* hb = (int*)pinned_.get("ew_bnd", sizeof(int) * 2 * ((size_t)ncell + 1));
  cuda_check(cudaMemcpyAsync(hb, sb, sizeof(int) * (ncell + 1), cudaMemcpyDeviceToHost, st_), "D2H cells");
  if (!alias)
    cuda_check(cudaMemcpyAsync(hb + ncell + 1, tbd, sizeof(int) * (ncell + 1), cudaMemcpyDeviceToHost, st_),
               "D2H cells");
  int* hflags = (int*)pinned_.get("hflags", 64);
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  if (hflags[2]) throw InvalidArgument("ParticleSystem: non-finite strength");
  if (hflags[0]) throw InvalidArgument("ParticleSystem: non-finite coordinate");
  cudaEventRecord(ev_[1], st_);
  const int* tb_h = alias ? hb : hb + ncell + 1;
  // ---- local part: residual kernel at scale nu = 2^-L over each cell's 27 neighbours (cells are
  // the leaves of a uniform tree; every range at the leaf scale, periodic image shifts)
  std::vector<dev::DBox> boxes(ncell);
  auto cell_xyz = [&](int c, int* xyz) {  // Morton cell index -> integer coordinates
    xyz[0] = xyz[1] = xyz[2] = 0;
    for (int b = 0; b < L; ++b)
      for (int a = 0; a < 3; ++a) xyz[a] |= ((c >> (3 * b + a)) & 1) << b;
  };
  auto cell_id = [&](const int* xyz) {
    int c = 0;
    for (int b = 0; b < L; ++b)
      for (int a = 0; a < 3; ++a) c |= ((xyz[a] >> b) & 1) << (3 * b + a);
    return c;
  };
  const double cside = std::ldexp(1.0, -L);
  for (int c = 0; c < ncell; ++c) {
    int xyz[3];
    cell_xyz(c, xyz);
    dev::DBox& o = boxes[c];
    o.sb = hb[c];
    o.se = hb[c + 1];
    o.tb = tb_h[c];
    o.te = tb_h[c + 1];
    o.level = L;
    o.parent = -1;
    o.first_child = -1;
    o.leaf = 1;
    for (int a = 0; a < 3; ++a)  // tree.cpp:221-228
      o.c[a] = std::ldexp(double(int64_t(xyz[a]) << (kMaxLevel - L)), -kMaxLevel) - 0.5 + 0.5 * cside;
    o.side = cside;
    o.half = 0.5 * cside;
  }
  std::vector<int> leaves, rs(1, 0), rbox, rinfo, chunks;
  for (int c = 0; c < ncell; ++c) {
    if (boxes[c].te == boxes[c].tb) continue;
    const int li = (int)leaves.size();
    leaves.push_back(c);
    int xyz[3];
    cell_xyz(c, xyz);
    auto add = [&](int sbx, const int* sh, bool self) {
      if (boxes[sbx].se == boxes[sbx].sb) return;
      rbox.push_back(sbx);
      rinfo.push_back((sh[0] + 1) + 3 * (sh[1] + 1) + 9 * (sh[2] + 1) + (self ? 64 : 0));  // fine-scale bit 0: nu = r_l
    };
    const int zero[3] = {0, 0, 0};
    add(c, zero, true);
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy && !dz) continue;
          const int dd[3] = {dx, dy, dz};
          int nb[3], sh[3];
          for (int a = 0; a < 3; ++a) {
            const int v = xyz[a] + dd[a];
            sh[a] = v < 0 ? -1 : (v >= side ? 1 : 0);
            nb[a] = v - sh[a] * side;
          }
          add(cell_id(nb), sh, false);
        }
    rs.push_back((int)rbox.size());
    for (int t0 = boxes[c].tb; t0 < boxes[c].te; t0 += 32) {
      chunks.push_back(li);
      chunks.push_back(t0);
    }
  }
  Packer pk;
  const size_t o_boxes = pk.add(boxes), o_leaves = pk.add(leaves), o_rs = pk.add(rs), o_rbox = pk.add(rbox),
               o_rinfo = pk.add(rinfo), o_chunks = pk.add(chunks);
  char* hp = (char*)pinned_.get("ew_lists", pk.total + 64);
  pk.copy_to(hp);
  char* dv = (char*)arena_.get("ew_lists", pk.total + 64);
  cuda_check(cudaMemcpyAsync(dv, hp, pk.total, cudaMemcpyHostToDevice, st_), "ewald lists upload");
  const dev::DBox* dboxes = (const dev::DBox*)(dv + o_boxes);
  int* subr = arena_.as<int>("ew_subrange", (size_t)ncell * 9);
  launch_leaf_subranges(dboxes, ncell, sq, n, d, subr, st_);
  const ResidTables rt = residual_tables(kStokeslet, 3);
  double* ures = arena_.as<double>("ures", (size_t)m * d);
  launch_residual(rt, dboxes, (const int*)(dv + o_leaves), (int)leaves.size(), (const int*)(dv + o_chunks),
                  (int)(chunks.size() / 2), (const int*)(dv + o_rs), (const int*)(dv + o_rbox),
                  (const int*)(dv + o_rinfo), subr, spts, n, sstr, arena_.as<double>("srec", (size_t)n * 6), 1, tpts,
                  m, tperm, alias ? 1 : 0, 0, tab_->self_const, ures, flags + 3, nullptr,
                  arena_.get("res_scratch", residual_scratch_bytes()), st_);
  cudaEventRecord(ev_[2], st_);
  // ---- far part: PSWF-window NUFFT on an Mg^3 grid
  const double nu = cside, c = P.c;
  const int kmax = (int)std::ceil(c / (2.0 * PI * nu) - 1e-12);  // gamma^(k nu) = 0 beyond k nu = c
  const double eps = std::max(P.tol, 1e-14);
  const int w = std::min(16, std::max(4, (int)std::ceil(std::log(100.0 / eps) / (0.75 * PI))));
  const int Mg = fft_size(std::max(2 * (2 * kmax + 1), 2 * w));
  const double cs = 0.75 * PI * w;  // spreading window bandwidth (oversampling 2)
  const WindowFn sw = make_prolate(cs);
  const double phi0 = win_phi(sw, 0.0);
  const int wni = 64, wdeg = 10;
  std::vector<double> wpoly = fit_pieces([&](double z) { return win_phi(sw, z) / phi0; }, wni, wdeg);
  const double h = 1.0 / Mg, alpha = 0.5 * w * h;
  std::vector<double> dfac(kmax + 1);  // h / Phi_1^(k) for the window phi / phi0 scaled by alpha
  for (int k = 0; k <= kmax; ++k) dfac[k] = h * phi0 / (alpha * win_hat(sw, 2.0 * PI * k * alpha));
  const long s2max = 3L * kmax * kmax;
  std::vector<double> A((size_t)s2max + 1, 0.0);  // gamma^(k nu) / k^4, the periodic mollified Stokeslet
  for (long s2 = 1; s2 <= s2max; ++s2) {
    const double k = 2.0 * PI * std::sqrt((double)s2);
    A[s2] = moll_hat(tab_->win, k * nu) / (k * k * k * k);
  }
  Packer pk2;
  const size_t o_w = pk2.add(wpoly), o_d = pk2.add(dfac), o_a = pk2.add(A);
  char* hp2 = (char*)pinned_.get("ew_tabs", pk2.total + 64);
  pk2.copy_to(hp2);
  char* dv2 = (char*)arena_.get("ew_tabs", pk2.total + 64);
  cuda_check(cudaMemcpyAsync(dv2, hp2, pk2.total, cudaMemcpyHostToDevice, st_), "ewald tables upload");
  EwGrid g{Mg, w, kmax, s2max, h, 1.0 / h, 1.0 / alpha, wni, wdeg, (const double*)(dv2 + o_w)};
  const size_t M3 = (size_t)Mg * Mg * Mg, S = (size_t)Mg * Mg * (Mg / 2 + 1);
  double* grid = arena_.as<double>("ew_grid", 3 * M3);
  double2* spec = arena_.as<double2>("ew_spec", 3 * S);
  // deterministic spreading (output-stationary 16^3 bricks, sources binned
  // by Morton cells of <= 16 grid points); the atomic form for windows wider
  // than the brick
  int Ls = 0;
  while (Ls < 8 && (double)Mg / (1 << Ls) > 16.0) ++Ls;
  const bool tiled = ew_spread_tiled_ok(g, Ls);
  if (tiled) {
    int* sbc = arena_.as<int>("ew_sbc", ((size_t)1 << (3 * Ls)) + 1);
    launch_cell_bounds(n, sq, Ls, sbc, st_);
    launch_ew_spread_tiled(g, Ls, sbc, n, spts, sstr, grid, st_);
  } else {
    cuda_check(cudaMemsetAsync(grid, 0, sizeof(double) * 3 * M3, st_), "memset grid");
    launch_ew_spread(g, n, spts, sstr, grid, st_);
  }
  fft_.plan(Mg, 3, st_);
  fft_.forward(grid, spec);
  launch_ew_symbol(g, spec, (const double*)(dv2 + o_a), (const double*)(dv2 + o_d), st_);
  fft_.inverse(spec, grid);
  double* ufar = arena_.as<double>("ufar", (size_t)m * d);
  launch_ew_gather(g, m, tpts, tperm, grid, arena_.get("ew_gi", M3 * 4 * sizeof(double)), ufar, st_);
  cudaEventRecord(ev_[3], st_);
  double* du = device_ptrs ? u : arena_.as<double>("u", (size_t)m * d);
  launch_combine(m, d, ufar, ures, nullptr, 0.0, nullptr, nullptr, nullptr, du, st_);
  if (!device_ptrs) copy_out(u, du, sizeof(double) * m * d);
  cudaEventRecord(ev_[4], st_);
  cuda_check(cudaMemcpyAsync(hflags, flags, 8 * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H flags");
  sync();
  cuda_check(cudaGetLastError(), "ewald kernels");
  if (hflags[3]) throw DomainError("residual_pass: coincident points");
  if (info) {
    info[0] = L;
    info[1] = Mg;
    info[2] = w;
    info[3] = kmax;
    info[4] = ev_ms(0, 1);
    info[5] = ev_ms(1, 2);
    info[6] = ev_ms(2, 3);
    info[7] = ev_ms(0, 4);
  }
}

}  // namespace sdmkb
