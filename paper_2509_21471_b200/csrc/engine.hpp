// The B200 DMK engine: owns the device, stream, buffers and the current
// problem; implements evaluate_with_plan (dmk.cpp:1036-1117) and the
// pass-level entry points of dmk.hpp on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sdmk.h"
#include "host/comm.hpp"
#include "host/fft.hpp"
#include "host/setup.hpp"
#include "host/tree.hpp"
#include "kernels/launch.hpp"

namespace sdmkb {

struct CudaError : std::exception {
  std::string msg;
  explicit CudaError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
struct OomError : std::exception {
  std::string msg;
  explicit OomError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

void cuda_check(cudaError_t e, const char* what);

// Grow-only named device buffers (cudaMalloc is far too slow per call).
class Arena {
 public:
  ~Arena();
  void* get(const std::string& name, size_t bytes);
  template <class T>
  T* as(const std::string& name, size_t count) { return static_cast<T*>(get(name, count * sizeof(T))); }
  size_t bytes() const;
  // Guard mode (a memcheck / initcheck stand-in for pools where
  // compute-sanitizer is closed): every buffer is allocated at exactly its
  // requested size between two 64 KB canary regions, and its contents are
  // poisoned with all-ones bytes (a NaN in every double, -1 in every integer)
  // so a read of an element no kernel wrote reaches the result.  check()
  // returns the names of buffers whose canaries were overwritten.
  void set_guard(bool on);
  bool guard() const { return guard_; }
  std::vector<std::string> check() const;
  // writes one byte past the end of a scratch buffer and one before its
  // start, and reports whether check() names it (the detector's self-test)
  bool selftest();

 private:
  static constexpr size_t kGuard = 64 * 1024;
  struct Buf {
    void* base;    // cudaMalloc'd pointer
    size_t alloc;  // bytes allocated
    size_t req;    // bytes the caller may touch (guard mode)
  };
  bool guard_ = false;
  std::map<std::string, Buf> bufs_;
};

class Pinned {
 public:
  ~Pinned();
  void* get(const std::string& name, size_t bytes);

 private:
  std::map<std::string, std::pair<void*, size_t>> bufs_;
};

// Device copy of one plane-wave grid (PWGrid + its arrays in one blob).
struct GridDev {
  PWGrid g{};
  int key_N = -1, key_p = -1, key_dim = -1;
  double key_theta = 0.0, key_band = -1.0;
  std::vector<int> col_lz_host;
};

struct Problem {
  bool ready = false;
  Plan plan;
  bool periodic = false;
  int dim = 3, nch = 3, sc = 3;
  int ns = 0, nt = 0;  // nt == ns when aliased
  bool alias = true;
  HostTree tree;
  // device views (arena-owned)
  double *spts = nullptr, *sstr = nullptr, *tpts = nullptr, *tpts_caller = nullptr;
  int *sperm = nullptr, *tperm = nullptr;
  const int32_t *sq = nullptr, *tq = nullptr;  // sorted quantized coordinates (device, SoA)
  // tree lists on device
  dev::DBox* boxes = nullptr;
  int *ant_leaves = nullptr, *int_leaves = nullptr;
  int n_ant = 0, n_int = 0;
  int *rng_start = nullptr, *rng_box = nullptr, *rng_info = nullptr, *subrange = nullptr;
  int64_t t_own0 = 0, t_own1 = 0;  // owned range of Morton-sorted targets (set_shard)
  std::vector<int64_t> t_bounds;   // every rank's owned range (nranks + 1), for the u all-gather
  int64_t* d_bounds = nullptr;
  // distributed upward pass (multi-GPU with an exchange): each rank forms the
  // outgoing expansions of its own cut subtrees, receives the halo it reads
  // and every cut box, and merges the boxes above the cut itself
  bool halo = false;
  HaloPlan hp;
  std::vector<int64_t> send_off, recv_off;  // per peer, in doubles
  int *send_ids = nullptr, *recv_ids = nullptr;
  int n_send = 0, n_recv = 0;
  bool lists_b = false;            // downward / residual lists uploaded
  int* res_chunks = nullptr;       // (leaf index, first target) per 32-target residual chunk
  int n_chunks = 0;
  struct LevelLists {
    int n_merge = 0, n_interp = 0, n_src = 0, n_tgt = 0;
    int *merge_out = nullptr, *merge_in = nullptr, *merge_ci = nullptr;
    int n_top = 0;  // merges above the cut (halo mode), after the exchange
    int *top_out = nullptr, *top_in = nullptr, *top_ci = nullptr;
    int *interp_in = nullptr, *interp_out = nullptr, *interp_ci = nullptr, *interp_seg = nullptr;
    int n_interp_seg = 0;
    int *src_boxes = nullptr, *tgt_boxes = nullptr;
    int *ent_start = nullptr, *ent_slot = nullptr, *ent_tau = nullptr;
    int max_entries = 0;
    // sibling groups for the plane-wave accumulation (empty: per-target kernel)
    std::vector<int> grp_start_h;  // host copy of grp_tstart, for chunking
    int *grp_tstart = nullptr, *grp_slot = nullptr, *t_meta = nullptr;
  };
  std::vector<LevelLists> levels;
};

class Context {
 public:
  explicit Context(int device);
  ~Context();

  void load_tables(const std::string& path);
  const Tables& tables_for(const Plan& plan);
  // Target sharding for multi-GPU runs (one process per GPU): rank owns a
  // contiguous Morton run of target leaves; outputs of other ranks' targets
  // are written as zeros, so a sum over ranks assembles the full result.
  void set_shard(int rank, int nranks);
  // NCCL communicator of this rank (one process per GPU): evaluations then
  // exchange outgoing expansions instead of replicating the upward pass, and
  // return the assembled u on every rank (all-reduce on the context stream).
  void comm_init(int rank, int nranks, const unsigned char* id);
  // Test / projection mode without NCCL: evaluate_begin stops after packing
  // the halo, the caller moves the slabs (halo_transfer), evaluate_end
  // finishes; u holds this rank's targets only (zeros elsewhere).
  void set_manual_exchange(bool on);
  void evaluate_begin(const Plan& plan, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                      const double* str, int mode, bool device_ptrs);
  void evaluate_end(double* u, sdmk_report* rep);
  // device slab this rank sends to / receives from `peer` (count in doubles)
  void halo_slab(int peer, bool recv, double** ptr, int64_t* count);
  int shard_rank() const { return rank_; }

  // Host-pointer evaluation; u may be host memory.  report may be null.
  void evaluate(const Plan& plan, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
                const double* str, int mode, double* u, sdmk_report* rep, bool device_ptrs);

  // pass-level API
  void setup(const Plan& plan, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt,
             const double* str, int mode);
  const Problem& problem() const { return prob_; }
  // the reference's tree dump needs coarse / fine lists of every box
  std::string tree_dump() {
    finish_topology(prob_.tree, true);
    return dump_topology(prob_.tree);
  }
  cudaStream_t stream() const { return st_; }
  // guard mode (Arena::set_guard): only on a context that has not allocated yet
  void set_guard(bool on) {
    if (arena_.bytes() > 0 && on != arena_.guard())
      throw InvalidArgument("sdmk_set_guard: call before the context's first setup or evaluation");
    arena_.set_guard(on);
  }
  std::vector<std::string> guard_check() const { return arena_.check(); }
  bool guard_selftest() { return arena_.selftest(); }
  void upward(double* host_out);
  void incoming(int stage, double* host_out);
  void target_far(double* host_out);
  void residual(double* host_out);

  // ---- the reference's pass-level API, tree first (tree.hpp:90-104,
  // dmk.hpp:84-131): build_tree, then each pass with its own plan, tables,
  // strengths and proxies passed in and out as host arrays ----
  void tree_build(int dim, bool periodic, int n_s, int p, int64_t ns, const double* src, int64_t nt,
                  const double* tgt);
  // counts[3 b + k] = entries of list k (colleague / coarse / fine) of box b;
  // entries (may be null) = 4 int32 per entry (box, shift0..2), box-major
  void tree_neighbors(int64_t* counts, int32_t* entries);
  // permuted point copies (point-major) and quantized coordinates (3 per point)
  void tree_sorted(double* src_pts, double* tgt_pts, int32_t* src_q, int32_t* tgt_q);
  void tree_perm(int32_t* src_perm, int32_t* tgt_perm);
  void pass_upward(const Plan& P, int64_t nstr, const double* str, double* outgoing);
  void pass_root(const Plan& P, const Tables* tab, int64_t nog, const double* og, bool periodic, int64_t nin,
                 double* in);
  void pass_downward(const Plan& P, const Tables* tab, int64_t nog, const double* og, bool periodic, int64_t nin,
                     double* in);
  void pass_target_far(const Plan& P, int64_t nin, const double* in, double* u);
  void pass_residual(const Plan& P, const Tables* tab, int64_t nstr, const double* str, bool periodic, double* u);
  // FFT Ewald: periodic 3D Stokeslet, single-level
  // split at nu = 2^-level (level < 0: chosen from N), local part by the
  // residual kernel over the 27 neighbour cells, far part by a PSWF-window
  // NUFFT on a uniform grid with cuFFT.  Host or device pointers; info[8]
  // (may be null) receives level, grid size, window width, kappa_max and
  // the times (ms) of sort, local, far, total.
  void ewald(const Plan& P, int64_t ns, const double* src, int64_t nt, const double* tgt, const double* str,
             double* u, int level, bool device_ptrs, double* info);
  // tables from an SDMKSPLT v1 memory image (cached by content)
  const Tables& tables_image(const void* bytes, size_t n);
  // tables an evaluation uses instead of the plan's (the reference's
  // evaluate_with_plan(..., tables)); null restores the plan's
  void set_tables_override(const Tables* t) { tab_override_ = t; }

  // O(N*M) reference sums on the GPU: direct_sum (tab == nullptr; exact
  // kernels) and direct_residual_sum (residual kernel of `tab` at scale
  // cutoff, periodic images), oracle.cpp:143-241.  Inputs are the caller's
  // point-major arrays; u is host or device memory as device_ptrs says.
  void direct(int kernel, int dim, int64_t ns, const double* src, int64_t nt, const double* tgt, const double* str,
              const Tables* tab, double cutoff, bool periodic, double* u, bool device_ptrs);

 private:
  void check_inputs(const Plan& plan, int dim, int64_t ns, int64_t nt, int mode);
  void bind_plan(const Plan& P, const Tables* tab, const char* who);
  void load_strengths(int64_t nstr, const double* str, const char* who);
  // inputs already in the arena ("src_in", "tgt_in", "str_in"): validate, wrap, sort, topology, upload
  void build_problem(const Plan& plan, int dim, int ns, int nt, int mode, bool defer_lists = false);
  void upload_tree_lists_a();
  void upload_tree_lists_b();
  void run_upward();
  void run_upward_top();
  void run_root();
  void run_downward();
  void run_target_far(double* ufar);
  void run_residual(double* ures, bool stats, int reserve_sms = 0);
  ResidTables residual_tables(int kernel, int dim);
  GridDev& grid(GridDev& cache, const std::string& name, int dim, int p, int N, double theta, double band_r2);
  void sync();
  double ev_ms(int a, int b);
  void copy_in(void* dst, const void* src, size_t bytes, bool device_ptrs);
  void copy_out(void* dst, const void* src, size_t bytes);
  void stage_events();
  std::vector<cudaEvent_t> stage_ev_;

  int device_;
  cudaStream_t st_ = nullptr;
  cudaStream_t st2_ = nullptr;     // side stream: strengths H2D overlapping the tree build
  bool lists_side_ = false;        // upload_tree_lists_b issues its device work on st2_ (evaluate_begin)
  cudaEvent_t str_ev_ = nullptr;
  cudaEvent_t x_ev_ = nullptr;     // the NCCL halo exchange on st2_ is done
  bool x_pending_ = false;         // an exchange is in flight (evaluate with a communicator)
  bool str_pending_ = false;       // strengths copy in flight on st2_
  cudaEvent_t ev_[20];
  bool interp_timed_ = false, anterp_timed_ = false;  // the DMMA kernels ran this call (events 16-19)
  Arena arena_;
  Pinned pinned_;
  std::map<std::string, Tables> tables_;
  const Tables* tab_ = nullptr;
  Problem prob_;
  GridDev grid_lev_, grid_root_;
  int launches_ = 0;
  int *root_dev_ids_ = nullptr, *root_dev_es_ = nullptr, *root_dev_slot_ = nullptr, *root_dev_tau_ = nullptr;
  const double *cheb_nodes_ = nullptr, *cheb_wts_ = nullptr, *mats_up_ = nullptr, *mats_down_ = nullptr;
  std::vector<cudaEvent_t> pw_ev_;
  int pw_used_ = 0;
  double planewave_ms();
  int rank_ = 0, nranks_ = 1;
  std::unique_ptr<Comm> comm_;
  bool manual_x_ = false;
  bool halo_run_ = false;  // the current evaluation exchanges outgoing expansions
  bool begun_ = false;     // between evaluate_begin and evaluate_end
  struct Call {
    int dim = 3, sc = 3, ntt = 0;
    int64_t ns = 0, nt = 0;
    bool alias = true, device_ptrs = false;
  } call_;
  bool zero_all_ = true;  // zero whole proxy arrays (pass-level API returns them)
  bool tree_only_ = false;     // build_problem for build_tree: no wrap, build_tree's checks
  bool accumulate_down_ = false;  // downward interpolation adds to the children (pass-level API)
  bool force_tbasis_ = false;  // target bases recomputed (the upward pass may not have run)
  const Tables* tab_override_ = nullptr;
  Fft3 fft_;
  std::map<std::string, Tables> image_tables_;
  std::map<std::pair<const Tables*, int>, std::pair<PiecewisePoly, PiecewisePoly>> pw_cache_;
  const int32_t* hq_ = nullptr;  // pinned sorted quantized coordinates of the current problem
  unsigned long long stats_[3] = {0, 0, 0};
};

}  // namespace sdmkb
