/*
 * sdmk.h -- C-ABI of the B200-native DMK hot path (libsdmk_b200.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * Every entry point returns an sdmk_status (0 = success) and never throws;
 * sdmk_last_error() describes the last failure on the calling thread.  The
 * C++ drop-in header include/stokesdmk_b200/dmk.hpp maps these codes back to
 * the reference's exception types.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference's proj/core):
 *
 *   sdmk_select_parameters   stokesdmk::select_parameters     include/stokesdmk/dmk.hpp:50-51, src/params.cpp:60-115
 *   sdmk_outgoing_channels   stokesdmk::outgoing_channels     dmk.hpp:59, params.cpp:117-125
 *   sdmk_evaluate_with_plan  stokesdmk::evaluate_with_plan    dmk.hpp:151-155, dmk.cpp:1036-1117
 *   sdmk_evaluate            stokesdmk::evaluate              dmk.hpp:159-161, dmk.cpp:1119-1124
 *   sdmk_evaluate_device     (device-resident variant of evaluate_with_plan; inputs/outputs in HBM)
 *   sdmk_setup               stokesdmk::build_tree + validate_system/wrap_into_box
 *                            (tree.hpp:90-92, oracle.hpp:54-58): builds the tree of one problem
 *                            in the context so the pass-level entry points can run on it
 *   sdmk_tree_info/boxes/perm/dump   Tree fields + dump_tree (tree.hpp:52-81, 104)
 *   sdmk_upward_pass         stokesdmk::upward_pass           dmk.hpp:84-85, dmk.cpp:555-655
 *   sdmk_incoming            make_incoming + root_far_field (+ downward_pass)  dmk.hpp:88-112
 *   sdmk_target_far_fields   stokesdmk::target_far_fields     dmk.hpp:116-117, dmk.cpp:861-915
 *   sdmk_residual_pass       stokesdmk::residual_pass         dmk.hpp:128-131, dmk.cpp:919-1032
 *   sdmk_load_tables / sdmk_save_tables   import/export_split_kernel (split.hpp:153-154, SDMKSPLT v1)
 *   sdmk_tree_build          stokesdmk::build_tree            tree.hpp:90-92, tree.cpp:230-298
 *   sdmk_tree_neighbors      neighbor_query / Tree::neighbors tree.hpp:44-51, 95
 *   sdmk_tree_sorted         Tree::src_points/tgt_points/src_q/tgt_q  tree.hpp:74-78
 *   sdmk_pass_upward         stokesdmk::upward_pass           dmk.hpp:84-85
 *   sdmk_pass_root_far_field stokesdmk::root_far_field        dmk.hpp:98-100, dmk.cpp:671-701
 *   sdmk_pass_downward       stokesdmk::downward_pass         dmk.hpp:110-112, dmk.cpp:705-857
 *   sdmk_pass_target_far_fields  stokesdmk::target_far_fields dmk.hpp:116-117
 *   sdmk_pass_residual       stokesdmk::residual_pass         dmk.hpp:128-131
 *   sdmk_evaluate_with_tables  evaluate_with_plan(..., const SplitKernel* tables)  dmk.hpp:151-155
 *   sdmk_host_build_tables   stokesdmk::build_split_kernel    split.hpp:89-90, split.cpp:319-396
 *   sdmk_ewald               (new: FFT Ewald for the periodic Stokeslet; ewald_reference's split, ewald.cpp:81-272)
 *   sdmk_direct_sum          stokesdmk::direct_sum            oracle.hpp:60-65, oracle.cpp:143-179
 *   sdmk_direct_residual_sum stokesdmk::direct_residual_sum   oracle.hpp:67-75, oracle.cpp:181-241
 *
 * Enumerations use the reference's enumerator order:
 *   kernel: 0 stokeslet, 1 stresslet, 2 rotlet  (KernelType, split.hpp:28)
 *   window: 0 prolate, 1 gaussian               (WindowKind, windows.hpp:19)
 *   mode:   0 free_space, 1 periodic            (EwaldMode, oracle.hpp:82)
 */
#ifndef SDMK_H
#define SDMK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sdmk_status {
  SDMK_OK = 0,
  SDMK_EINVAL = 1,   /* std::invalid_argument in the reference */
  SDMK_EDOMAIN = 2,  /* std::domain_error (coincident points) */
  SDMK_ERUNTIME = 3, /* std::runtime_error (I/O, fit non-convergence) */
  SDMK_ECUDA = 4,    /* CUDA runtime / launch failure */
  SDMK_EOOM = 5      /* device allocation failed */
} sdmk_status;

/* Field order and meaning of stokesdmk::DmkPlan (dmk.hpp:27-40). */
typedef struct sdmk_plan {
  int32_t kernel;
  int32_t dim;
  int32_t window;
  double tol;
  double c;
  double sigma;
  int32_t p;
  int32_t N1;
  int32_t N_per;
  int32_t n_s;
  double table_tol;
} sdmk_plan;

/* stokesdmk::DmkReport (dmk.hpp:134-145) plus device-side detail.  The
   t_* fields are seconds of the same passes as the reference report, taken
   with CUDA events on the context stream. */
typedef struct sdmk_report {
  int32_t num_boxes;
  int32_t max_level;
  int32_t num_sources;
  int32_t num_targets;
  double t_tree;
  double t_upward;
  double t_root;
  double t_downward;
  double t_residual;
  /* extras */
  double t_h2d;          /* host->device copies (host-pointer entry points) */
  double t_d2h;          /* device->host copy of u */
  double t_total;        /* whole call, CUDA events */
  int64_t p2p_candidates; /* source-target pairs tested in the residual kernel */
  int64_t p2p_in_support; /* pairs evaluated (r < nu * support) */
  int32_t kernel_launches;
  double t_residual_kernel; /* residual kernel alone */
  double t_planewave;       /* forward/accumulate/inverse kernels of the downward pass */
  double t_exchange;        /* multi-GPU: halo pack + exchange + unpack of outgoing expansions */
  int64_t halo_bytes_sent;  /* multi-GPU: outgoing-expansion bytes this rank sent / received */
  int64_t halo_bytes_recv;
  double t_interp_kernel;   /* target interpolation kernel alone (DMMA path; 0 otherwise) */
  double t_anterp_kernel;   /* leaf anterpolation kernel alone (DMMA path; 0 otherwise) */
} sdmk_report;

typedef struct sdmk_context sdmk_context;

int sdmk_create(int device, sdmk_context** out);
int sdmk_destroy(sdmk_context* ctx);
const char* sdmk_last_error(void);
/* 1 when the library was built for and is running on an sm_100 device */
int sdmk_device_ok(int device);

int sdmk_select_parameters(int kernel, double eps, int window, int dim, sdmk_plan* out);
int sdmk_outgoing_channels(int kernel, int dim);
int sdmk_strength_components(int kernel, int dim);

/* Split tables: built from the plan on first use and cached in the context
   (keyed by kernel/dim/window/c|sigma/table_tol).  load/save use the
   reference's SDMKSPLT v1 format, so a table cache written by either library
   can be read by the other. */
int sdmk_load_tables(sdmk_context* ctx, const char* path);
int sdmk_save_tables(sdmk_context* ctx, const sdmk_plan* plan, const char* path);

/* Full evaluation from HOST buffers (caller point order, point-major AoS as in
   ParticleSystem, oracle.hpp:29-46).  n_tgt == 0 (tgt may be NULL) means the
   targets alias the sources.  u receives dim * max(n_tgt, n_src-if-alias)
   doubles.  report may be NULL. */
int sdmk_evaluate_with_plan(sdmk_context* ctx, const sdmk_plan* plan, int dim, int64_t n_src,
                            const double* src, int64_t n_tgt, const double* tgt, const double* str,
                            int mode, double* u, sdmk_report* report);

int sdmk_evaluate(sdmk_context* ctx, int kernel, int dim, int64_t n_src, const double* src,
                  int64_t n_tgt, const double* tgt, const double* str, double eps, int window,
                  int mode, double* u, sdmk_report* report);

/* Same as sdmk_evaluate_with_plan with every array already in device memory
   (the device-resident "value" path of the benchmark). */
int sdmk_evaluate_device(sdmk_context* ctx, const sdmk_plan* plan, int dim, int64_t n_src,
                         const double* d_src, int64_t n_tgt, const double* d_tgt,
                         const double* d_str, int mode, double* d_u, sdmk_report* report);

/* ---- pass-level API on one problem held by the context ---- */
int sdmk_setup(sdmk_context* ctx, const sdmk_plan* plan, int dim, int64_t n_src, const double* src,
               int64_t n_tgt, const double* tgt, const double* str, int mode);
/* info[7]: num_boxes, max_level, n_src, n_tgt, alias, depth_capped, channels */
int sdmk_tree_info(sdmk_context* ctx, int32_t* info);
/* 11 int32 per box: level parent first_child leaf a0 a1 a2 src_begin src_end tgt_begin tgt_end */
int sdmk_tree_boxes(sdmk_context* ctx, int32_t* out);
int sdmk_tree_perm(sdmk_context* ctx, int32_t* src_perm, int32_t* tgt_perm);
/* returns the dump length; copies at most cap bytes into buf (may be NULL) */
int64_t sdmk_tree_dump(sdmk_context* ctx, char* buf, int64_t cap);
/* outgoing proxies: num_boxes * channels * p^dim doubles (ProxyData layout) */
int sdmk_upward_pass(sdmk_context* ctx, double* outgoing);
/* incoming proxies: num_boxes * dim * p^dim doubles; stage 0 = root far field
   only, 1 = after the downward pass */
int sdmk_incoming(sdmk_context* ctx, int stage, double* incoming);
int sdmk_target_far_fields(sdmk_context* ctx, double* u);
int sdmk_residual_pass(sdmk_context* ctx, double* u);

/* ---- the reference's tree-first pass-level API ----
   One tree per context: sdmk_tree_build replaces build_tree (tree.hpp:90-92,
   tree.cpp:230-298) -- no wrap, points must lie in [-1/2, 1/2]^dim, the
   reference's messages -- and the sdmk_pass_* functions replace the passes
   of dmk.hpp:84-131 with the plan, split tables, strengths and proxies the
   caller holds (ProxyData layout: boxes x channels x p^dim, axis 0 fastest,
   host memory).  The tree's fields come back through sdmk_tree_info /
   sdmk_tree_boxes / sdmk_tree_perm / sdmk_tree_dump above and: */
int sdmk_tree_build(sdmk_context* ctx, int dim, int periodic, int n_s, int proxy_order, int64_t n_src,
                    const double* src, int64_t n_tgt, const double* tgt);
/* TreeNeighbors (tree.hpp:44-51): counts[3*b + k] = length of list k
   (0 colleagues, 1 coarse, 2 fine) of box b; entries (NULL: counts only) =
   4 int32 per entry (box, shift[0..2]) in box order, lists in that order */
int sdmk_tree_neighbors(sdmk_context* ctx, int64_t* counts, int32_t* entries);
/* Tree::src_points / tgt_points (point-major) and src_q / tgt_q (3 int32 per
   point, zero third axis in 2D); any output may be NULL */
int sdmk_tree_sorted(sdmk_context* ctx, double* src_points, double* tgt_points, int32_t* src_q, int32_t* tgt_q);
/* upward_pass (dmk.hpp:84-85): strengths in caller order, n_str doubles */
int sdmk_pass_upward(sdmk_context* ctx, const sdmk_plan* plan, int64_t n_str, const double* str,
                     double* outgoing);
/* root_far_field (dmk.hpp:98-100): incoming (n_in doubles) += root far field.
   tables: an SDMKSPLT v1 image (the SplitKernel), or NULL for the plan's */
int sdmk_pass_root_far_field(sdmk_context* ctx, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                             int64_t n_out, const double* outgoing, int periodic, int64_t n_in, double* incoming);
/* downward_pass (dmk.hpp:110-112): incoming updated in place */
int sdmk_pass_downward(sdmk_context* ctx, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                       int64_t n_out, const double* outgoing, int periodic, int64_t n_in, double* incoming);
/* target_far_fields (dmk.hpp:116-117): u = dim * targets doubles, caller order */
int sdmk_pass_target_far_fields(sdmk_context* ctx, const sdmk_plan* plan, int64_t n_in, const double* incoming,
                                double* u);
/* residual_pass (dmk.hpp:128-131); coincident points -> SDMK_EDOMAIN */
int sdmk_pass_residual(sdmk_context* ctx, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                       int64_t n_str, const double* str, int periodic, double* u);
/* evaluate_with_plan(plan, sys, mode, report, &tables) (dmk.hpp:151-155) with
   the caller's split tables as an SDMKSPLT v1 image (NULL: the plan's) */
int sdmk_evaluate_with_tables(sdmk_context* ctx, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                              int dim, int64_t n_src, const double* src, int64_t n_tgt, const double* tgt,
                              const double* str, int mode, double* u, sdmk_report* report);
/* build_split_kernel(kernel, dim, build_prolate(c) | build_gaussian(sigma), tol)
   (split.cpp:319-396) on the host: writes the SDMKSPLT v1 image (at most cap
   bytes; buf may be NULL) and returns its length, -1 on error */
int64_t sdmk_host_build_tables(int kernel, int dim, int window, double c, double sigma, double tol,
                               unsigned char* buf, int64_t cap);
/* build_prolate(c) / build_gaussian(sigma) (windows.cpp): scalars[5] =
   lambda0, norm_r, trunc_error, psi0, chi0; coeffs (at most cap) = the
   Legendre coefficients; returns their count, -1 on error */
int sdmk_host_build_window(int window, double c, double sigma, double* scalars, double* coeffs, int cap);
/* window_eval (what 0), window_deriv (1), window_fourier (2), phi_tail (3),
   mollifier_fourier (4) of a window given by its fields, at n points */
int sdmk_host_window_eval(int window, double c, double sigma, const double* coeffs, int ncoef,
                          const double* scalars, int what, int64_t n, const double* x, double* out);
/* direct_residual_sum(sk, sys, cutoff, periodic) with the caller's tables */
int sdmk_direct_residual_sum_tables(sdmk_context* ctx, const unsigned char* tables, int64_t nbytes, int dim,
                                    int64_t n_src, const double* src, int64_t n_tgt, const double* tgt,
                                    const double* str, double cutoff, int periodic, double* u);

/* ---- FFT Ewald (no reference counterpart:
   SPEC.md lists it as "noted but not built") ----
   The periodic 3D Stokeslet sum by the single-level split of
   ewald_reference (ewald.cpp:81-272) at scale nu = 2^-level instead of 1:
   u = residual sum over pairs closer than nu (the residual kernel over each
   cell's 27 periodic neighbour cells) + the mollified far field
   sum_{kappa != 0} gamma^(|k| nu) / k^4 (k^2 f^ - k (k . f^)) e^{i k x}
   (a prolate-window NUFFT on a uniform grid, cuFFT, opened at run time)
   + the self term (targets aliased).  The plan supplies the window (c) and
   tolerance; the zero mode is dropped as in periodic DMK (net force zero).
   level < 0 chooses ~200 sources per cell.  Host (sdmk_ewald) or device
   (sdmk_ewald_device) buffers, caller point order; n_tgt == 0 aliases.
   info (8 doubles, may be NULL): level, grid points per axis, window width,
   kappa_max, and times in ms (sort, local, far, total). */
int sdmk_ewald(sdmk_context* ctx, const sdmk_plan* plan, int64_t n_src, const double* src, int64_t n_tgt,
               const double* tgt, const double* str, double* u, int level, double* info);
int sdmk_ewald_device(sdmk_context* ctx, const sdmk_plan* plan, int64_t n_src, const double* d_src, int64_t n_tgt,
                      const double* d_tgt, const double* d_str, double* d_u, int level, double* info);

/* ---- O(N*M) reference sums on the GPU ----
   Same per-target source order, Kahan accumulation and unfused expression
   trees as the reference (3D results are bitwise equal to it; the 2D
   Stokeslet's log may differ by 1 ulp per pair).  Host buffers in caller
   point order; n_tgt == 0 aliases (self pairs excluded).  direct_sum:
   exact free-space kernels, coincident points -> SDMK_EDOMAIN.
   direct_residual_sum: the plan's residual kernel at scale `cutoff`
   (0 < cutoff, <= 1 when periodic), image shifts {-1,0,1}^dim when
   periodic (inputs wrapped first). */
int sdmk_direct_sum(sdmk_context* ctx, int kernel, int dim, int64_t n_src, const double* src, int64_t n_tgt,
                    const double* tgt, const double* str, double* u);
int sdmk_direct_residual_sum(sdmk_context* ctx, const sdmk_plan* plan, int dim, int64_t n_src, const double* src,
                             int64_t n_tgt, const double* tgt, const double* str, double cutoff, int periodic,
                             double* u);
/* ---- multi-GPU (one process per GPU) ----
   Shard the following evaluations by target leaves:
   rank owns a contiguous Morton run of target leaves (balanced by a cost
   model of its near-field pairs and plane-wave boxes).  Without a
   communicator (sdmk_comm_init below) the upward pass stays replicated, the
   downward, far-field and residual passes run only for the owned leaves and
   their ancestors, and u is written as zeros for other ranks' targets, so an
   element-wise sum over ranks (an all-reduce) is the full result, bitwise
   equal to nranks = 1.  No reference counterpart (the reference is a
   single-process library). */
int sdmk_set_shard(sdmk_context* ctx, int rank, int nranks);

/* Distributed upward pass ("source halos exchanged").
   sdmk_comm_unique_id on rank 0 (128 bytes, shared with the other ranks by
   any means, e.g. torch.distributed), then sdmk_comm_init on every rank:
   the context gets an NCCL communicator (libnccl.so.2 opened at run time)
   and fixes (rank, nranks) as sdmk_set_shard would.  Evaluations then
   (1) anterpolate and merge only this rank's cut subtrees (the tree is cut
   into subtrees of <= N/(8 nranks) sources, dealt to ranks in Morton runs),
   (2) exchange, in one NCCL group on the context stream, the outgoing
   expansions every other rank reads (colleagues of its plane-wave targets)
   plus all cut boxes, (3) merge the boxes above the cut on every rank, run
   the sharded downward / far-field / residual passes, and (4) all-gather
   every rank's owned Morton range of u (sdmk_host_shard_bounds) and scatter
   it to caller order, so every rank returns the full result, bitwise equal
   to nranks = 1. */
int sdmk_comm_unique_id(unsigned char id[128]);
int sdmk_comm_init(sdmk_context* ctx, int rank, int nranks, const unsigned char id[128]);
/* The same evaluation without NCCL, in two halves, for tests and per-rank
   timing on one GPU: with manual exchange on (and nranks > 1 from
   sdmk_set_shard), sdmk_evaluate_begin runs everything up to the packed
   halo; sdmk_halo_transfer(from, to) copies `from`'s slab for `to` into
   `to`'s receive slab (device to device); sdmk_evaluate_end finishes and
   writes u for this rank's targets only (zeros elsewhere; no all-reduce).
   report->t_total then excludes the time between begin and end. */
int sdmk_set_manual_exchange(sdmk_context* ctx, int on);
int sdmk_evaluate_begin(sdmk_context* ctx, const sdmk_plan* plan, int dim, int64_t n_src, const double* src,
                        int64_t n_tgt, const double* tgt, const double* str, int mode, int device_ptrs);
int sdmk_halo_transfer(sdmk_context* from, sdmk_context* to);
int sdmk_evaluate_end(sdmk_context* ctx, double* u, sdmk_report* report);

/* ---- instrumentation ----
   the context's CUDA stream (cudaStream_t) so callers can time on it */
int sdmk_get_stream(sdmk_context* ctx, void** stream);
/* measured FP64 FMA throughput of the device (TFLOP/s, best of 5) */
int sdmk_fp64_peak(sdmk_context* ctx, double* tflops);
/* the same for the FP64 tensor cores (mma.sync.m8n8k4.f64, the DMMA kernels' roofline) */
int sdmk_fp64_mma_peak(sdmk_context* ctx, double* tflops);
/* guard mode, a memcheck / initcheck stand-in (test infrastructure): on a
   context that has not allocated yet, every device buffer is allocated at
   exactly its requested size between two 64 KB canary regions and is
   poisoned with all-ones bytes (NaN doubles, -1 integers), so a kernel
   writing out of bounds trips a canary and a read of an element nothing wrote
   reaches the result.  sdmk_guard_check returns how many buffers had a canary
   overwritten (their names, newline-separated, into names[cap]), or -1 on
   error. */
int sdmk_set_guard(sdmk_context* ctx, int on);
int64_t sdmk_guard_check(sdmk_context* ctx, char* names, int64_t cap);
/* the detector's self-test on a guarded context: stores one byte past the end
   and one before the start of a scratch buffer; 1 when sdmk_guard_check named
   it both times, 0 when not (or the context is not guarded), -1 on error */
int sdmk_guard_selftest(sdmk_context* ctx);

/* ---- host-only helpers (no GPU needed; used by the CPU test suite) ----
   Plan-level setup exactly as the GPU path uses it. */
int sdmk_host_save_tables(const sdmk_plan* plan, const char* path);
/* symbol table of one grid (dmk.cpp:259-318); kind 0 level_diff, 1 root_free,
   2 root_periodic; out receives s2max + 1 doubles */
int sdmk_host_symbol_table(const sdmk_plan* plan, double h, int s2max, int kind, double r_coarse,
                           double r_fine, double* out);
/* box topology from SORTED quantized coordinates (SoA int32, q[axis*n+i]);
   n_tgt == 0 aliases; returns the dump_tree text length, copies <= cap bytes */
int64_t sdmk_host_topology_dump(int dim, int periodic, int n_s, int p, int64_t n_src,
                                const int32_t* q_src, int64_t n_tgt, const int32_t* q_tgt, char* buf,
                                int64_t cap);

/* the shard plan sdmk_set_shard applies, from the same host topology:
   out[0..4] = owned Morton target range [t0, t1), owned target leaves,
   boxes whose incoming expansions the rank forms, target leaves in total */
int sdmk_host_shard_plan(int dim, int periodic, int n_s, int p, int64_t n_src, const int32_t* q_src,
                         int64_t n_tgt, const int32_t* q_tgt, int rank, int nranks, int64_t* out);

/* every rank's owned range of sorted targets at once (out: nranks + 1
   bounds; rank r owns [out[r], out[r+1])): the layout of the u all-gather
   that sdmk_comm_init evaluations end with */
int sdmk_host_shard_bounds(int dim, int periodic, int n_s, int p, int64_t n_src, const int32_t* q_src,
                           int64_t n_tgt, const int32_t* q_tgt, int nranks, int64_t* out);

/* the exchange plan sdmk_comm_init evaluations use, from the same host
   topology: out[f * nranks + r] = boxes rank r receives from rank f;
   out[nranks^2 + r] = leaves with sources owned by rank r;
   out[nranks^2 + nranks] = boxes above the cut; [.. + 1] = cut boxes */
int sdmk_host_halo_plan(int dim, int periodic, int n_s, int p, int64_t n_src, const int32_t* q_src,
                        int64_t n_tgt, const int32_t* q_tgt, int nranks, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* SDMK_H */
