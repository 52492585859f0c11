// Host-callable launchers for the sm_100a kernels (one .cu per stage).
// All pointers are device pointers; every launcher enqueues on `st`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>

namespace sdmkb {
namespace dev {
// Per-box record in HBM (64 B, one line per box).  Centers/half sides are
// computed on the host with the reference's formula (tree.cpp:217-228) so the
// leaf-local coordinates (x - c) / half agree bit for bit (dmk.cpp:600-603).
struct DBox {
  int sb, se, tb, te;
  int level, parent, first_child, leaf;
  double c[3];
  double half;
  double side;
};

}  // namespace dev

// ---- tree_kernels.cu -------------------------------------------------------
// flags[0]: non-finite coordinate, flags[1]: coordinate outside [-1/2, 1/2]
// (ignored when periodic), flags[2]: non-finite strength.
void launch_validate(const double* pts, int64_t nvals, int periodic, int* flags, int flag_base,
                     cudaStream_t st);
void launch_wrap(double* pts, int64_t nvals, cudaStream_t st);
// 90/60-bit Morton keys of quantized points (tree.cpp:19-35) split in two
// 64-bit words, with the identity permutation in idx.
void launch_morton(const double* pts, int n, int dim, uint64_t* klo, uint64_t* khi, uint64_t* ktop, int* idx,
                   cudaStream_t st);
// 3D fast path: one 64-bit sort on the top 64 key bits; *tie_flag = 1 when two
// sorted keys tie there (then the full two-word sort below must be used).
void sort_morton_top(int n, uint64_t* ktop, uint64_t* ktop2, int* idx, int* perm, void* temp, size_t temp_bytes,
                     int* tie_flag, cudaStream_t st);
// Stable LSD radix sort of (key, index): exactly std::sort over (key, idx)
// pairs (tree.cpp:262-267).  perm receives the sorted original indices.
size_t sort_temp_bytes(int n);
void sort_morton(int n, int dim, uint64_t* klo, uint64_t* khi, int* idx, uint64_t* klo2,
                 uint64_t* khi2, int* idx2, int* perm, void* temp, size_t temp_bytes, cudaStream_t st);
// AoS caller-order points -> SoA sorted points + SoA quantized coordinates.
void launch_gather_points(const double* pts, const int* perm, int n, int dim, double* soa,
                          int32_t* q, cudaStream_t st);
// AoS caller-order strengths -> SoA sorted strengths (sc components).
void launch_gather_strengths(const double* str, const int* perm, int n, int sc, double* soa,
                             cudaStream_t st);
// Child boundaries of nbox Morton-sorted ranges (rng[2i], rng[2i+1]) at
// levels lvl[i]: bnd[9i + c], c = 0..2^d (tree.cpp:38-43, 109-123).
void launch_split_ranges(int nbox, const int* lvl, const int* rng, const int32_t* q, int n, int dim, int* bnd,
                         cudaStream_t st);
// refine_to_capacity on the device (tree.cpp:109-123): the boxes in the
// reference's id order, in the layout of host/tree.hpp's Box.  hdr (>= 48 ints):
// [0] boxes, [1] levels, [2] depth cap reached, [3] more than `cap` boxes
// (nothing usable was written); nodes: cap * refine_node_bytes() of scratch.
struct RefBox {
  int level, parent, first_child, leaf;
  int32_t anchor[3];
  int sb, se, tb, te;
};
size_t refine_node_bytes();
// the 2:1 repair's first sweep over launch_refine's boxes, read-only: cand[b] bit k
// set when the k-th of leaf b's 3^d neighbour-centre probes (o0 fastest, the centre
// counted) lands in a leaf two or more levels coarser
void launch_repair_scan(const RefBox* boxes, int nb, int dim, int periodic, uint32_t* cand, cudaStream_t st);
// returns false when the cooperative launch is refused (the caller refines on the host)
bool launch_refine(const int32_t* qs, int ns, const int32_t* qt, int nt, int alias, int dim, int n_s, int cap,
                   void* nodes, int* hdr, RefBox* out, cudaStream_t st);
// The residual's source sub-cells: 9 boundaries per box (children of leaves
// with sources, else [sb, se) once), as host/tree.hpp leaf_subranges.
void launch_leaf_subranges(const dev::DBox* boxes, int nb, const int32_t* q, int n, int dim, int* out,
                           cudaStream_t st);

// ---- anterp.cu (K3 leaf anterpolation, K11 target interpolation) -----------
struct ChebDev {
  int p, pz, dim;
  const double* nodes;  // p
  const double* wts;    // p
};
// outgoing[b][ch][node] for leaves `leaves[0..nleaf)` (outgoing zeroed first)
void launch_anterp(int kernel, const ChebDev& cb, const dev::DBox* boxes, const int* leaves,
                   int nleaf, const double* pts, int n, const double* str, double* outgoing,
                   int nch, cudaStream_t st);
// u_far[perm[t]*d + j] for targets of leaves `leaves`
void launch_interp_targets(const ChebDev& cb, const dev::DBox* boxes, const int* leaves, int nleaf,
                           const double* tpts, int nt, const int* tperm, const double* incoming,
                           double* ufar, cudaStream_t st);

// ---- anterp_mma.cu (DMMA versions of K3 / K11) ------------------------------
bool mma_anterp_supported(int p);
// basis[axis][i][p] for the source (use_targets = 0) or target points of `leaves`
void launch_basis(const ChebDev& cb, const dev::DBox* boxes, const int* leaves, int nleaf, const double* pts,
                  int n, int use_targets, double* basis, cudaStream_t st);
void launch_anterp_mma(int kernel, const ChebDev& cb, const dev::DBox* boxes, const int* leaves, int nleaf,
                       const double* basis, const double* str, int n, double* out, int nch, cudaStream_t st);
void launch_interp_mma(const ChebDev& cb, const dev::DBox* boxes, const int* leaves, int nleaf,
                       const double* tbasis, int nt, const int* tperm, const double* incoming, double* ufar,
                       cudaStream_t st);

// ---- tensor.cu (K4 child->parent merge, K9 parent->child interpolation) ----
// For each pair i: dst[out_box[i]] (+)= (Mz (x) My (x) Mx) src[in_box[i]] on
// `nch` channels, matrices chosen by the child index bits of ci[i]
// (dmk.cpp:82-121, 481-490).  mats: [2][p][p] (bit 0 / bit 1).
// accumulate: 1 -> dst += (one input per pair, downward interpolation);
//             2 -> merge mode: 2^d inputs per pair (-1 = skip), dst = sum.
void launch_tensor_apply(int p, int pz, int dim, const double* mats, const int* in_box,
                         const int* out_box, const int* ci, int npairs, int nch,
                         const double* src, double* dst, int accumulate, cudaStream_t st);

// ---- tensor_mma.cu: DMMA version of the above (3D, p <= 32) ----
bool tensor_mma_supported(int p, int dim);
// Downward interpolation by parent segment: pairs seg[k]..seg[k+1]-1 share one
// parent (in_list), each adds into its own child (out_box) -- one CTA per
// (segment, channel), so the per-CTA setup and the input prefetch pipeline
// are shared by the parent's children.  3D, p = 17..24.
bool tensor_seg_supported(int p, int dim);
void launch_tensor_mma_seg(int p, const double* mats, const int* in_list, const int* out_box, const int* ci,
                           const int* seg, int nseg, int nch, const double* src, double* dst, cudaStream_t st);
void launch_tensor_mma(int p, const double* mats, const int* in_list, const int* out_box, const int* ci,
                       int npairs, int nch, const double* src, double* dst, int accumulate, int dim,
                       cudaStream_t st);

// ---- planewave.cu (K5-K8/K10: forward DFT, phased accumulation + symbol,
// inverse DFT) -----------------------------------------------------------------
struct PWGrid {
  int N, M, Nz, Mz, p, pz, dim;
  int ncol, nhalf;
  const double2* E;      // [N][p]  exp(-i theta m s_i)
  const double2* Ez;     // [Nz][pz] (identity in 2D)
  const int* col_my;     // [ncol]
  const int* col_m0;
  const int* col_lz;     // in-band |mz| <= lz
  const int* slab_off;   // [Nz + 1]
  const int* slab_ncol;  // [Nz]
  const int* m0_start;   // [M + 2] CSR of columns grouped by m0
  const int* m0_cols;    // column ids
  const int* mode_code;  // [nhalf]: (mz + Mz) << 16 | column
};
// G[slot][ch][mode] from outgoing[box(slot)][ch]; B is scratch
// [nbox][nch][pz][ncol] double2.
void launch_forward(const PWGrid& g, const int* boxes, int nbox, int nch, const double* outgoing,
                    double2* B, double2* G, cudaStream_t st);
// F[t][j][mode] = symbol(sum_e phase(m, tau_e) G[slot_e]) for target boxes t
void launch_accumulate_symbol(const PWGrid& g, int kernel, int ntb, const int* ent_start,
                              const int* ent_slot, const int* ent_tau, const double2* G, int nch,
                              const double* A, double h, double2* F, cudaStream_t st);
// Same sums by sibling group: grp_tstart[ngroups + 1] indexes the level's
// target list; grp_slot[group][64] is the G slot at each parent-relative
// position (x + 4 y + 16 z over {-1..2}^d shifted by 1; 2D uses z = 0) or -1;
// t_meta[target] = child code | 8 if the target's own G must be removed.
// F rows are target index - t_base.
void launch_accumulate_group(const PWGrid& g, int kernel, int ngroups, const int* grp_tstart, const int* grp_slot,
                             const int* t_meta, int t_base, const double2* G, const double* A, double h,
                             double2* F, cudaStream_t st);
// incoming[box(t)][j] += pf * Re(inverse(F[t][j])); C is scratch
void launch_inverse(const PWGrid& g, const int* tboxes, int ntb, int d, const double2* F,
                    double2* C, double pf, double* incoming, cudaStream_t st);

// ---- planewave_mma.cu: DMMA versions of the transforms (3D, p <= 32, N <= 48) ----
bool pw_mma_supported(const PWGrid& g);
void launch_forward_mma(const PWGrid& g, const int* boxes, int nbox, int nch, const double* outgoing,
                        double2* B, double2* G, cudaStream_t st);
void launch_inverse_mma(const PWGrid& g, const int* tboxes, int ntb, int d, const double2* F,
                        double2* C, double pf, double* incoming, cudaStream_t st);

// ---- residual.cu (K12) -------------------------------------------------------
// Radial residual tables as piecewise monomials (host/setup.hpp PiecewisePoly):
// ni sub-intervals of [lo, hi], degree deg; device arrays of ni*(deg+1).
struct ResidTables {
  int ni, deg;
  double lo, hi;       // table domain (shared by both tables)
  double support;
  int kernel, dim;
  const double* pw_d;  // diag table (unused for the rotlet)
  const double* pw_o;  // offd table
  // the reference's Chebyshev tables themselves (chebyshev.hpp ChebTable),
  // evaluated by its Clenshaw recurrence, unfused, for s < s_exact: near
  // s = 0 the residual kernels multiply table values by up to 1/r^3, so
  // there the values must match the reference's to its own rounding (~1e-17)
  const double* cheb_d;  // n_d coefficients (n_d = 0 for the rotlet)
  const double* cheb_o;
  int n_d, n_o;
  double s_exact;
  // the piecewise tables are stored multiplied by these (the kernel's constant
  // factors, 1 for the 2D Stokeslet); the exact branch scales the same way
  double scale_d, scale_o;
};
constexpr int kResidMaxCheb = 80;  // longest Chebyshev table the exact branch holds in shared memory
int residual_max_pw();
// u_res[perm[t]*d+j] for all targets of leaves `leaves`; flags[0] <- coincident
// points; stats[0..1] <- candidates / in-support pairs (if stats != nullptr)
// chunks: (leaf index into `leaves`, first target) pairs, 32 targets each,
// one per warp (a leaf's targets split into ceil(n / 32) chunks).  srec is
// scratch for the packed source records (ns * (d + sc rounded up to even)
// doubles).
void launch_residual(const ResidTables& rt, const dev::DBox* boxes, const int* leaves, int nleaf,
                     const int* chunks, int nchunks, const int* rng_start, const int* rng_box, const int* rng_info, const int* subrange,
                     const double* spts, int ns, const double* sstr, double* srec, int periodic,
                     const double* tpts, int nt,
                     const int* tperm, int alias, int reserve_sms, double self_const,
                     double* ures, int* flags, unsigned long long* stats, void* scratch, cudaStream_t st);
// scratch for launch_residual (chunk counter + per-warp source interval lists)
size_t residual_scratch_bytes();

// ---- finalize.cu --------------------------------------------------------------
// sums[j] = sum_a col_j(a) for j < ncomp (deterministic block tree)
void launch_column_sums(const double* soa, int n, int ncomp, double* sums, double* scratch,
                        cudaStream_t st);
// periodic stresslet zero mode moments: out[0] = W = sum f.n, out[1..d] = sum x_a (f.n)
void launch_zero_mode_moments(const double* spts, const double* sstr, int n, int dim,
                              double* out, double* scratch, cudaStream_t st);
// u = ((ufar + ures) + corr_scale * sums[j]) (+ (mom[j] - W x_t[j])) in caller order
void launch_combine(int nt, int dim, const double* ufar, const double* ures, const double* sums, double corr_scale,
                    const double* zm, const double* tpts_caller, const unsigned char* own, double* u,
                    cudaStream_t st);
// own[tperm[s]] = (t0 <= s < t1): the caller-order mask of a shard's targets
void launch_own_mask(int nt, const int* tperm, int64_t t0, int64_t t1, unsigned char* own, cudaStream_t st);
// out[i][j] = u[tperm[t0 + i]][j], i < n: this rank's owned targets in sorted order
void launch_pack_owned(int64_t t0, int64_t n, int dim, const int* tperm, const double* u, double* out, cudaStream_t st);
// u[tperm[s]][j] = in[r * stride + (s - bounds[r]) * dim + j] for the rank r owning sorted target s
void launch_scatter_ranges(int nt, int dim, const int64_t* bounds, int nranks, int64_t stride, const int* tperm,
                           const double* in, double* u, cudaStream_t st);
// dst box (dst_ids ? dst_ids[i] : i) = src box (src_ids ? src_ids[i] : i), boxes of `elems` doubles
void launch_copy_boxes(int n, const int* src_ids, const double* src, const int* dst_ids, double* dst, int64_t elems,
                       cudaStream_t st);

// ---- ewald.cu: FFT Ewald far field (periodic 3D Stokeslet) ---------------------
struct EwGrid {
  int Mg;            // grid points per axis
  int w;             // window width in grid points (<= 16)
  int kmax;          // |kappa_i| <= kmax in the band
  long s2max;        // |kappa|^2 <= s2max
  double h, inv_h;   // grid spacing 1 / Mg
  double inv_alpha;  // 1 / (w h / 2)
  int ni, deg;       // window phi(|z|): piecewise monomials on [0, 1)
  const double* wpoly;
};
void launch_ew_spread(const EwGrid& g, int n, const double* spts, const double* sstr, double* grid, cudaStream_t st);
void launch_ew_symbol(const EwGrid& g, double2* spec, const double* A, const double* dfac, cudaStream_t st);
// gi: scratch of Mg^3 x 32 bytes (the grid interleaved per point)
void launch_ew_gather(const EwGrid& g, int n, const double* tpts, const int* tperm, const double* grid, void* gi,
                      double* u, cudaStream_t st);
// deterministic spreading (no atomics): sources binned by Morton cells at
// level Lc (bnd as launch_cell_bounds); usable when ew_spread_tiled_ok(g, Lc)
bool ew_spread_tiled_ok(const EwGrid& g, int Lc);
void launch_ew_spread_tiled(const EwGrid& g, int Lc, const int* bnd, int n, const double* spts, const double* sstr,
                            double* grid, cudaStream_t st);
// bnd[c] = first sorted point in Morton cell >= c at level L (3D), c = 0..8^L
void launch_cell_bounds(int n, const int32_t* q, int L, int* bnd, cudaStream_t st);

// ---- direct.cu: O(N*M) reference sums (oracle.cpp:143-241) ---------------------
constexpr int kDirectMaxCheb = 1024;
struct DirectTables {
  double cutoff = 1.0, support = 1.0;  // residual scale nu and the table support
  int periodic = 0;                    // 3^d image shifts (residual sum only)
  const double* cd = nullptr;          // diag / offd Chebyshev coefficients (device)
  const double* co = nullptr;
  int nd = 0, no = 0;
  double dlo = 0.0, dhi = 1.0, olo = 0.0, ohi = 1.0;
};
// u[b*dim + j] for targets b (tgt == src when alias); residual = false: the
// exact kernels (direct_sum), true: residual_apply at scale T.cutoff
// (direct_residual_sum).  flags[0] <- coincident points.  Inputs are the
// caller's point-major arrays (already wrapped when periodic).
void launch_direct(int kernel, int dim, const double* src, int ns, const double* tgt, int nt, const double* str,
                   int alias, const DirectTables& T, bool residual, double* u, int* flags, cudaStream_t st);

// ---- peak.cu ----------------------------------------------------------------
double measure_fp64_peak_tflops(cudaStream_t st);
double measure_dmma_peak_tflops(cudaStream_t st);

}  // namespace sdmkb
