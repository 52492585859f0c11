// Point validation, periodic wrap, Morton keys and the radix sort (K1).
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "launch.hpp"

#include <algorithm>

namespace sdmkb {

namespace {

constexpr int kQBits = 30;
constexpr double kCellsD = 1073741824.0;  // 2^30

// validate_system (oracle.cpp:103-131): finiteness, and the unit box in free space
__global__ void k_validate(const double* __restrict__ v, int64_t n, int periodic, int* flags, int base) {
  int bad_fin = 0, bad_box = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x = v[i];
    if (!isfinite(x)) bad_fin = 1;
    else if (!periodic && (x < -0.5 || x > 0.5)) bad_box = 1;
  }
  if (__any_sync(0xffffffffu, bad_fin) && (threadIdx.x & 31) == 0) atomicOr(flags + base, 1);
  if (__any_sync(0xffffffffu, bad_box) && (threadIdx.x & 31) == 0) atomicOr(flags + base + 1, 1);
}

// wrap_into_box: v -= floor(v + 0.5) (oracle.cpp:133-141)
__global__ void k_wrap(double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __dsub_rn(v[i], floor(__dadd_rn(v[i], 0.5)));
}

// quantize (tree.cpp:19-27): floor((x + 1/2) 2^30) clamped to [0, 2^30 - 1]
__device__ __forceinline__ int32_t quantize(double x) {
  double f = floor(__dmul_rn(__dadd_rn(x, 0.5), kCellsD));
  long long q = (long long)f;
  q = q < 0 ? 0 : (q > (1ll << kQBits) - 1 ? (1ll << kQBits) - 1 : q);
  return (int32_t)q;
}

// bit i of x to bit 3 i (x < 2^21) / bit 2 i (x < 2^32)
__host__ __device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}
__host__ __device__ __forceinline__ uint64_t spread2(uint64_t x) {
  x &= 0xffffffffull;
  x = (x | x << 16) & 0x0000ffff0000ffffull;
  x = (x | x << 8) & 0x00ff00ff00ff00ffull;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
  x = (x | x << 2) & 0x3333333333333333ull;
  x = (x | x << 1) & 0x5555555555555555ull;
  return x;
}

// Morton key with axis 0 in the least-significant interleaved bit
// (tree.cpp:29-35): bit b of axis a sits at position b dim + a.  3D: the 90
// bits are two words, lo = positions 0..63 (bits 0..20 of every axis and bit
// 21 of axis 0), hi = positions 64..89; 2D: 60 bits in lo.
__host__ __device__ __forceinline__ void morton_key(const int32_t* q, int dim, uint64_t& lo, uint64_t& hi) {
  if (dim == 3) {
    const uint64_t w = spread3((uint64_t)q[0] >> 21) | spread3((uint64_t)q[1] >> 21) << 1 |
                       spread3((uint64_t)q[2] >> 21) << 2;  // bits 21..29, position 3 (b - 21) + a
    lo = spread3((uint64_t)q[0]) | spread3((uint64_t)q[1]) << 1 | spread3((uint64_t)q[2]) << 2 | (w & 1) << 63;
    hi = w >> 1;
  } else {
    lo = spread2((uint64_t)q[0]) | spread2((uint64_t)q[1]) << 1;
    hi = 0;
  }
}

__global__ void k_morton(const double* __restrict__ pts, int n, int dim, uint64_t* klo, uint64_t* khi,
                         uint64_t* ktop, int* idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t q[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) q[a] = quantize(pts[(size_t)i * dim + a]);
  uint64_t lo, hi;
  morton_key(q, dim, lo, hi);
  klo[i] = lo;
  khi[i] = hi;
  if (ktop) ktop[i] = (hi << 38) | (lo >> 26);  // 3D: the top 64 of the 90 key bits
  idx[i] = i;
}

// flag |= 1 when two neighbours of the sorted top-64-bit keys are equal
__global__ void k_adjacent_equal(const uint64_t* __restrict__ k, int n, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 1 < n && k[i] == k[i + 1]) *flag = 1;
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const int* __restrict__ idx, int n,
                             uint64_t* dst) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_gather_points(const double* __restrict__ pts, const int* __restrict__ perm, int n, int dim,
                                double* soa, int32_t* q) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = perm[i];
  for (int a = 0; a < dim; ++a) {
    double x = pts[(size_t)s * dim + a];
    soa[(size_t)a * n + i] = x;
    q[(size_t)a * n + i] = quantize(x);
  }
}

__global__ void k_gather_strengths(const double* __restrict__ str, const int* __restrict__ perm, int n, int sc,
                                   double* soa) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = perm[i];
  for (int c = 0; c < sc; ++c) soa[(size_t)c * n + i] = str[(size_t)s * sc + c];
}

int grid_for(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 148 * 64) g = 148 * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_validate(const double* pts, int64_t nvals, int periodic, int* flags, int base, cudaStream_t st) {
  if (nvals <= 0) return;
  k_validate<<<grid_for(nvals, 256), 256, 0, st>>>(pts, nvals, periodic, flags, base);
}

void launch_wrap(double* pts, int64_t nvals, cudaStream_t st) {
  if (nvals <= 0) return;
  k_wrap<<<grid_for(nvals, 256), 256, 0, st>>>(pts, nvals);
}

void launch_morton(const double* pts, int n, int dim, uint64_t* klo, uint64_t* khi, uint64_t* ktop, int* idx,
                   cudaStream_t st) {
  k_morton<<<(n + 255) / 256, 256, 0, st>>>(pts, n, dim, klo, khi, dim == 3 ? ktop : nullptr, idx);
}

void sort_morton_top(int n, uint64_t* ktop, uint64_t* ktop2, int* idx, int* perm, void* temp, size_t temp_bytes,
                     int* tie_flag, cudaStream_t st) {
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, ktop, ktop2, idx, perm, n, 0, 64, st);
  k_adjacent_equal<<<(n + 255) / 256, 256, 0, st>>>(ktop2, n, tie_flag);
}

size_t sort_temp_bytes(int n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t*)nullptr, (uint64_t*)nullptr, (int*)nullptr,
                                  (int*)nullptr, n, 0, 64);
  cub::DeviceRadixSort::SortPairs(nullptr, b, (uint64_t*)nullptr, (uint64_t*)nullptr, (int*)nullptr,
                                  (int*)nullptr, n, 0, 26);
  return a > b ? a : b;
}

void sort_morton(int n, int dim, uint64_t* klo, uint64_t* khi, int* idx, uint64_t* klo2, uint64_t* khi2,
                 int* idx2, int* perm, void* temp, size_t temp_bytes, cudaStream_t st) {
  int lo_bits = dim == 3 ? 64 : 2 * kQBits;
  // pass 1: stable sort by the low word
  int* first_out = dim == 3 ? idx2 : perm;
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, klo, klo2, idx, first_out, n, 0, lo_bits, st);
  if (dim == 3) {
    // pass 2: stable sort by the high 26 bits; ties keep (low word, index) order
    k_gather_u64<<<(n + 255) / 256, 256, 0, st>>>(khi, idx2, n, khi2);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, khi2, khi, idx2, perm, n, 0, 3 * kQBits - 64, st);
  }
}

void launch_gather_points(const double* pts, const int* perm, int n, int dim, double* soa, int32_t* q,
                          cudaStream_t st) {
  k_gather_points<<<(n + 255) / 256, 256, 0, st>>>(pts, perm, n, dim, soa, q);
}

void launch_gather_strengths(const double* str, const int* perm, int n, int sc, double* soa, cudaStream_t st) {
  k_gather_strengths<<<(n + 255) / 256, 256, 0, st>>>(str, perm, n, sc, soa);
}

// ---- box splitting on the device (the refine of tree.cpp:109-123 and the
// residual's child sub-ranges) ----------------------------------------------
namespace {
__device__ __forceinline__ int child_index(const int32_t* __restrict__ q, int n, int m, int level, int dim) {
  int ci = 0;
  for (int a = 0; a < dim; ++a) ci |= ((q[(size_t)a * n + m] >> (29 - level)) & 1) << a;
  return ci;
}

// first m in [lo, hi) whose child index at `level` is >= c (indices are
// non-decreasing inside a box's Morton-sorted range)
__device__ __forceinline__ int lower_child(const int32_t* __restrict__ q, int n, int lo, int hi, int level, int dim,
                                           int c) {
  int a = lo, b = hi;
  while (a < b) {
    const int m = a + (b - a) / 2;
    if (child_index(q, n, m, level, dim) < c) a = m + 1;
    else b = m;
  }
  return a;
}

__global__ void k_split_ranges(int nbox, const int* __restrict__ lvl, const int* __restrict__ rng,
                               const int32_t* __restrict__ q, int n, int dim, int* __restrict__ bnd) {
  const int nchild = 1 << dim;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nbox * (nchild + 1); e += gridDim.x * blockDim.x) {
    const int b = e / (nchild + 1), c = e % (nchild + 1);
    const int lo = rng[2 * b], hi = rng[2 * b + 1];
    bnd[b * 9 + c] = c == 0 ? lo : (c == nchild ? hi : lower_child(q, n, lo, hi, lvl[b], dim, c));
  }
}

__global__ void k_leaf_subranges(const dev::DBox* __restrict__ boxes, int nb, const int32_t* __restrict__ q, int n,
                                 int dim, int* __restrict__ out) {
  const int nchild = 1 << dim;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nb * 9; e += gridDim.x * blockDim.x) {
    const int b = e / 9, c = e % 9;
    const dev::DBox x = boxes[b];
    int v;
    if (!x.leaf || x.se == x.sb || x.level >= 30) v = c == 0 ? x.sb : x.se;
    else v = c == 0 ? x.sb : (c >= nchild ? x.se : lower_child(q, n, x.sb, x.se, x.level, dim, c));
    out[e] = v;
  }
}
}  // namespace

// ---- refine_to_capacity on the device (tree.cpp:109-123) --------------------
// One cooperative launch builds the whole capacity refinement: the boxes of a
// level decide to split (more than n_s sources, depth below the cap), claim 2^d
// child slots with one atomic, and the children find their ranges by binary
// search on the Morton-sorted quantized coordinates; grid-wide barriers
// separate the levels.  The working order (breadth first, slot claims in any
// order) does not matter: the reference allocates ids when its DFS stack pops
// a box that subdivides, so a subdividing box whose pre-order rank among the
// subdividing boxes is r has children 1 + 2^d r ... -- found from the subtree
// counts (bottom up) and the ranks (top down), and the boxes are written at
// their final ids in the host's Box layout.
namespace {
namespace cg = cooperative_groups;

struct RNode {
  int level, parent, kids, cnt, rank, fid;
  int32_t anchor[3];
  int sb, se, tb, te;
};

__global__ void __launch_bounds__(256) k_refine(const int32_t* qs, int ns, const int32_t* qt, int nt, int alias,
                                                 int dim, int n_s, int cap, RNode* nodes, int* hdr, RefBox* out) {
  // hdr: [0] node count, [1] levels, [2] depth capped, [3] overflow, [8 + l] first node of level l
  cg::grid_group grid = cg::this_grid();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  const int nchild = 1 << dim;
  volatile int* vh = hdr;
  if (gtid == 0) {
    RNode r;
    r.level = 0; r.parent = -1; r.kids = -1; r.cnt = 0; r.rank = 0; r.fid = 0;
    r.anchor[0] = r.anchor[1] = r.anchor[2] = 0;
    r.sb = 0; r.se = ns; r.tb = 0; r.te = alias ? ns : nt;
    nodes[0] = r;
    hdr[0] = 1; hdr[1] = 1; hdr[2] = 0; hdr[3] = 0; hdr[8] = 0; hdr[9] = 1;
  }
  grid.sync();
  int lev = 0, lb = 0, le = 1;
  for (;;) {
    for (int i = lb + gtid; i < le; i += gsz) {  // split decisions of level lev
      RNode& nd = nodes[i];
      if (nd.se - nd.sb <= n_s) continue;
      if (nd.level >= kQBits) {
        hdr[2] = 1;
        continue;
      }
      const int k = atomicAdd(hdr, nchild);
      if (k + nchild > cap) {
        hdr[3] = 1;
        continue;
      }
      nd.kids = k;
      for (int c = 0; c < nchild; ++c) nodes[k + c].parent = i;
    }
    grid.sync();
    if (vh[3]) return;  // out of node slots: the host refines instead
    const int nle = vh[0];
    if (nle == le) break;
    for (int i = le + gtid; i < nle; i += gsz) {  // the new children
      RNode& c = nodes[i];
      const RNode& par = nodes[c.parent];
      const int ci = i - par.kids, pl = par.level;
      c.level = pl + 1;
      c.kids = -1;
      for (int a = 0; a < 3; ++a) c.anchor[a] = a < dim ? par.anchor[a] + (((ci >> a) & 1) << (kQBits - 1 - pl)) : 0;
      c.sb = ci == 0 ? par.sb : lower_child(qs, ns, par.sb, par.se, pl, dim, ci);
      c.se = ci == nchild - 1 ? par.se : lower_child(qs, ns, par.sb, par.se, pl, dim, ci + 1);
      if (alias) {
        c.tb = c.sb;
        c.te = c.se;
      } else {
        c.tb = ci == 0 ? par.tb : lower_child(qt, nt, par.tb, par.te, pl, dim, ci);
        c.te = ci == nchild - 1 ? par.te : lower_child(qt, nt, par.tb, par.te, pl, dim, ci + 1);
      }
    }
    lb = le;
    le = nle;
    ++lev;
    if (gtid == 0) {
      hdr[1] = lev + 1;
      hdr[8 + lev + 1] = nle;
    }
    grid.sync();
  }
  const int L = lev + 1;  // levels 0 .. lev
  for (int l = L - 1; l >= 0; --l) {  // subdividing boxes per subtree
    for (int i = vh[8 + l] + gtid; i < vh[8 + l + 1]; i += gsz) {
      RNode& nd = nodes[i];
      int cnt = 0;
      if (nd.kids >= 0) {
        cnt = 1;
        for (int c = 0; c < nchild; ++c) cnt += nodes[nd.kids + c].cnt;
      }
      nd.cnt = cnt;
    }
    grid.sync();
  }
  for (int l = 0; l < L; ++l) {  // pre-order ranks and final ids
    for (int i = vh[8 + l] + gtid; i < vh[8 + l + 1]; i += gsz) {
      const RNode& nd = nodes[i];
      if (nd.kids < 0) continue;
      int run = nd.rank + 1;
      for (int c = 0; c < nchild; ++c) {
        RNode& ch = nodes[nd.kids + c];
        ch.fid = 1 + nchild * nd.rank + c;
        ch.rank = run;
        run += ch.cnt;
      }
    }
    grid.sync();
  }
  for (int i = gtid; i < le; i += gsz) {
    const RNode& nd = nodes[i];
    RefBox b;
    b.level = nd.level;
    b.parent = nd.parent < 0 ? -1 : nodes[nd.parent].fid;
    b.first_child = nd.kids < 0 ? -1 : 1 + nchild * nd.rank;
    b.leaf = nd.kids < 0 ? 1 : 0;
    for (int a = 0; a < 3; ++a) b.anchor[a] = nd.anchor[a];
    b.sb = nd.sb; b.se = nd.se; b.tb = nd.tb; b.te = nd.te;
    out[nd.fid] = b;
  }
}
}  // namespace

// First sweep of the 2:1 repair (tree.cpp:125-165), read-only: does one of the
// 3^d - 1 neighbour-centre probes of leaf b land in a leaf two or more levels
// coarser?  The probe's box is found from b's parent: climb to the first
// ancestor containing it, descend to a leaf or to level(b) - 1 (the host's
// Builder::probe_triggers / locate).  One thread per box of the refined tree.
namespace {
__global__ void k_repair_scan(const RefBox* __restrict__ boxes, int nb, int dim, int periodic,
                              uint32_t* __restrict__ cand) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const RefBox bx = boxes[b];
  uint32_t hit = 0;  // bit k: the k-th offset (o0 fastest, the centre counted) triggers
  if (bx.leaf && bx.level >= 2) {
    const long long cells = 1ll << kQBits, side = cells >> bx.level;
    const int zr = dim == 3 ? 1 : 0;
    int k = 0;
    for (int o2 = -zr; o2 <= zr; ++o2)
      for (int o1 = -1; o1 <= 1; ++o1)
        for (int o0 = -1; o0 <= 1; ++o0, ++k) {
          if (!o0 && !o1 && !o2) continue;
          const int off[3] = {o0, o1, o2};
          int probe[3] = {0, 0, 0};
          bool inside = true;
          for (int a = 0; a < dim && inside; ++a) {
            long long v = bx.anchor[a] + off[a] * side + side / 2;
            if (periodic) v = ((v % cells) + cells) % cells;
            else if (v < 0 || v >= cells) inside = false;
            probe[a] = (int)v;
          }
          if (!inside) continue;
          int x = bx.parent;
          for (;;) {
            const int lv = boxes[x].level, par = boxes[x].parent;
            const long long sd = cells >> lv;
            bool in = true;
            for (int a = 0; a < dim; ++a) {
              const int an = boxes[x].anchor[a];
              in = in && probe[a] >= an && (long long)probe[a] < an + sd;
            }
            if (in || par < 0) break;
            x = par;
          }
          while (!boxes[x].leaf && boxes[x].level < bx.level - 1) {
            const int lv = boxes[x].level;
            int ci = 0;
            for (int a = 0; a < dim; ++a) ci |= ((probe[a] >> (kQBits - 1 - lv)) & 1) << a;
            x = boxes[x].first_child + ci;
          }
          if (boxes[x].leaf && boxes[x].level <= bx.level - 2) hit |= 1u << k;
        }
  }
  cand[b] = hit;
}
}  // namespace

void launch_repair_scan(const RefBox* boxes, int nb, int dim, int periodic, uint32_t* cand, cudaStream_t st) {
  if (nb <= 0) return;
  k_repair_scan<<<(nb + 127) / 128, 128, 0, st>>>(boxes, nb, dim, periodic, cand);
}

size_t refine_node_bytes() { return sizeof(RNode); }

bool launch_refine(const int32_t* qs, int ns, const int32_t* qt, int nt, int alias, int dim, int n_s, int cap,
                   void* nodes, int* hdr, RefBox* out, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_refine, 256, 0);
    grid = sms * (per < 1 ? 1 : (per > 2 ? 2 : per));
  }
  RNode* nd = (RNode*)nodes;
  void* args[] = {&qs, &ns, &qt, &nt, &alias, &dim, &n_s, &cap, &nd, &hdr, &out};
  if (cudaLaunchCooperativeKernel((const void*)k_refine, dim3(grid), dim3(256), args, 0, st) != cudaSuccess) {
    cudaGetLastError();  // no cooperative launch here (e.g. a partitioned device): the host refines
    return false;
  }
  return true;
}

void launch_split_ranges(int nbox, const int* lvl, const int* rng, const int32_t* q, int n, int dim, int* bnd,
                         cudaStream_t st) {
  if (nbox <= 0) return;
  const int tot = nbox * ((1 << dim) + 1);
  k_split_ranges<<<std::min((tot + 255) / 256, 148 * 16), 256, 0, st>>>(nbox, lvl, rng, q, n, dim, bnd);
}

void launch_leaf_subranges(const dev::DBox* boxes, int nb, const int32_t* q, int n, int dim, int* out,
                           cudaStream_t st) {
  if (nb <= 0) return;
  k_leaf_subranges<<<std::min((nb * 9 + 255) / 256, 148 * 16), 256, 0, st>>>(boxes, nb, q, n, dim, out);
}

}  // namespace sdmkb
