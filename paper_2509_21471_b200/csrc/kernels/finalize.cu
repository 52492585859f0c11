// K13: global scalars and the final combine (dmk.cpp:1086-1102,
// oracle.cpp:250-274).  Sums use compensated per-thread accumulation and a
// fixed-shape reduction tree, so results are deterministic run to run.
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

constexpr int kSumBlocks = 256;
constexpr int kSumThreads = 256;
constexpr int kMaxComp = 4;

struct KSum {
  double s = 0.0, c = 0.0;
  __device__ void add(double v) {  // Neumaier
    double t = s + v;
    if (fabs(s) >= fabs(v)) c += (s - t) + v;
    else c += (v - t) + s;
    s = t;
  }
  __device__ double value() const { return s + c; }
};

// mode 0: columns of soa (ncomp <= 4); mode 1: zero-mode moments (W, sum x (f.n))
__global__ void __launch_bounds__(kSumThreads) k_partial(int mode, const double* __restrict__ a,
                                                         const double* __restrict__ b, int n, int ncomp,
                                                         int dim, double* part) {
  __shared__ double sh[kMaxComp][kSumThreads];
  KSum acc[kMaxComp];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (mode == 0) {
      for (int j = 0; j < ncomp; ++j) acc[j].add(a[(size_t)j * n + i]);
    } else {
      double fn = 0.0;
      for (int k = 0; k < dim; ++k) fn += b[(size_t)k * n + i] * b[(size_t)(dim + k) * n + i];
      acc[0].add(fn);
      for (int k = 0; k < dim; ++k) acc[1 + k].add(a[(size_t)k * n + i] * fn);
    }
  }
  for (int j = 0; j < ncomp; ++j) sh[j][threadIdx.x] = acc[j].value();
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int j = 0; j < ncomp; ++j) sh[j][threadIdx.x] += sh[j][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int j = 0; j < ncomp; ++j) part[(size_t)j * gridDim.x + blockIdx.x] = sh[j][0];
}

__global__ void k_final(const double* part, int nblk, int ncomp, double* out) {
  if (threadIdx.x != 0) return;
  for (int j = 0; j < ncomp; ++j) {
    KSum s;
    for (int b = 0; b < nblk; ++b) s.add(part[(size_t)j * nblk + b]);
    out[j] = s.value();
  }
}

__global__ void k_combine(int nt, int dim, const double* __restrict__ ufar, const double* __restrict__ ures,
                          const double* __restrict__ corr, double cs, const double* __restrict__ zm,
                          const double* __restrict__ tp, const unsigned char* __restrict__ own,
                          double* __restrict__ u) {
  int64_t n = (int64_t)nt * dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(i % dim);
    double v = ufar[i] + ures[i];
    if (corr) v += cs * corr[j];
    if (zm) v += zm[1 + j] - zm[0] * tp[i];
    if (own && !own[i / dim]) v = 0.0;  // another rank's target
    u[i] = v;
  }
}

__global__ void k_own_mask(int nt, const int* __restrict__ tperm, int64_t t0, int64_t t1,
                           unsigned char* __restrict__ own) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nt; s += (int64_t)gridDim.x * blockDim.x)
    own[tperm[s]] = (s >= t0 && s < t1) ? 1 : 0;
}

// All-gather of the owned target ranges (multi-GPU): pack this rank's rows
// in sorted order, then every rank scatters all ranks' rows to caller order.
__global__ void k_pack_owned(int64_t t0, int64_t n, int dim, const int* __restrict__ tperm,
                             const double* __restrict__ u, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * dim; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t0 + i / dim;
    out[i] = u[(int64_t)tperm[s] * dim + i % dim];
  }
}

__global__ void k_scatter_ranges(int nt, int dim, const int64_t* __restrict__ bounds, int nranks, int64_t stride,
                                 const int* __restrict__ tperm, const double* __restrict__ in,
                                 double* __restrict__ u) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nt * dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / dim;
    int lo = 0, hi = nranks - 1;  // the rank r with bounds[r] <= s < bounds[r + 1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (bounds[mid] <= s) lo = mid;
      else hi = mid - 1;
    }
    u[(int64_t)tperm[s] * dim + i % dim] = in[lo * stride + (s - bounds[lo]) * dim + i % dim];
  }
}

// Halo pack / unpack of whole boxes: dst box i = src box i, where a null
// id list means the boxes are contiguous from 0.  One CTA per box, a
// grid-stride over its elements (coalesced; the halo is a few % of the proxies).
__global__ void k_copy_boxes(int n, const int* __restrict__ src_ids, const double* __restrict__ src,
                             const int* __restrict__ dst_ids, double* __restrict__ dst, int64_t elems) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const double* s = src + (src_ids ? (int64_t)src_ids[i] : (int64_t)i) * elems;
    double* d = dst + (dst_ids ? (int64_t)dst_ids[i] : (int64_t)i) * elems;
    for (int64_t k = threadIdx.x; k < elems; k += blockDim.x) d[k] = s[k];
  }
}

}  // namespace

void launch_copy_boxes(int n, const int* src_ids, const double* src, const int* dst_ids, double* dst, int64_t elems,
                       cudaStream_t st) {
  if (n <= 0) return;
  k_copy_boxes<<<n < 148 * 8 ? n : 148 * 8, 512, 0, st>>>(n, src_ids, src, dst_ids, dst, elems);
}

void launch_column_sums(const double* soa, int n, int ncomp, double* sums, double* scratch, cudaStream_t st) {
  k_partial<<<kSumBlocks, kSumThreads, 0, st>>>(0, soa, nullptr, n, ncomp, 0, scratch);
  k_final<<<1, 32, 0, st>>>(scratch, kSumBlocks, ncomp, sums);
}

void launch_zero_mode_moments(const double* spts, const double* sstr, int n, int dim, double* out, double* scratch,
                              cudaStream_t st) {
  k_partial<<<kSumBlocks, kSumThreads, 0, st>>>(1, spts, sstr, n, 1 + dim, dim, scratch);
  k_final<<<1, 32, 0, st>>>(scratch, kSumBlocks, 1 + dim, out);
}

void launch_combine(int nt, int dim, const double* ufar, const double* ures, const double* corr, double cs,
                    const double* zm, const double* tpts_caller, const unsigned char* own, double* u,
                    cudaStream_t st) {
  int64_t n = (int64_t)nt * dim;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_combine<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(nt, dim, ufar, ures, corr, cs, zm, tpts_caller, own, u);
}

void launch_pack_owned(int64_t t0, int64_t n, int dim, const int* tperm, const double* u, double* out, cudaStream_t st) {
  if (n <= 0) return;
  int64_t g = (n * dim + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_pack_owned<<<(int)g, 256, 0, st>>>(t0, n, dim, tperm, u, out);
}

void launch_scatter_ranges(int nt, int dim, const int64_t* bounds, int nranks, int64_t stride, const int* tperm,
                           const double* in, double* u, cudaStream_t st) {
  int64_t g = ((int64_t)nt * dim + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_scatter_ranges<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(nt, dim, bounds, nranks, stride, tperm, in, u);
}

void launch_own_mask(int nt, const int* tperm, int64_t t0, int64_t t1, unsigned char* own, cudaStream_t st) {
  int64_t g = ((int64_t)nt + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  k_own_mask<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(nt, tperm, t0, t1, own);
}

}  // namespace sdmkb
