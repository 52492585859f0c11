// Point validation, periodic wrap, Morton keys and the radix sort (K1).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "launch.hpp"

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

// Morton key with axis 0 in the least-significant interleaved bit (tree.cpp:29-35)
__global__ void k_morton(const double* __restrict__ pts, int n, int dim, uint64_t* klo, uint64_t* khi,
                         int* idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t q[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) q[a] = quantize(pts[(size_t)i * dim + a]);
  uint64_t lo = 0, hi = 0;
  for (int bit = 0; bit < kQBits; ++bit)
    for (int a = 0; a < dim; ++a) {
      uint64_t b = (uint64_t)((q[a] >> bit) & 1);
      int pos = bit * dim + a;
      if (pos < 64) lo |= b << pos;
      else hi |= b << (pos - 64);
    }
  klo[i] = lo;
  khi[i] = hi;
  idx[i] = i;
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

void launch_morton(const double* pts, int n, int dim, uint64_t* klo, uint64_t* khi, int* idx, cudaStream_t st) {
  k_morton<<<(n + 255) / 256, 256, 0, st>>>(pts, n, dim, klo, khi, idx);
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

}  // namespace sdmkb
