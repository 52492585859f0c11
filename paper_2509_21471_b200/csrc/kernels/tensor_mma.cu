// K4 / K9 separable tensor applies on the FP64 tensor cores (3D, p <= 32):
//   out[iz,iy,ix] (+)= sum_j Mz[iz,jz] My[iy,jy] Mx[ix,jx] in[jz,jy,jx]
// (dmk.cpp:82-121, used by the upward merge dmk.cpp:624-653 and the downward
// interpolation dmk.cpp:835-855).
//
// One CTA per (pair, channel).  The input streams through shared memory four
// z-slabs at a time (cp.async, double buffered: the next group is in flight
// while the current one is multiplied); per group
//   x stage : T1[(s,jy), ix] = in[(s,jy), jx] * Mx^T      (DMMA, K = p)
//   y stage : T2[s][iy, ix]  = My * T1[s]                  (DMMA, K = p)
//   z stage : C[iz, (iy,ix)] += Mz[iz, jz0..jz0+3] * T2    (DMMA, K = 4 slabs)
// The z-stage accumulators stay in registers for the whole box (and, for the
// merge, across the 2^d children), so the p^3 intermediate never touches HBM.
// Every dimension is padded to PT*8 with zeros; fragment loads use
// bank-conflict-free strides (== 4 mod 16 for row-indexed A / B^T, == 8 mod 16
// for k-indexed B).
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

using dev::cp_async8;
using dev::cp_commit;
using dev::cp_wait0;
using dev::cp_wait1;

template <int PT, int NW, int ZT>  // PT: 8-tiles per axis; NW warps; ZT max z-stage tiles per warp
__global__ void __launch_bounds__(NW * 32, 1) k_tensor_mma(int p, const double* __restrict__ mats,
                                                           const int* __restrict__ in_list,
                                                           const int* __restrict__ out_box,
                                                           const int* __restrict__ ci_list, int nin, int nch,
                                                           const double* __restrict__ src, double* __restrict__ dst,
                                                           int accumulate) {
  constexpr int P8 = PT * 8;
  constexpr int SA = P8 + 4;
  constexpr int S1 = P8 % 8 == 4 ? P8 : P8 + 4;
  extern __shared__ double sm[];
  const int pp = p * p, nodes = p * pp;
  const int NP = (pp + 7) / 8 * 8;
  const int SS = NP % 8 == 4 ? NP : NP + 4;
  double* Mm = sm;                    // [2][P8][SA]
  double* inS = Mm + 2 * P8 * SA;     // [2 buffers][4*P8][SA]
  double* T1 = inS + 2 * 4 * P8 * SA; // [4*P8][S1]
  double* T2 = T1 + 4 * P8 * S1;      // [4][SS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int e = tid; e < 2 * P8 * SA; e += blockDim.x) {
    const int bsel = e / (P8 * SA), r = (e / SA) % P8, c = e % SA;
    Mm[e] = (r < p && c < p) ? mats[(size_t)bsel * pp + r * p + c] : 0.0;
  }
  for (int e = tid; e < 4 * SS; e += blockDim.x) T2[e] = 0.0;
  for (int e = tid; e < 2 * 4 * P8 * SA; e += blockDim.x) inS[e] = 0.0;  // padding stays zero
  const int pair = blockIdx.x, ch = blockIdx.y;
  const int ngroups = (p + 3) / 4;
  // work items: (input q, z-group)
  int qs[8];
  int nq = 0;
  for (int q = 0; q < nin; ++q)
    if (in_list[pair * nin + q] >= 0) qs[nq++] = q;
  const int nitems = nq * ngroups;
  const int ntn = NP / 8, ntiles = PT * ntn;
  double acc[ZT][2];
#pragma unroll
  for (int i = 0; i < ZT; ++i) acc[i][0] = acc[i][1] = 0.0;
  __syncthreads();
  auto issue = [&](int item, int buf) {
    const int q = qs[item / ngroups], jz0 = (item % ngroups) * 4;
    const double* in = src + ((size_t)in_list[pair * nin + q] * nch + ch) * nodes;
    double* dstb = inS + buf * 4 * P8 * SA;
    const int cnt = 4 * pp;
    for (int e = tid; e < cnt; e += blockDim.x) {
      const int s = e / pp, r = (e / p) % p, c = e % p, jz = jz0 + s;
      const bool v = jz < p;
      cp_async8(dstb + (s * P8 + r) * SA + c, v ? in + (size_t)jz * pp + r * p + c : in, v);
    }
    cp_commit();
  };
  if (nitems > 0) issue(0, 0);
  for (int item = 0; item < nitems; ++item) {
    const int buf = item & 1;
    if (item + 1 < nitems) {
      issue(item + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    const int q = qs[item / ngroups], jz0 = (item % ngroups) * 4;
    const int cb = ci_list[pair * nin + q];
    const double* Mx = Mm + (cb & 1) * P8 * SA;
    const double* My = Mm + ((cb >> 1) & 1) * P8 * SA;
    const double* Mz = Mm + ((cb >> 2) & 1) * P8 * SA;
    const double* A = inS + buf * 4 * P8 * SA;
    {  // x stage: this warp's tiles interleaved (independent DMMA chains)
      constexpr int NTL = 4 * PT * PT;
      constexpr int TPW = (NTL + NW - 1) / NW;
      double c[TPW][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks)
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int tile = warp + NW * i;
          if (tile < NTL) {
            const int mt = tile / PT, nt = tile % PT;
            dev::dmma(c[i][0], c[i][1], A[(mt * 8 + g) * SA + ks * 4 + t], Mx[(nt * 8 + g) * SA + ks * 4 + t]);
          }
        }
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int tile = warp + NW * i;
        if (tile < NTL) {
          const int mt = tile / PT, nt = tile % PT;
          const int r = mt * 8 + g, cidx = nt * 8 + 2 * t;
          T1[r * S1 + cidx] = c[i][0];
          T1[r * S1 + cidx + 1] = c[i][1];
        }
      }
    }
    __syncthreads();
    {  // y stage, interleaved likewise
      constexpr int NTL = 4 * PT * PT;
      constexpr int TPW = (NTL + NW - 1) / NW;
      double c[TPW][2];
#pragma unroll
      for (int i = 0; i < TPW; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks)
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int tile = warp + NW * i;
          if (tile < NTL) {
            const int s = tile / (PT * PT), mt = (tile / PT) % PT, nt = tile % PT;
            dev::dmma(c[i][0], c[i][1], My[(mt * 8 + g) * SA + ks * 4 + t],
                      T1[(s * P8 + ks * 4 + t) * S1 + nt * 8 + g]);
          }
        }
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int tile = warp + NW * i;
        if (tile < NTL) {
          const int s = tile / (PT * PT), mt = (tile / PT) % PT, nt = tile % PT;
          const int iy = mt * 8 + g, ix = nt * 8 + 2 * t;
          if (iy < p) {
            if (ix < p) T2[s * SS + iy * p + ix] = c[i][0];
            if (ix + 1 < p) T2[s * SS + iy * p + ix + 1] = c[i][1];
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ZT; ++i) {  // z stage
      const int id = warp + NW * i;
      if (id < ntiles) {
        const int zt = id / ntn, nt = id % ntn;
        dev::dmma(acc[i][0], acc[i][1], Mz[(zt * 8 + g) * SA + jz0 + t], T2[t * SS + nt * 8 + g]);
      }
    }
    __syncthreads();
  }
  double* out = dst + ((size_t)out_box[pair] * nch + ch) * nodes;
#pragma unroll
  for (int i = 0; i < ZT; ++i) {
    const int id = warp + NW * i;
    if (id >= ntiles) continue;
    const int zt = id / ntn, nt = id % ntn;
    const int iz = zt * 8 + g, n = nt * 8 + 2 * t;
    if (iz >= p) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (n + e < pp) {
        double* o = out + (size_t)iz * pp + n + e;
        *o = accumulate ? *o + acc[i][e] : acc[i][e];
      }
    }
  }
}

template <int PT, int NW, int ZT>
void tensor_mma_t(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs,
                  int nin, int nch, const double* src, double* dst, int accumulate, cudaStream_t st) {
  constexpr int P8 = PT * 8, SA = P8 + 4, S1 = P8 % 8 == 4 ? P8 : P8 + 4;
  const int NP = (p * p + 7) / 8 * 8, SS = NP % 8 == 4 ? NP : NP + 4;
  size_t smem = sizeof(double) * (2 * P8 * SA + 2 * 4 * P8 * SA + 4 * P8 * S1 + 4 * SS);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tensor_mma<PT, NW, ZT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(npairs, nch);
  k_tensor_mma<PT, NW, ZT><<<grid, NW * 32, smem, st>>>(p, mats, in_list, out_box, ci, nin, nch, src, dst,
                                                         accumulate);
}

}  // namespace

bool tensor_mma_supported(int p, int dim) { return dim == 3 && p >= 4 && p <= 32; }

void launch_tensor_mma(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs,
                       int nch, const double* src, double* dst, int accumulate, int dim, cudaStream_t st) {
  if (npairs <= 0) return;
  const int nin = accumulate >= 2 ? (1 << dim) : 1;
  const int acc = accumulate == 1 ? 1 : 0;
  const int PT = (p + 7) / 8;
  if (PT <= 1) tensor_mma_t<1, 4, 8>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (PT == 2) tensor_mma_t<2, 8, 12>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (PT == 3) tensor_mma_t<3, 16, 13>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else tensor_mma_t<4, 16, 32>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
}

}  // namespace sdmkb
