// K4 (child -> parent proxy merge, dmk.cpp:624-653) and K9 (parent -> child
// potential interpolation, dmk.cpp:835-855): separable p x p x p tensor
// applies  out[i2,i1,i0] (+)= sum_j Mz[i2,j2] My[i1,j1] Mx[i0,j0] in[j2,j1,j0]
// (dmk.cpp:82-121).
//
// One CTA per (pair, channel, z-chunk).  The input is streamed one z-slab at
// a time through shared memory; the x and y stages are done in shared memory
// and every thread folds its (iy, ix) columns of the transformed slab into
// register accumulators for all output iz of its z-chunk, so the full p^3
// intermediate never leaves the SM.  For the upward merge a CTA loops over
// the parent's 2^d children and accumulates them in registers (fixed child
// order, deterministic).
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

template <int BS, int CPT, int ZC>
__global__ void __launch_bounds__(BS) k_tensor(int p, int pz, int dim, const double* __restrict__ mats,
                                                    const int* __restrict__ in_list,
                                                    const int* __restrict__ out_box,
                                                    const int* __restrict__ ci_list, int nin, int nch,
                                                    const double* __restrict__ src, double* __restrict__ dst,
                                                    int accumulate) {
  extern __shared__ double sm[];
  const int pp = p * p;
  double* MT = sm;             // [2][p][p], transposed: MT[b][j][i] = M_b[i][j]
  double* Mzs = MT + 2 * pp;   // [2][p][p] untransposed (z stage reads M[iz][jz])
  double* s_in = Mzs + 2 * pp; // p*p
  double* t1 = s_in + pp;      // p*p
  const int tid = threadIdx.x;
  for (int e = tid; e < 2 * pp; e += blockDim.x) {
    int bsel = e / pp, r = e % pp, i = r / p, j = r % p;
    MT[bsel * pp + j * p + i] = mats[e];
    Mzs[e] = mats[e];
  }
  const int pair = blockIdx.x, ch = blockIdx.y, iz0 = blockIdx.z * ZC;
  const int nodes = pz * pp;
  double acc[CPT][ZC];
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int k = 0; k < ZC; ++k) acc[c][k] = 0.0;
  __syncthreads();
  for (int q = 0; q < nin; ++q) {
    const int ib = in_list[pair * nin + q];
    if (ib < 0) continue;
    const int cbits = ci_list[pair * nin + q];
    const double* Mx = MT + (cbits & 1) * pp;
    const double* My = MT + ((cbits >> 1) & 1) * pp;
    const double* Mz = Mzs + ((cbits >> 2) & 1) * pp;
    const double* in = src + ((size_t)ib * nch + ch) * nodes;
    for (int jz = 0; jz < pz; ++jz) {
      for (int e = tid; e < pp; e += blockDim.x) s_in[e] = in[(size_t)jz * pp + e];
      __syncthreads();
      for (int e = tid; e < pp; e += blockDim.x) {  // x stage: t1[jy][ix]
        int jy = e / p, ix = e % p;
        const double* row = s_in + jy * p;
        double s = 0.0;
        for (int jx = 0; jx < p; ++jx) s = fma(Mx[jx * p + ix], row[jx], s);
        t1[e] = s;
      }
      __syncthreads();
      for (int e = tid; e < pp; e += blockDim.x) {  // y stage: s_in[iy][ix]
        int iy = e / p, ix = e % p;
        double s = 0.0;
        for (int jy = 0; jy < p; ++jy) s = fma(My[jy * p + iy], t1[jy * p + ix], s);
        s_in[e] = s;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < CPT; ++c) {  // z stage into registers
        int col = tid + c * BS;
        if (col < pp) {
          double v = s_in[col];
          if (dim == 3) {
#pragma unroll
            for (int k = 0; k < ZC; ++k) {
              int iz = iz0 + k;
              if (iz < pz) acc[c][k] = fma(Mz[iz * p + jz], v, acc[c][k]);
            }
          } else {
            acc[c][0] += v;
          }
        }
      }
      __syncthreads();
    }
  }
  double* out = dst + ((size_t)out_box[pair] * nch + ch) * nodes;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    int col = tid + c * BS;
    if (col < pp) {
#pragma unroll
      for (int k = 0; k < ZC; ++k) {
        int iz = iz0 + k;
        if (iz < pz) {
          double* o = out + (size_t)iz * pp + col;
          *o = accumulate ? *o + acc[c][k] : acc[c][k];
        }
      }
    }
  }
}

template <int BS, int CPT, int ZC>
void tensor_t(int p, int pz, int dim, const double* mats, const int* in_list, const int* out_box, const int* ci,
              int npairs, int nin, int nch, const double* src, double* dst, int accumulate, cudaStream_t st) {
  dim3 grid(npairs, nch, (pz + ZC - 1) / ZC);
  size_t smem = sizeof(double) * 6 * p * p;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tensor<BS, CPT, ZC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_tensor<BS, CPT, ZC><<<grid, BS, smem, st>>>(p, pz, dim, mats, in_list, out_box, ci, nin, nch, src, dst,
                                                 accumulate);
}

}  // namespace

// in_list/ci: [npairs][nin]; nin = 2^d for the upward merge (entries -1 are
// skipped), 1 for the downward interpolation.
void launch_tensor_apply(int p, int pz, int dim, const double* mats, const int* in_list, const int* out_box,
                         const int* ci, int npairs, int nch, const double* src, double* dst, int accumulate,
                         cudaStream_t st) {
  if (npairs <= 0) return;
  int nin = accumulate >= 2 ? (1 << dim) : 1;  // accumulate==2 -> merge mode (write, not add)
  int acc = accumulate == 1 ? 1 : 0;
  int pp = p * p;
#define TA(BS, CPT, ZC) tensor_t<BS, CPT, ZC>(p, pz, dim, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st)
  if (dim == 2) {
    if (pp <= 512) TA(512, 1, 1);
    else if (pp <= 1024) TA(512, 2, 1);
    else if (pp <= 2048) TA(512, 4, 1);
    else TA(512, 8, 1);
  } else if (pp <= 512) {
    TA(512, 1, 24);
  } else if (pp <= 576) {
    TA(576, 1, 24);
  } else if (pp <= 1024) {
    TA(512, 2, 16);
  } else if (pp <= 2048) {
    TA(512, 4, 8);
  } else {  // p = 46..64: 8 columns per thread, shorter z chunks
    TA(512, 8, 4);
  }
#undef TA
}

}  // namespace sdmkb
