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
// bank-conflict-free strides (== 4 mod 8 doubles).
//
// PC > 0 compiles the kernel for a fixed p (the BASELINE orders 22, 23, 30):
// all index arithmetic then folds to constants -- with a runtime p the
// integer division sequences outnumbered the DMMAs ~8:1 (ncu source page).
#include "common.cuh"
#include "launch.hpp"

#include <cstdlib>

namespace sdmkb {

namespace {

using dev::cp_async8;
using dev::cp_commit;
using dev::cp_wait0;
using dev::cp_wait1;

template <int PC, int PT, int NW, int ZT>
__global__ void __launch_bounds__(NW * 32, 1) k_tensor_mma(int p_rt, const double* __restrict__ mats,
                                                           const int* __restrict__ in_list,
                                                           const int* __restrict__ out_box,
                                                           const int* __restrict__ ci_list, int nin, int nch,
                                                           const double* __restrict__ src, double* __restrict__ dst,
                                                           int accumulate) {
  constexpr int P8 = PT * 8;
  constexpr int SA = P8 + 4;
  constexpr int S1 = P8 % 8 == 4 ? P8 : P8 + 4;
  const int p = PC > 0 ? PC : p_rt;
  extern __shared__ double sm[];
  const int pp = p * p, nodes = p * pp;
  const int NP = (pp + 7) / 8 * 8;
  const int SS = NP % 8 == 4 ? NP : NP + 4;
  __shared__ int s_in[8], s_ci[8], s_nq;
  double* Mm = sm;                    // [2][P8][SA]
  double* inS = Mm + 2 * P8 * SA;     // [2 buffers][4*P8][SA]
  double* T1 = inS + 2 * 4 * P8 * SA; // [4*P8][S1]
  double* T2 = T1 + 4 * P8 * S1;      // [4][SS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int r = warp; r < 2 * P8; r += NW) {  // zero-padded bit-0 / bit-1 matrices
    const int bsel = r / P8, rr = r % P8;
    for (int c = lane; c < SA; c += 32) Mm[r * SA + c] = (rr < p && c < p) ? mats[(size_t)bsel * pp + rr * p + c] : 0.0;
  }
  for (int e = tid; e < 4 * SS; e += blockDim.x) T2[e] = 0.0;
  for (int e = tid; e < 2 * 4 * P8 * SA; e += blockDim.x) inS[e] = 0.0;  // padding stays zero
  const int pair = blockIdx.x, ch = blockIdx.y;
  if (tid == 0) {
    int nq = 0;
    for (int q = 0; q < nin; ++q) {
      const int ib = in_list[pair * nin + q];
      if (ib >= 0) {
        s_in[nq] = ib;
        s_ci[nq] = ci_list[pair * nin + q];
        ++nq;
      }
    }
    s_nq = nq;
  }
  __syncthreads();
  const int ngroups = (p + 3) / 4;
  const int nitems = s_nq * ngroups;
  const int ntn = NP / 8, ntiles = PT * ntn;
  double acc[ZT][2];
#pragma unroll
  for (int i = 0; i < ZT; ++i) acc[i][0] = acc[i][1] = 0.0;
  auto issue = [&](int item, int buf) {
    const int q = item / ngroups, jz0 = (item % ngroups) * 4;
    const double* in = src + ((size_t)s_in[q] * nch + ch) * nodes;
    double* dstb = inS + buf * 4 * P8 * SA;
    for (int row = warp; row < 4 * p; row += NW) {  // rows (s, r) of the group, lanes along c
      const int s = row / p, r = row % p, jz = jz0 + s;
      const bool v = jz < p;
      const double* srow = in + (size_t)(v ? jz : 0) * pp + r * p;
      for (int c = lane; c < p; c += 32) cp_async8(dstb + (s * P8 + r) * SA + c, srow + c, v);
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
    const int q = item / ngroups, jz0 = (item % ngroups) * 4;
    const int cb = s_ci[q];
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

// PT = 3 (p = 17..24) variant: 12 warps, 8 z-slabs per group, every stage
// register-blocked so each shared fragment feeds several DMMAs:
//   x: warp owns 2 of the 24 row tiles (s, jy) x all 3 ix tiles; its A
//      fragments come straight from global memory (L2), prefetched into
//      registers one group ahead, so the input never round-trips through
//      shared memory;
//   y: warp owns 2 of the 24 (slab, iy-tile) units x all 3 ix tiles;
//   z: warp owns n-tiles w, w + 12, ... of the (iy, ix) plane x all 3 iz tiles,
//      accumulated in registers over every group of every input box.
// 2 barriers per group; the per-warp tile counts divide evenly (72 x/y
// tiles, 67 z column tiles over 12 warps).
constexpr int kT3W = 12;
constexpr int kT3SG = 8;
template <int PC>
__global__ void __launch_bounds__(kT3W * 32, 1)
    k_tensor3(int p_rt, const double* __restrict__ mats, const int* __restrict__ in_list,
              const int* __restrict__ out_box, const int* __restrict__ ci_list, int nin, int nch,
              const double* __restrict__ src, double* __restrict__ dst, int accumulate,
              const int* __restrict__ seg) {
  constexpr int PT = 3, P8 = 24, SA = 28, S1 = 28, SG = kT3SG, NWp = kT3W;
  const int p = PC > 0 ? PC : p_rt;
  const int pp = p * p, nodes = p * pp;
  const int NN = (pp + 7) / 8;               // z-stage column tiles
  const int SS = NN * 8 + 4;                 // T2 row stride (== 4 mod 8)
  constexpr int ZN = (9 * 8 + NWp - 1) / NWp; // max column tiles per warp (p <= 24: NN <= 72)
  extern __shared__ double sm[];
  __shared__ int s_in[8], s_ci[8], s_out[8], s_nq;
  double* Mm = sm;                       // [2][P8][SA]
  double* T1 = Mm + 2 * P8 * SA;         // [SG * P8][S1]
  double* T2 = T1 + SG * P8 * S1;        // [SG][SS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int r = warp; r < 2 * P8; r += NWp) {
    const int bsel = r / P8, rr = r % P8;
    for (int c = lane; c < SA; c += 32) Mm[r * SA + c] = (rr < p && c < p) ? mats[(size_t)bsel * pp + rr * p + c] : 0.0;
  }
  for (int e = tid; e < SG * SS; e += blockDim.x) T2[e] = 0.0;
  const int pair = blockIdx.x, ch = blockIdx.y;
  if (tid == 0) {
    int nq = 0;
    if (seg) {  // downward: one parent, its children (one output each) in this segment
      for (int q = seg[pair]; q < seg[pair + 1]; ++q) {
        s_in[nq] = in_list[q];
        s_ci[nq] = ci_list[q];
        s_out[nq] = out_box[q];
        ++nq;
      }
    } else {
      for (int q = 0; q < nin; ++q) {
        const int ib = in_list[pair * nin + q];
        if (ib >= 0) {
          s_in[nq] = ib;
          s_ci[nq] = ci_list[pair * nin + q];
          ++nq;
        }
      }
    }
    s_nq = nq;
  }
  __syncthreads();
  const int ngroups = (p + SG - 1) / SG;
  const int nitems = s_nq * ngroups;
  double acc[ZN][PT][2];
#pragma unroll
  for (int i = 0; i < ZN; ++i)
#pragma unroll
    for (int m = 0; m < PT; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
  // this lane's x-stage A fragments: rows (s, jy) of tiles warp, warp + 12; columns 4 ks + t
  int roff[2];
  bool rok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int row = (warp + NWp * h) * 8 + g, sl = row / P8, jy = row % P8;
    roff[h] = sl * pp + jy * p;
    rok[h] = jy < p;
  }
  double af[2][2 * PT];
  auto load_a = [&](int item) {
    const int q = item / ngroups, jz0 = (item % ngroups) * SG;
    const double* in = src + ((size_t)s_in[q] * nch + ch) * nodes + (size_t)jz0 * pp;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sl = ((warp + NWp * h) * 8 + g) / P8;
      const bool ok = rok[h] && jz0 + sl < p;
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks) {
        const int jx = ks * 4 + t;
        af[h][ks] = (ok && jx < p) ? __ldg(in + roff[h] + jx) : 0.0;
      }
    }
  };
  if (nitems > 0) load_a(0);
  for (int item = 0; item < nitems; ++item) {
    const int q = item / ngroups, jz0 = (item % ngroups) * SG;
    const int cb = s_ci[q];
    const double* Mx = Mm + (cb & 1) * P8 * SA;
    const double* My = Mm + ((cb >> 1) & 1) * P8 * SA;
    const double* Mz = Mm + ((cb >> 2) & 1) * P8 * SA;
    double ax[2][2 * PT];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks) ax[h][ks] = af[h][ks];
    if (item + 1 < nitems) load_a(item + 1);  // in flight during this group
    {  // x stage: T1[(s,jy), ix] = sum_jx in[(s,jy), jx] Mx[ix, jx]
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int mt = warp + NWp * h;  // of SG * PT = 24 row tiles
        double c[PT][2];
#pragma unroll
        for (int n = 0; n < PT; ++n) c[n][0] = c[n][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2 * PT; ++ks)
#pragma unroll
          for (int n = 0; n < PT; ++n) dev::dmma(c[n][0], c[n][1], ax[h][ks], Mx[(n * 8 + g) * SA + ks * 4 + t]);
#pragma unroll
        for (int n = 0; n < PT; ++n) {
          double* o = T1 + (mt * 8 + g) * S1 + n * 8 + 2 * t;
          o[0] = c[n][0];
          o[1] = c[n][1];
        }
      }
    }
    __syncthreads();
    {  // y stage: T2[s][iy, ix] = sum_jy My[iy, jy] T1[(s,jy), ix]
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = warp + NWp * h, sl = u / PT, mt = u % PT;  // of SG * PT = 24 units
        double c[PT][2];
#pragma unroll
        for (int n = 0; n < PT; ++n) c[n][0] = c[n][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2 * PT; ++ks) {
          const double av = My[(mt * 8 + g) * SA + ks * 4 + t];
#pragma unroll
          for (int n = 0; n < PT; ++n)
            dev::dmma(c[n][0], c[n][1], av, T1[(sl * P8 + ks * 4 + t) * S1 + n * 8 + g]);
        }
        const int iy = mt * 8 + g;
        if (iy < p) {
#pragma unroll
          for (int n = 0; n < PT; ++n) {
            const int ix = n * 8 + 2 * t;
            if (ix < p) T2[sl * SS + iy * p + ix] = c[n][0];
            if (ix + 1 < p) T2[sl * SS + iy * p + ix + 1] = c[n][1];
          }
        }
      }
    }
    __syncthreads();
    // z stage: C[iz, n] += sum_{jz in group} Mz[iz, jz] T2[jz][n]
#pragma unroll
    for (int ks = 0; ks < SG / 4; ++ks) {
      double av[PT];
#pragma unroll
      for (int m = 0; m < PT; ++m) av[m] = Mz[(m * 8 + g) * SA + jz0 + ks * 4 + t];
#pragma unroll
      for (int i = 0; i < ZN; ++i) {
        const int nt = warp + NWp * i;
        if (nt < NN) {
          const double bv = T2[(ks * 4 + t) * SS + nt * 8 + g];
#pragma unroll
          for (int m = 0; m < PT; ++m) dev::dmma(acc[i][m][0], acc[i][m][1], av[m], bv);
        }
      }
    }
    // the next group's x stage rewrites T1 only (read by this y stage, fenced
    // by the barrier above); its y stage rewrites T2 after the next barrier
    const bool last = seg ? (item % ngroups == ngroups - 1) : (item == nitems - 1);
    if (last) {
      double* out = dst + ((size_t)(seg ? s_out[q] : out_box[pair]) * nch + ch) * nodes;
#pragma unroll
      for (int i = 0; i < ZN; ++i) {
        const int nt = warp + NWp * i;
        if (nt >= NN) continue;
#pragma unroll
        for (int m = 0; m < PT; ++m) {
          const int iz = m * 8 + g, n = nt * 8 + 2 * t;
          if (iz >= p) continue;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (n + e < pp) {
              double* o = out + (size_t)iz * pp + n + e;
              *o = accumulate ? *o + acc[i][m][e] : acc[i][m][e];
            }
            acc[i][m][e] = 0.0;  // the next child (downward) starts from zero
          }
        }
      }
    }
  }

}

// PT = 4 (p = 25..32): the same schedule with the output's ix columns split
// over two CTAs (blockIdx.z).  The x stage only needs the CTA's ix half of
// Mx, the y stage contracts jy and keeps ix, the z stage contracts jz and
// keeps (iy, ix) -- so the split duplicates no work and halves the z
// accumulators (which would not fit in registers for p^3 = 27 000 outputs).
constexpr int kT4W = 12;
template <int PC>
__global__ void __launch_bounds__(kT4W * 32, 1)
    k_tensor4(int p_rt, const double* __restrict__ mats, const int* __restrict__ in_list,
              const int* __restrict__ out_box, const int* __restrict__ ci_list, int nin, int nch,
              const double* __restrict__ src, double* __restrict__ dst, int accumulate) {
  constexpr int PT = 4, P8 = 32, SA = 36, NXH = 2, XW = 16, S1 = 20, SG = 8, NWp = kT4W;
  const int p = PC > 0 ? PC : p_rt;
  const int pp = p * p, nodes = p * pp;
  const int ix0 = blockIdx.z * XW;
  const int NC = p * XW;                      // z-stage columns (iy, ix local)
  const int NN = NC / 8;
  const int SS = NC + 4;                      // T2 row stride (== 4 mod 8)
  constexpr int ZN = (32 * XW / 8 + NWp - 1) / NWp;  // max column tiles per warp
  constexpr int XR = (SG * PT + NWp - 1) / NWp;      // x-stage row tiles per warp
  extern __shared__ double sm[];
  __shared__ int s_in[8], s_ci[8], s_nq;
  double* Mm = sm;                       // [2][P8][SA]
  double* T1 = Mm + 2 * P8 * SA;         // [SG * P8][S1]
  double* T2 = T1 + SG * P8 * S1;        // [SG][SS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int r = warp; r < 2 * P8; r += NWp) {
    const int bsel = r / P8, rr = r % P8;
    for (int c = lane; c < SA; c += 32) Mm[r * SA + c] = (rr < p && c < p) ? mats[(size_t)bsel * pp + rr * p + c] : 0.0;
  }
  for (int e = tid; e < SG * SS; e += blockDim.x) T2[e] = 0.0;
  const int pair = blockIdx.x, ch = blockIdx.y;
  if (tid == 0) {
    int nq = 0;
    for (int q = 0; q < nin; ++q) {
      const int ib = in_list[pair * nin + q];
      if (ib >= 0) {
        s_in[nq] = ib;
        s_ci[nq] = ci_list[pair * nin + q];
        ++nq;
      }
    }
    s_nq = nq;
  }
  __syncthreads();
  const int ngroups = (p + SG - 1) / SG;
  const int nitems = s_nq * ngroups;
  double acc[ZN][PT][2];
#pragma unroll
  for (int i = 0; i < ZN; ++i)
#pragma unroll
    for (int m = 0; m < PT; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
  int roff[XR];
  bool rok[XR];
#pragma unroll
  for (int h = 0; h < XR; ++h) {
    const int mt = warp + NWp * h;
    const int row = mt * 8 + g, sl = row / P8, jy = row % P8;
    roff[h] = sl * pp + jy * p;
    rok[h] = mt < SG * PT && jy < p;
  }
  double af[XR][2 * PT];
  auto load_a = [&](int item) {
    const int q = item / ngroups, jz0 = (item % ngroups) * SG;
    const double* in = src + ((size_t)s_in[q] * nch + ch) * nodes + (size_t)jz0 * pp;
#pragma unroll
    for (int h = 0; h < XR; ++h) {
      const int sl = ((warp + NWp * h) * 8 + g) / P8;
      const bool ok = rok[h] && jz0 + sl < p;
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks) {
        const int jx = ks * 4 + t;
        af[h][ks] = (ok && jx < p) ? __ldg(in + roff[h] + jx) : 0.0;
      }
    }
  };
  if (nitems > 0) load_a(0);
  for (int item = 0; item < nitems; ++item) {
    const int q = item / ngroups, jz0 = (item % ngroups) * SG;
    const int cb = s_ci[q];
    const double* Mx = Mm + (cb & 1) * P8 * SA;
    const double* My = Mm + ((cb >> 1) & 1) * P8 * SA;
    const double* Mz = Mm + ((cb >> 2) & 1) * P8 * SA;
    // x stage: T1[(s,jy), ixl] = sum_jx in[(s,jy), jx] Mx[ix0 + ixl, jx]
#pragma unroll
    for (int h = 0; h < XR; ++h) {
      const int mt = warp + NWp * h;
      if (mt >= SG * PT) continue;
      double c[NXH][2];
#pragma unroll
      for (int n = 0; n < NXH; ++n) c[n][0] = c[n][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks)
#pragma unroll
        for (int n = 0; n < NXH; ++n)
          dev::dmma(c[n][0], c[n][1], af[h][ks], Mx[(ix0 + n * 8 + g) * SA + ks * 4 + t]);
#pragma unroll
      for (int n = 0; n < NXH; ++n) {
        double* o = T1 + (mt * 8 + g) * S1 + n * 8 + 2 * t;
        o[0] = c[n][0];
        o[1] = c[n][1];
      }
    }
    if (item + 1 < nitems) load_a(item + 1);  // in flight during the y and z stages
    __syncthreads();
    // y stage: T2[s][iy, ixl] = sum_jy My[iy, jy] T1[(s,jy), ixl]
    for (int u = warp; u < SG * PT; u += NWp) {
      const int sl = u / PT, mt = u % PT;
      double c[NXH][2];
#pragma unroll
      for (int n = 0; n < NXH; ++n) c[n][0] = c[n][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks) {
        const double av = My[(mt * 8 + g) * SA + ks * 4 + t];
#pragma unroll
        for (int n = 0; n < NXH; ++n)
          dev::dmma(c[n][0], c[n][1], av, T1[(sl * P8 + ks * 4 + t) * S1 + n * 8 + g]);
      }
      const int iy = mt * 8 + g;
      if (iy < p) {
#pragma unroll
        for (int n = 0; n < NXH; ++n) {
          T2[sl * SS + iy * XW + n * 8 + 2 * t] = c[n][0];
          T2[sl * SS + iy * XW + n * 8 + 2 * t + 1] = c[n][1];
        }
      }
    }
    __syncthreads();
    // z stage: C[iz, (iy, ixl)] += sum_{jz in group} Mz[iz, jz] T2[jz][(iy, ixl)]
#pragma unroll
    for (int ks = 0; ks < SG / 4; ++ks) {
      double av[PT];
#pragma unroll
      for (int m = 0; m < PT; ++m) av[m] = Mz[(m * 8 + g) * SA + jz0 + ks * 4 + t];
#pragma unroll
      for (int i = 0; i < ZN; ++i) {
        const int nt = warp + NWp * i;
        if (nt < NN) {
          const double bv = T2[(ks * 4 + t) * SS + nt * 8 + g];
#pragma unroll
          for (int m = 0; m < PT; ++m) dev::dmma(acc[i][m][0], acc[i][m][1], av[m], bv);
        }
      }
    }
  }
  double* out = dst + ((size_t)out_box[pair] * nch + ch) * nodes;
#pragma unroll
  for (int i = 0; i < ZN; ++i) {
    const int nt = warp + NWp * i;
    if (nt >= NN) continue;
#pragma unroll
    for (int m = 0; m < PT; ++m) {
      const int iz = m * 8 + g;
      if (iz >= p) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nt * 8 + 2 * t + e, iy = col / XW, ix = ix0 + col % XW;
        if (ix < p) {
          double* o = out + (size_t)iz * pp + iy * p + ix;
          *o = accumulate ? *o + acc[i][m][e] : acc[i][m][e];
        }
      }
    }
  }
}

template <int PC>
void tensor4_t(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs, int nin,
               int nch, const double* src, double* dst, int accumulate, cudaStream_t st) {
  const size_t smem = sizeof(double) * (2 * 32 * 36 + 8 * 32 * 20 + 8 * ((size_t)p * 16 + 4));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tensor4<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(npairs, nch, 2);
  k_tensor4<PC><<<grid, kT4W * 32, smem, st>>>(p, mats, in_list, out_box, ci, nin, nch, src, dst, accumulate);
}

template <int PC>
void tensor3_t(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs, int nin,
               int nch, const double* src, double* dst, int accumulate, cudaStream_t st) {
  const int NN = (p * p + 7) / 8;
  const size_t smem = sizeof(double) * (2 * 24 * 28 + kT3SG * 24 * 28 + kT3SG * (NN * 8 + 4));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tensor3<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(npairs, nch);
  k_tensor3<PC><<<grid, kT3W * 32, smem, st>>>(p, mats, in_list, out_box, ci, nin, nch, src, dst, accumulate,
                                                nullptr);
}

template <int PC, int PT, int NW, int ZT>
void tensor_mma_t(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs,
                  int nin, int nch, const double* src, double* dst, int accumulate, cudaStream_t st) {
  constexpr int P8 = PT * 8, SA = P8 + 4, S1 = P8 % 8 == 4 ? P8 : P8 + 4;
  const int NP = (p * p + 7) / 8 * 8, SS = NP % 8 == 4 ? NP : NP + 4;
  size_t smem = sizeof(double) * (2 * P8 * SA + 2 * 4 * P8 * SA + 4 * P8 * S1 + 4 * SS);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tensor_mma<PC, PT, NW, ZT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(npairs, nch);
  k_tensor_mma<PC, PT, NW, ZT><<<grid, NW * 32, smem, st>>>(p, mats, in_list, out_box, ci, nin, nch, src, dst,
                                                             accumulate);
}

template <int PC>
void tensor3_seg_t(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, const int* seg,
                   int nseg, int nch, const double* src, double* dst, cudaStream_t st) {
  const int NN = (p * p + 7) / 8;
  const size_t smem = sizeof(double) * (2 * 24 * 28 + kT3SG * 24 * 28 + kT3SG * (NN * 8 + 4));
  cudaFuncSetAttribute(k_tensor3<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  dim3 grid(nseg, nch);
  // write, not add: a child's incoming receives nothing before its parent's
  // interpolation (its own plane waves come at the next level), so the RMW
  // of the reference's "+=" (dmk.cpp:850) is an add to exact zeros
  k_tensor3<PC><<<grid, kT3W * 32, smem, st>>>(p, mats, in_list, out_box, ci, 1, nch, src, dst, 0, seg);
}


// Downward interpolation of one parent into its 2^3 children with the
// shared prefix of the separable applies (dmk.cpp:835-855):
//   out_c = (Mz_cz (x) My_cy (x) Mx_cx) in,   c = cx | cy << 1 | cz << 2.
// z is contracted first, per group of 8 output slabs iz0..iz0+7:
//   Z  : Z_cz[s][jy][jx]  = sum_jz Mz_cz[iz0+s][jz] in[jz][jy][jx]   (2 variants)
//   Y  : Y_cz,cy[s][iy][jx] = sum_jy My_cy[iy][jy] Z_cz[s][jy][jx]   (4, two at a time)
//   X  : out_c[iz0+s][iy][ix] = sum_jx Y_cz,cy[s][iy][jx] Mx_cx[ix][jx] (8)
// -- 14 p^4 DMMA work per parent and channel instead of 24 p^4 for eight
// independent children, and every output is final when written (write-only:
// a child's incoming is zero before its parent's interpolation).  One CTA per
// (parent, channel), 12 warps; Z and Y live in shared memory (fragment
// strides == 4 mod 8 doubles); the input is read from L2 once per group.
constexpr int kTDW = 12;
template <int PC>
__global__ void __launch_bounds__(kTDW * 32, 1)
    k_tensor_down(const double* __restrict__ mats, const int* __restrict__ in_list, const int* __restrict__ out_box,
                  const int* __restrict__ ci_list, const int* __restrict__ seg, int nch, const double* __restrict__ src,
                  double* __restrict__ dst) {
  constexpr int p = PC, pp = p * p, nodes = p * pp;
  constexpr int P8 = 24, SA = 28, SZ = 28, PL = P8 * SZ;  // plane: 24 rows x SZ
  constexpr int NN = (pp + 7) / 8;                        // Z-stage column tiles
  constexpr int ZNT = (NN + kTDW - 1) / kTDW;             // per warp
  static_assert(p >= 17 && p <= 24, "PT = 3 shapes");
  extern __shared__ double sm[];
  double* Mm = sm;            // [2][P8][SA]
  double* Zs = Mm + 2 * P8 * SA;  // [2 cz][8 s] planes [jy][jx]
  double* Ys = Zs + 16 * PL;      // [2 cz][8 s] planes [iy][jx] for one cy
  __shared__ int s_out[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int r = warp; r < 2 * P8; r += kTDW) {
    const int bsel = r / P8, rr = r % P8;
    for (int c = lane; c < SA; c += 32) Mm[r * SA + c] = (rr < p && c < p) ? mats[(size_t)bsel * pp + rr * p + c] : 0.0;
  }
  for (int e = tid; e < 32 * PL; e += blockDim.x) Zs[e] = 0.0;  // padding rows / columns stay zero (Zs and Ys)
  const int par = blockIdx.x, ch = blockIdx.y;
  if (tid < 8) s_out[tid] = -1;
  __syncthreads();
  int parent = 0;
  for (int q = seg[par]; q < seg[par + 1]; ++q) {
    parent = in_list[q];
    if (tid == 0) s_out[ci_list[q] & 7] = out_box[q];
  }
  __syncthreads();
  unsigned have = 0;  // children present
#pragma unroll
  for (int c = 0; c < 8; ++c) have |= (s_out[c] >= 0 ? 1u : 0u) << c;
  const double* in = src + ((size_t)parent * nch + ch) * nodes;
  for (int iz0 = 0; iz0 < p; iz0 += 8) {
    // ---- Z stage: rows (cz, s), columns n = jy * p + jx, K = jz
    {
      double c[2][ZNT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int i = 0; i < ZNT; ++i) c[m][i][0] = c[m][i][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 6; ++ks) {
        const int jz = ks * 4 + t;
        double b[ZNT];
#pragma unroll
        for (int i = 0; i < ZNT; ++i) {
          const int n = (warp + kTDW * i) * 8 + g;
          b[i] = (jz < p && n < pp && warp + kTDW * i < NN) ? __ldg(in + (size_t)jz * pp + n) : 0.0;
        }
        const double a0 = Mm[(0 * P8 + iz0 + g) * SA + jz], a1 = Mm[(1 * P8 + iz0 + g) * SA + jz];
#pragma unroll
        for (int i = 0; i < ZNT; ++i) {
          dev::dmma(c[0][i][0], c[0][i][1], a0, b[i]);
          dev::dmma(c[1][i][0], c[1][i][1], a1, b[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < ZNT; ++i) {
        const int nt = warp + kTDW * i;
        if (nt >= NN) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = nt * 8 + 2 * t + e;
          if (n >= pp) continue;
          const int jy = n / p, jx = n - jy * p;
#pragma unroll
          for (int m = 0; m < 2; ++m) Zs[(m * 8 + g) * PL + jy * SZ + jx] = c[m][i][e];
        }
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int cy = 0; cy < 2; ++cy) {
      const unsigned need = have & (cy ? 0xCCu : 0x33u);  // children with this cy
      if (!need) continue;
      // ---- Y stage: plane P = (cz, s): Y[iy][jx] = sum_jy My[iy][jy] Z[jy][jx];
      // unit (P, iy tile) x the 3 jx tiles
      const double* My = Mm + cy * P8 * SA;
      for (int u = warp; u < 48; u += kTDW) {
        const int P = u / 3, it = u % 3;
        if (!(need & (0x0Fu << (4 * (P >> 3))))) continue;  // no child with this cz
        const double* Zp = Zs + P * PL;
        double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int ks = 0; ks < 6; ++ks) {
          const double a = My[(it * 8 + g) * SA + ks * 4 + t];
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dev::dmma(c[nt][0], c[nt][1], a, Zp[(ks * 4 + t) * SZ + nt * 8 + g]);
        }
        double* Yp = Ys + P * PL + (it * 8 + g) * SZ;
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) {
          Yp[nt * 8 + 2 * t] = c[nt][0];
          Yp[nt * 8 + 2 * t + 1] = c[nt][1];
        }
      }
      __syncthreads();
      // ---- X stage: unit (P, cx, iy tile) x the 3 ix tiles, straight to the child
      for (int u = warp; u < 96; u += kTDW) {
        const int P = u / 6, cx = (u / 3) & 1, it = u % 3;
        const int cz = P >> 3, s = P & 7, child = cx | (cy << 1) | (cz << 2);
        const int iz = iz0 + s;
        if (s_out[child] < 0 || iz >= p) continue;
        const double* Yp = Ys + P * PL;
        const double* Mx = Mm + cx * P8 * SA;
        double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int ks = 0; ks < 6; ++ks) {
          const double a = Yp[(it * 8 + g) * SZ + ks * 4 + t];
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dev::dmma(c[nt][0], c[nt][1], a, Mx[(nt * 8 + g) * SA + ks * 4 + t]);
        }
        const int iy = it * 8 + g;
        if (iy < p) {
          double* o = dst + ((size_t)s_out[child] * nch + ch) * nodes + (size_t)iz * pp + iy * p;
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) {
            const int ix = nt * 8 + 2 * t;
            if (ix < p) o[ix] = c[nt][0];
            if (ix + 1 < p) o[ix + 1] = c[nt][1];
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int PC>
void tensor_down_t(const double* mats, const int* in_list, const int* out_box, const int* ci, const int* seg,
                   int nseg, int nch, const double* src, double* dst, cudaStream_t st) {
  const size_t smem = sizeof(double) * (2 * 24 * 28 + 32 * 24 * 28);
  cudaFuncSetAttribute(k_tensor_down<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(nseg, nch);
  k_tensor_down<PC><<<grid, kTDW * 32, smem, st>>>(mats, in_list, out_box, ci, seg, nch, src, dst);
}


// Upward merge of the 2^3 children into their parent with the shared suffix
// of the separable applies (dmk.cpp:624-653), the mirror of k_tensor_down:
//   parent = sum_c (Mz_cz (x) My_cy (x) Mx_cx) child_c,   c = cx | cy << 1 | cz << 2.
// Per group of G input slabs jz0..jz0+G-1 (children streamed from L2):
//   X : S_cz,cy[s][jy][ix] = sum_cx sum_jx child_c[jz0+s][jy][jx] Mx_cx[ix][jx]   (K = 2p)
//   Y : T_cz[s][iy][ix]    = sum_cy sum_jy My_cy[iy][jy] S_cz,cy[s][jy][ix]       (K = 2p)
//   Z : parent[iz][iy,ix] += sum_cz sum_s Mz_cz[iz][jz0+s] T_cz[s][iy][ix]       (K = 2G)
// -- 14 p^4 DMMA work per parent and channel instead of 24 p^4 for eight
// independent children; the parent accumulates in registers over the groups
// (12 warps x up to 6 column tiles x 3 row tiles) and is written once.
// Missing children (no sources) read as zeros.
constexpr int kTUW = 12, kTUG = 4;
template <int PC>
__global__ void __launch_bounds__(kTUW * 32, 1)
    k_tensor_up(const double* __restrict__ mats, const int* __restrict__ in_list, const int* __restrict__ out_box,
                const int* __restrict__ ci_list, int nch, const double* __restrict__ src, double* __restrict__ dst) {
  constexpr int p = PC, pp = p * p, nodes = p * pp, G = kTUG;
  constexpr int P8 = 24, SA = 28, SZ = 28, PL = P8 * SZ;  // plane: 24 rows x SZ
  constexpr int NN = (pp + 7) / 8;                        // Z-stage column tiles
  constexpr int ZNT = (NN + kTUW - 1) / kTUW;             // per warp
  static_assert(p >= 17 && p <= 24, "PT = 3 shapes");
  extern __shared__ double sm[];
  double* Mm = sm;                // [2][P8][SA]
  double* Ss = Mm + 2 * P8 * SA;  // [4 (cz,cy)][G] planes [jy][ix]
  double* Ts = Ss + 4 * G * PL;   // [2 cz][G] planes [iy][ix]
  __shared__ int s_in[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  for (int r = warp; r < 2 * P8; r += kTUW) {
    const int bsel = r / P8, rr = r % P8;
    for (int c = lane; c < SA; c += 32) Mm[r * SA + c] = (rr < p && c < p) ? mats[(size_t)bsel * pp + rr * p + c] : 0.0;
  }
  const int par = blockIdx.x, ch = blockIdx.y;
  if (tid < 8) s_in[tid] = -1;
  __syncthreads();
  if (tid < 8) {
    const int ib = in_list[par * 8 + tid];
    if (ib >= 0) s_in[ci_list[par * 8 + tid] & 7] = ib;
  }
  __syncthreads();
#ifndef SDMK_TU_REGB
#define SDMK_TU_REGB 0
#endif
#if SDMK_TU_REGB
  // X-stage B fragments (Mx_cx, all ix tiles and k-steps) stay in registers
  double bx[2][3][6];
#pragma unroll
  for (int cx = 0; cx < 2; ++cx)
#pragma unroll
    for (int nt = 0; nt < 3; ++nt)
#pragma unroll
      for (int ks = 0; ks < 6; ++ks) bx[cx][nt][ks] = Mm[(cx * P8 + nt * 8 + g) * SA + ks * 4 + t];
#define TU_BX(cx, nt, ks) bx[cx][nt][ks]
#else
#define TU_BX(cx, nt, ks) Mm[((cx) * P8 + (nt) * 8 + g) * SA + (ks) * 4 + t]
#endif
  double acc[ZNT][3][2];
#pragma unroll
  for (int i = 0; i < ZNT; ++i)
#pragma unroll
    for (int m = 0; m < 3; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
  for (int jz0 = 0; jz0 < p; jz0 += G) {
    // ---- X stage: unit (pair (cz,cy), slab s, jy tile) x the 3 ix tiles
    for (int u = warp; u < 4 * G * 3; u += kTUW) {
      const int pr = u / (3 * G), s = (u / 3) % G, it = u % 3;
      const int jz = jz0 + s, jy = it * 8 + g;
      double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        const int cb = s_in[cx | (pr << 1)];
        const bool ok = cb >= 0 && jz < p && jy < p;
        const double* in = src + ((size_t)(cb >= 0 ? cb : 0) * nch + ch) * nodes + (size_t)(jz < p ? jz : 0) * pp +
                           (jy < p ? jy : 0) * p;
        double a[6];
#pragma unroll
        for (int ks = 0; ks < 6; ++ks) {
          const int jx = ks * 4 + t;
          a[ks] = (ok && jx < p) ? __ldg(in + jx) : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < 6; ++ks)
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dev::dmma(c[nt][0], c[nt][1], a[ks], TU_BX(cx, nt, ks));
      }
      double* Sp = Ss + (pr * G + s) * PL + jy * SZ;
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        Sp[nt * 8 + 2 * t] = c[nt][0];
        Sp[nt * 8 + 2 * t + 1] = c[nt][1];
      }
    }
    __syncthreads();
    // ---- Y stage: unit (cz, slab s, iy tile) x the 3 ix tiles, K = (cy, jy)
    for (int u = warp; u < 2 * G * 3; u += kTUW) {
      const int cz = u / (3 * G), s = (u / 3) % G, it = u % 3;
      double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int cy = 0; cy < 2; ++cy) {
        const double* My = Mm + cy * P8 * SA + (it * 8 + g) * SA;
        const double* Sp = Ss + ((cz * 2 + cy) * G + s) * PL;
#pragma unroll
        for (int ks = 0; ks < 6; ++ks) {
          const double a = My[ks * 4 + t];
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dev::dmma(c[nt][0], c[nt][1], a, Sp[(ks * 4 + t) * SZ + nt * 8 + g]);
        }
      }
      double* Tp = Ts + (cz * G + s) * PL + (it * 8 + g) * SZ;
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        Tp[nt * 8 + 2 * t] = c[nt][0];
        Tp[nt * 8 + 2 * t + 1] = c[nt][1];
      }
    }
    __syncthreads();
    // ---- Z stage: parent[iz][n] += sum_(cz, s) Mz_cz[iz][jz0 + s] T_cz[s][n], n = iy p + ix
    {
      double a[3][2];
#pragma unroll
      for (int mt = 0; mt < 3; ++mt)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = kk * 4 + t, cz = k / G, sl = k % G;
          a[mt][kk] = jz0 + sl < p ? Mm[(cz * P8 + mt * 8 + g) * SA + jz0 + sl] : 0.0;
        }
#pragma unroll
      for (int i = 0; i < ZNT; ++i) {
        const int nt = warp + kTUW * i;
        if (nt >= NN) continue;
        const int n = nt * 8 + g;
        const int iy = n / p, ix = n - iy * p;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = kk * 4 + t, cz = k / G, sl = k % G;
          const double b = n < pp ? Ts[(cz * G + sl) * PL + iy * SZ + ix] : 0.0;
#pragma unroll
          for (int mt = 0; mt < 3; ++mt) dev::dmma(acc[i][mt][0], acc[i][mt][1], a[mt][kk], b);
        }
      }
    }
    __syncthreads();
  }
  double* out = dst + ((size_t)out_box[par] * nch + ch) * nodes;
#pragma unroll
  for (int i = 0; i < ZNT; ++i) {
    const int nt = warp + kTUW * i;
    if (nt >= NN) continue;
#pragma unroll
    for (int mt = 0; mt < 3; ++mt) {
      const int iz = mt * 8 + g;
      if (iz >= p) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = nt * 8 + 2 * t + e;
        if (n < pp) out[(size_t)iz * pp + n] = acc[i][mt][e];
      }
    }
  }
}

template <int PC>
void tensor_up_t(const double* mats, const int* in_list, const int* out_box, const int* ci, int nparents, int nch,
                 const double* src, double* dst, cudaStream_t st) {
  const size_t smem = sizeof(double) * (2 * 24 * 28 + 6 * kTUG * 24 * 28);
  cudaFuncSetAttribute(k_tensor_up<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(nparents, nch);
  k_tensor_up<PC><<<grid, kTUW * 32, smem, st>>>(mats, in_list, out_box, ci, nch, src, dst);
}
}  // namespace

bool tensor_seg_supported(int p, int dim) { return dim == 3 && p >= 17 && p <= 24; }

void launch_tensor_mma_seg(int p, const double* mats, const int* in_list, const int* out_box, const int* ci,
                           const int* seg, int nseg, int nch, const double* src, double* dst, cudaStream_t st) {
  if (nseg <= 0) return;
  if (p == 23) tensor_down_t<23>(mats, in_list, out_box, ci, seg, nseg, nch, src, dst, st);
  else if (p == 22) tensor_down_t<22>(mats, in_list, out_box, ci, seg, nseg, nch, src, dst, st);
  else tensor3_seg_t<0>(p, mats, in_list, out_box, ci, seg, nseg, nch, src, dst, st);
}


bool tensor_mma_supported(int p, int dim) { return dim == 3 && p >= 4 && p <= 32; }

void launch_tensor_mma(int p, const double* mats, const int* in_list, const int* out_box, const int* ci, int npairs,
                       int nch, const double* src, double* dst, int accumulate, int dim, cudaStream_t st) {
  if (npairs <= 0) return;
  // accumulate: 1 dst += (one input per pair), 2 merge (2^d inputs, dst =),
  // 3 one input per pair, dst = (downward interpolation into zeroed children)
  const int nin = accumulate == 2 ? (1 << dim) : 1;
  const int acc = accumulate == 1 ? 1 : 0;
  const int PT = (p + 7) / 8;
#define TM(PC_, PT_, NW_, ZT_) \
  tensor_mma_t<PC_, PT_, NW_, ZT_>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st)
  if (accumulate == 2 && dim == 3 && (p == 22 || p == 23)) {  // merges: shared suffix
    if (p == 23) tensor_up_t<23>(mats, in_list, out_box, ci, npairs, nch, src, dst, st);
    else tensor_up_t<22>(mats, in_list, out_box, ci, npairs, nch, src, dst, st);
    return;
  }
  if (p == 22) tensor3_t<22>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (p == 23) tensor3_t<23>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (PT == 3) tensor3_t<0>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (p == 30) tensor4_t<30>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (PT == 4) tensor4_t<0>(p, mats, in_list, out_box, ci, npairs, nin, nch, src, dst, acc, st);
  else if (PT <= 1) TM(0, 1, 4, 8);
  else TM(0, 2, 8, 12);
#undef TM
}

}  // namespace sdmkb
