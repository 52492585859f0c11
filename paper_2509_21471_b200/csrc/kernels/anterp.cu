// K3 leaf anterpolation (dmk.cpp:587-622) and K11 target interpolation
// (dmk.cpp:877-913) on sm_100a, FP64.
//
// K3 is a per-leaf GEMM  W[(ch,iz,iy), ix] = sum_a A[(ch,iz,iy), a] bx[a, ix]
// with A = s_ch(a) bz(a,iz) by(a,iy) formed on the fly: the CTA stages the
// Lagrange bases of a tile of points in shared memory and every thread keeps
// two output rows (2 x p doubles) in registers, so each broadcast shared load
// of bx feeds two FMAs.  K11 is the transposed contraction; each thread owns
// one target and streams the leaf's incoming grid slab by slab.
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

using dev::DBox;

constexpr int kTile = 32;       // points per shared-memory tile (K3)
constexpr int kAntBlock = 256;  // threads per CTA (K3); 2 rows per thread
constexpr int kIntBlock = 128;  // threads (targets) per CTA (K11)

// build_source_channels (dmk.cpp:492-525) from SoA strengths
__device__ __forceinline__ void source_channels(int kernel, int dim, const double* __restrict__ str, int n,
                                                int a, double* ch) {
  if (kernel == 0) {  // stokeslet force
    for (int j = 0; j < dim; ++j) ch[j] = str[(size_t)j * n + a];
    return;
  }
  if (kernel == 1) {  // stresslet: f n^T + n f^T + (f.n) I, packed diagonal first
    double f[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, w = 0.0;
    for (int j = 0; j < dim; ++j) {
      f[j] = str[(size_t)j * n + a];
      nn[j] = str[(size_t)(dim + j) * n + a];
    }
    for (int j = 0; j < dim; ++j) w += f[j] * nn[j];
    if (dim == 3) {
      ch[0] = 2.0 * f[0] * nn[0] + w;
      ch[1] = 2.0 * f[1] * nn[1] + w;
      ch[2] = 2.0 * f[2] * nn[2] + w;
      ch[3] = f[0] * nn[1] + f[1] * nn[0];
      ch[4] = f[0] * nn[2] + f[2] * nn[0];
      ch[5] = f[1] * nn[2] + f[2] * nn[1];
    } else {
      ch[0] = 2.0 * f[0] * nn[0] + w;
      ch[1] = 2.0 * f[1] * nn[1] + w;
      ch[2] = f[0] * nn[1] + f[1] * nn[0];
    }
    return;
  }
  int nc = dim == 3 ? 3 : 1;  // rotlet torque
  for (int j = 0; j < nc; ++j) ch[j] = str[(size_t)j * n + a];
}

template <int PM>
__global__ void __launch_bounds__(kAntBlock) k_anterp(int kernel, ChebDev cb, const DBox* __restrict__ boxes,
                                                      const int* __restrict__ leaves,
                                                      const double* __restrict__ pts, int n,
                                                      const double* __restrict__ str,
                                                      double* __restrict__ out, int nch) {
  extern __shared__ double sm[];
  const int p = cb.p, pz = cb.pz, dim = cb.dim;
  double* nodes = sm;                      // p
  double* wts = nodes + p;                 // p
  double* bxs = wts + p;                   // kTile * p
  double* bys = bxs + kTile * p;           // kTile * p
  double* bzs = bys + kTile * p;           // kTile * p
  double* svs = bzs + kTile * p;           // kTile * 6
  const int tid = threadIdx.x;
  for (int i = tid; i < p; i += blockDim.x) {
    nodes[i] = cb.nodes[i];
    wts[i] = cb.wts[i];
  }
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  const int plane = pz * p, nrows = nch * plane;
  const int r0 = blockIdx.y * (2 * kAntBlock) + tid, r1 = r0 + kAntBlock;
  const bool v0 = r0 < nrows, v1 = r1 < nrows;
  const int ch0 = v0 ? r0 / plane : 0, iz0 = v0 ? (r0 % plane) / p : 0, iy0 = v0 ? r0 % p : 0;
  const int ch1 = v1 ? r1 / plane : 0, iz1 = v1 ? (r1 % plane) / p : 0, iy1 = v1 ? r1 % p : 0;
  double acc0[PM], acc1[PM];
#pragma unroll
  for (int i = 0; i < PM; ++i) acc0[i] = acc1[i] = 0.0;
  const double hinv = 1.0 / box.half;  // half is a power of two: (x-c)/half == (x-c)*hinv
  __syncthreads();
  for (int a0 = box.sb; a0 < box.se; a0 += kTile) {
    const int tp = min(kTile, box.se - a0);
    for (int task = tid; task < tp * dim; task += blockDim.x) {
      int pt = task / dim, ax = task % dim;
      double x = __dmul_rn(__dsub_rn(pts[(size_t)ax * n + a0 + pt], box.c[ax]), hinv);
      double* dst = (ax == 0 ? bxs : (ax == 1 ? bys : bzs)) + pt * p;
      dev::cheb_basis(p, nodes, wts, x, dst, 1);
    }
    if (dim == 2)
      for (int pt = tid; pt < tp; pt += blockDim.x) bzs[pt * p] = 1.0;
    for (int pt = tid; pt < tp; pt += blockDim.x) source_channels(kernel, dim, str, n, a0 + pt, svs + pt * 6);
    __syncthreads();
    for (int pt = 0; pt < tp; ++pt) {
      const double* bxr = bxs + pt * p;
      double A0 = v0 ? svs[pt * 6 + ch0] * (bzs[pt * p + iz0] * bys[pt * p + iy0]) : 0.0;
      double A1 = v1 ? svs[pt * 6 + ch1] * (bzs[pt * p + iz1] * bys[pt * p + iy1]) : 0.0;
#pragma unroll
      for (int ix = 0; ix < PM; ++ix) {
        if (ix < p) {
          double bv = bxr[ix];
          acc0[ix] = fma(A0, bv, acc0[ix]);
          acc1[ix] = fma(A1, bv, acc1[ix]);
        }
      }
    }
    __syncthreads();
  }
  double* ob = out + (size_t)b * nrows * p;
  if (v0) {
#pragma unroll
    for (int ix = 0; ix < PM; ++ix)
      if (ix < p) ob[(size_t)r0 * p + ix] = acc0[ix];
  }
  if (v1) {
#pragma unroll
    for (int ix = 0; ix < PM; ++ix)
      if (ix < p) ob[(size_t)r1 * p + ix] = acc1[ix];
  }
}

// BLK targets per CTA (one per thread): BLK, or 64 for p > 48 (the three
// basis columns per target would not fit shared memory)
template <int PM, int BLK>
__global__ void __launch_bounds__(BLK) k_interp(ChebDev cb, const DBox* __restrict__ boxes,
                                                      const int* __restrict__ leaves,
                                                      const double* __restrict__ tpts, int nt,
                                                      const int* __restrict__ tperm,
                                                      const double* __restrict__ incoming,
                                                      double* __restrict__ ufar) {
  extern __shared__ double sm[];
  const int p = cb.p, pz = cb.pz, dim = cb.dim;
  double* nodes = sm;
  double* wts = nodes + p;
  double* bxs = wts + p;               // p * BLK (column per thread)
  double* bys = bxs + p * BLK;   // p * BLK
  double* bzs = bys + p * BLK;   // p * BLK
  double* slab = bzs + p * BLK;  // dim * p * p
  const int tid = threadIdx.x;
  for (int i = tid; i < p; i += blockDim.x) {
    nodes[i] = cb.nodes[i];
    wts[i] = cb.wts[i];
  }
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  const int pp = p * p, nodes_per = pz * pp;
  const double* win = incoming + (size_t)b * dim * nodes_per;
  const double hinv = 1.0 / box.half;
  __syncthreads();
  for (int t0 = box.tb; t0 < box.te; t0 += BLK) {
    const int t = t0 + tid;
    const bool act = t < box.te;
    if (act) {
      for (int ax = 0; ax < dim; ++ax) {
        double x = __dmul_rn(__dsub_rn(tpts[(size_t)ax * nt + t], box.c[ax]), hinv);
        double* dst = (ax == 0 ? bxs : (ax == 1 ? bys : bzs)) + tid;
        dev::cheb_basis(p, nodes, wts, x, dst, BLK);
      }
      if (dim == 2) bzs[tid] = 1.0;
    }
    double bx[PM];
#pragma unroll
    for (int i = 0; i < PM; ++i) bx[i] = (i < p && act) ? bxs[i * BLK + tid] : 0.0;
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    for (int iz = 0; iz < pz; ++iz) {
      __syncthreads();
      for (int e = tid; e < dim * pp; e += blockDim.x) {
        int j = e / pp, r = e % pp;
        slab[e] = win[(size_t)j * nodes_per + (size_t)iz * pp + r];
      }
      __syncthreads();
      const double wz = act ? bzs[iz * BLK + tid] : 0.0;
      for (int iy = 0; iy < p; ++iy) {
        const double wzy = wz * (act ? bys[iy * BLK + tid] : 0.0);
        const double* r0 = slab + iy * p;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int ix = 0; ix < PM; ++ix) {
          if (ix < p) {
            s0 = fma(bx[ix], r0[ix], s0);
            s1 = fma(bx[ix], r0[pp + ix], s1);
            if (dim == 3) s2 = fma(bx[ix], r0[2 * pp + ix], s2);
          }
        }
        u0 = fma(wzy, s0, u0);
        u1 = fma(wzy, s1, u1);
        u2 = fma(wzy, s2, u2);
      }
    }
    if (act) {
      double* ut = ufar + (size_t)tperm[t] * dim;
      ut[0] = u0;
      ut[1] = u1;
      if (dim == 3) ut[2] = u2;
    }
  }
}

template <int PM>
void anterp_t(int kernel, const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* pts,
              int n, const double* str, double* out, int nch, cudaStream_t st) {
  int rows = nch * cb.pz * cb.p;
  dim3 grid(nleaf, (rows + 2 * kAntBlock - 1) / (2 * kAntBlock));
  size_t smem = sizeof(double) * (2 * cb.p + 3 * kTile * cb.p + kTile * 6);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_anterp<PM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_anterp<PM><<<grid, kAntBlock, smem, st>>>(kernel, cb, boxes, leaves, pts, n, str, out, nch);
}

template <int PM>
void interp_t(const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* tpts, int nt,
              const int* tperm, const double* incoming, double* ufar, cudaStream_t st) {
  constexpr int BLK = PM > 48 ? 64 : kIntBlock;
  size_t smem = sizeof(double) * (2 * cb.p + 3 * cb.p * BLK + cb.dim * cb.p * cb.p);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_interp<PM, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  k_interp<PM, BLK><<<nleaf, BLK, smem, st>>>(cb, boxes, leaves, tpts, nt, tperm, incoming, ufar);
}

}  // namespace

#define SDMK_PDISPATCH(P, CALL)                   \
  do {                                            \
    if ((P) <= 8) CALL(8);                        \
    else if ((P) <= 12) CALL(12);                 \
    else if ((P) <= 16) CALL(16);                 \
    else if ((P) <= 20) CALL(20);                 \
    else if ((P) <= 24) CALL(24);                 \
    else if ((P) <= 28) CALL(28);                 \
    else if ((P) <= 32) CALL(32);                 \
    else if ((P) <= 40) CALL(40);                 \
    else if ((P) <= 48) CALL(48);                 \
    else CALL(64);                                \
  } while (0)

void launch_anterp(int kernel, const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf,
                   const double* pts, int n, const double* str, double* outgoing, int nch, cudaStream_t st) {
  if (nleaf <= 0) return;
#define CALL(PMV) anterp_t<PMV>(kernel, cb, boxes, leaves, nleaf, pts, n, str, outgoing, nch, st)
  SDMK_PDISPATCH(cb.p, CALL);
#undef CALL
}

void launch_interp_targets(const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* tpts,
                           int nt, const int* tperm, const double* incoming, double* ufar, cudaStream_t st) {
  if (nleaf <= 0) return;
#define CALL(PMV) interp_t<PMV>(cb, boxes, leaves, nleaf, tpts, nt, tperm, incoming, ufar, st)
  SDMK_PDISPATCH(cb.p, CALL);
#undef CALL
}

}  // namespace sdmkb
