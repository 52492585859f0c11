// K3 (leaf anterpolation, dmk.cpp:587-622) and K11 (target interpolation,
// dmk.cpp:877-913) on the FP64 tensor cores (mma.sync m8n8k4 f64, "DMMA").
//
// k_basis   : barycentric Lagrange bases of every point of every leaf, three
//             axes, written once to HBM ([axis][point][p]); K3 and K11 (alias
//             targets) share them.
// K3        : per leaf, C[(ch,iz,iy), ix] = sum_a A[(ch,iz,iy), a] * bx[a, ix]
//             with A = (s_ch(a) bz(a,iz)) by(a,iy) formed while building the A
//             fragment.  Warps own up to 8 m-tiles x all n-tiles; the points
//             stream through shared memory 32 at a time.
// K11       : per leaf, C[a, (j,iz,iy)] = sum_ix bx[a, ix] W[(j,iz,iy), ix]
//             (W = the leaf's incoming proxy grid streamed through shared
//             memory in 256-row chunks), reduced on the fly with the weights
//             bz(a,iz) by(a,iy) into u[a][j]; one 8-target m-tile per warp.
// Shared-memory row strides are chosen = 8 (mod 16) doubles (resp. KP + 4)
// so every fragment load is bank-conflict free.
#include "common.cuh"
#include "launch.hpp"

#include <cstdlib>

namespace sdmkb {

namespace {

using dev::DBox;

// Shared-memory row stride (in doubles) for fragment loads: a warp-wide 8-byte
// load is served per half-warp, whose 16 lanes touch 4 rows x 4 consecutive
// columns; a stride == 4 (mod 8) puts the 4 rows on disjoint bank quads.
__host__ __device__ __forceinline__ int cstride(int x) {  // smallest y >= x with y % 8 == 4
  int y = (x + 3) / 4 * 4;
  return (y % 8 == 4) ? y : y + 4;
}

// ---------------------------------------------------------------- bases --
// Barycentric Lagrange basis (dmk.cpp:39-53) without p divisions per point:
// with d_j = x - x_j, w_i / d_i = w_i q_i / P where q_i = prod_{j != i} d_j and
// P = prod_j d_j, and P cancels in the normalisation, so
//   l_i(x) = w_i q_i / sum_j w_j q_j
// (q from prefix / suffix products; one division per point and axis).  The
// exact-hit rule is kept.  A warp owns 32 consecutive points of one axis; the
// rows are assembled in shared memory and stored coalesced.
// PC > 0: p known at compile time -- the products stay in registers and each
// row is written to shared memory once (the generic form passes through it
// three times); the arithmetic and its order are the same.
constexpr int kBasisW = 8;
template <int PC>
__global__ void __launch_bounds__(kBasisW * 32) k_basis(ChebDev cb, const DBox* __restrict__ boxes,
                                                       const int* __restrict__ leaves, const double* __restrict__ pts,
                                                       int n, int use_targets, double* __restrict__ basis) {
  __shared__ double nodes[64], wts[64];
  extern __shared__ double rowbuf[];  // [kBasisW][32][p | 1]: odd row stride, conflict-free lanes
  const int p = PC > 0 ? PC : cb.p, dim = cb.dim, P1 = p | 1;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    nodes[i] = cb.nodes[i];
    wts[i] = cb.wts[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* rb = rowbuf + warp * 32 * P1;
  const DBox box = boxes[leaves[blockIdx.x]];
  const int b0 = use_targets ? box.tb : box.sb, b1 = use_targets ? box.te : box.se;
  const double hinv = 1.0 / box.half;
  const int cnt = b1 - b0, nchunk = (cnt + 31) / 32;
  for (int task = warp; task < nchunk * dim; task += kBasisW) {
    const int ax = task / nchunk, i0 = b0 + (task % nchunk) * 32, i = i0 + lane;
    const int nv = min(32, b1 - i0);
    double* r = rb + lane * P1;
    if (PC > 0) {
      if (lane < nv) {
        constexpr int PR = PC > 0 ? PC : 1;
        const double x = __dmul_rn(__dsub_rn(pts[(size_t)ax * n + i], box.c[ax]), hinv);
        double rr[PR];
        int hit = -1;
        double pre = 1.0;
#pragma unroll
        for (int k = 0; k < PR; ++k) {  // rr[k] = prod_{j < k} d_j
          const double dk = x - nodes[k];
          if (dk == 0.0) hit = hit < 0 ? k : hit;
          rr[k] = pre;
          pre *= dk;
        }
        if (hit >= 0) {
#pragma unroll
          for (int k = 0; k < PR; ++k) r[k] = k == hit ? 1.0 : 0.0;
        } else {
          double suf = 1.0, sum = 0.0;
#pragma unroll
          for (int k = PR - 1; k >= 0; --k) {  // rr[k] = w_k prod_{j != k} d_j
            const double v = wts[k] * (rr[k] * suf);
            rr[k] = v;
            sum += v;
            suf *= x - nodes[k];
          }
          const double inv = 1.0 / sum;
#pragma unroll
          for (int k = 0; k < PR; ++k) r[k] = rr[k] * inv;
        }
      }
    } else if (lane < nv) {
      const double x = __dmul_rn(__dsub_rn(pts[(size_t)ax * n + i], box.c[ax]), hinv);
      int hit = -1;
      for (int k = 0; k < p; ++k)
        if (x == nodes[k]) hit = hit < 0 ? k : hit;
      if (hit >= 0) {
        for (int k = 0; k < p; ++k) r[k] = k == hit ? 1.0 : 0.0;
      } else {
        double pre = 1.0;
        for (int k = 0; k < p; ++k) {  // r[k] = prod_{j < k} d_j
          r[k] = pre;
          pre *= x - nodes[k];
        }
        double suf = 1.0, sum = 0.0;
        for (int k = p - 1; k >= 0; --k) {  // r[k] = w_k prod_{j != k} d_j
          const double v = wts[k] * (r[k] * suf);
          r[k] = v;
          sum += v;
          suf *= x - nodes[k];
        }
        const double inv = 1.0 / sum;
        for (int k = 0; k < p; ++k) r[k] *= inv;
      }
    }
    __syncwarp();
    double* dst = basis + ((size_t)ax * n + i0) * p;
    for (int e = lane; e < nv * p; e += 32) dst[e] = rb[(e / p) * P1 + e % p];
    __syncwarp();
  }
}

// build_source_channels (dmk.cpp:492-525) from SoA strengths
__device__ __forceinline__ void channels(int kernel, int dim, const double* __restrict__ str, int n, int a, double* ch) {
  if (kernel == 1) {
    double f[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, w = 0.0;
    for (int j = 0; j < dim; ++j) {
      f[j] = str[(size_t)j * n + a];
      nn[j] = str[(size_t)(dim + j) * n + a];
      w += f[j] * nn[j];
    }
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
  const int nc = kernel == 0 ? dim : (dim == 3 ? 3 : 1);
  for (int j = 0; j < nc; ++j) ch[j] = str[(size_t)j * n + a];
}

// -------------------------------------------------------------------- K3 --
constexpr int kKC = 32;     // points per shared chunk
constexpr int kAWarps = 8;

// Raw per-chunk data arrives by cp.async (double buffered): bx rows (the B
// operand, zero padded to NT*8), by rows, bz rows and the raw strengths.  The
// product s_ch * bz is formed once per chunk in shared memory; the A fragment
// is (s_ch bz) * by.
// PC / KC / DC > 0 (resp. >= 0 for KC) fix p, the kernel and the dimension at
// compile time so the staging index arithmetic folds (BASELINE cases).
template <int NT, int kMTW, int PC, int KC, int DC>
__global__ void __launch_bounds__(kAWarps * 32, 2) k_anterp_mma(int kernel_rt, ChebDev cb, const DBox* __restrict__ boxes,
                                                               const int* __restrict__ leaves,
                                                               const double* __restrict__ basis,
                                                               const double* __restrict__ str, int n,
                                                               double* __restrict__ out, int nch, int mt_per_cta) {
  extern __shared__ double sm[];
  const int p = PC > 0 ? PC : cb.p, dim = DC > 0 ? DC : cb.dim, pz = dim == 3 ? p : 1;
  const int kernel = KC >= 0 ? KC : kernel_rt;
  const int sc = kernel == 0 ? dim : (kernel == 1 ? 2 * dim : (dim == 3 ? 3 : 1));
  nch = kernel == 0 ? dim : (kernel == 1 ? dim * (dim + 1) / 2 : (dim == 3 ? 3 : 1));
  const int RS = cstride(nch * pz), BS = cstride(p), XS = cstride(NT * 8);
  const int RAW = kKC * (XS + 2 * BS + 8);   // one raw buffer
  double* sbz = sm;                          // [kKC][RS]  s_ch * bz(iz)
  double* raw = sbz + kKC * RS;              // 2 x { bx[kKC][XS], by[kKC][BS], bz[kKC][BS], str[kKC][8] }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  const int M = nch * pz * p, total_mt = (M + 7) / 8;
  const int mt0 = blockIdx.y * mt_per_cta, mt1 = min(total_mt, mt0 + mt_per_cta);
  int chiz[kMTW], iyv[kMTW];
  bool val[kMTW];
#pragma unroll
  for (int i = 0; i < kMTW; ++i) {
    const int mt = mt0 + warp + kAWarps * i;
    const int m = mt * 8 + g;
    val[i] = mt < mt1;
    const bool ok = val[i] && m < M;
    chiz[i] = ok ? m / p : 0;
    iyv[i] = ok ? m % p : 0;
  }
  double acc[kMTW][NT][2];
#pragma unroll
  for (int i = 0; i < kMTW; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const double* bxg = basis;
  const double* byg = basis + (size_t)n * p;
  const double* bzg = basis + (size_t)2 * n * p;
  const int nchunks = (box.se - box.sb + kKC - 1) / kKC;
  auto issue = [&](int c, int buf) {
    const int a0 = box.sb + c * kKC, kc = min(kKC, box.se - a0);
    double* rb = raw + buf * RAW;
    double* bx = rb;
    double* by = bx + kKC * XS;
    double* bz = by + kKC * BS;
    double* ss = bz + kKC * BS;
    for (int e = tid; e < kKC * XS; e += blockDim.x) {
      const int pt = e / XS, i = e % XS;
      const bool v = pt < kc && i < p;
      dev::cp_async8(bx + e, v ? bxg + (size_t)(a0 + pt) * p + i : bxg, v);
    }
    for (int e = tid; e < kKC * p; e += blockDim.x) {
      const int pt = e / p, i = e % p;
      const bool v = pt < kc;
      dev::cp_async8(by + pt * BS + i, v ? byg + (size_t)(a0 + pt) * p + i : byg, v);
      if (dim == 3) dev::cp_async8(bz + pt * BS + i, v ? bzg + (size_t)(a0 + pt) * p + i : bzg, v);
    }
    for (int e = tid; e < kKC * sc; e += blockDim.x) {
      const int pt = e / sc, j = e % sc;
      const bool v = pt < kc;
      dev::cp_async8(ss + pt * 8 + j, v ? str + (size_t)j * n + a0 + pt : str, v);
    }
    dev::cp_commit();
  };
  if (nchunks > 0) issue(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    __syncthreads();  // everyone is done with the buffer the next issue overwrites
    if (c + 1 < nchunks) {
      issue(c + 1, buf ^ 1);
      dev::cp_wait1();
    } else {
      dev::cp_wait0();
    }
    __syncthreads();
    const double* bx = raw + buf * RAW;
    const double* by = bx + kKC * XS;
    const double* bz = by + kKC * BS;
    const double* ss = bz + kKC * BS;
    for (int e = tid; e < kKC * nch; e += blockDim.x) {  // s_ch * bz (dmk.cpp:492-525 channels)
      const int pt = e / nch, ch = e % nch;
      double chv[6];
      if (kernel == 1) {
        const double* s = ss + pt * 8;
        double w = 0.0;
        for (int j = 0; j < dim; ++j) w += s[j] * s[dim + j];
        if (dim == 3) {
          chv[0] = 2.0 * s[0] * s[3] + w;
          chv[1] = 2.0 * s[1] * s[4] + w;
          chv[2] = 2.0 * s[2] * s[5] + w;
          chv[3] = s[0] * s[4] + s[1] * s[3];
          chv[4] = s[0] * s[5] + s[2] * s[3];
          chv[5] = s[1] * s[5] + s[2] * s[4];
        } else {
          chv[0] = 2.0 * s[0] * s[2] + w;
          chv[1] = 2.0 * s[1] * s[3] + w;
          chv[2] = s[0] * s[3] + s[1] * s[2];
        }
      } else {
        for (int j = 0; j < 6; ++j) chv[j] = j < sc ? ss[pt * 8 + j] : 0.0;
      }
      double sv = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j)
        if (j == ch) sv = chv[j];
      for (int iz = 0; iz < pz; ++iz) sbz[pt * RS + ch * pz + iz] = sv * (dim == 3 ? bz[pt * BS + iz] : 1.0);
    }
    __syncthreads();
    const int kc = min(kKC, box.se - (box.sb + c * kKC));
    const int ksteps = (kc + 3) / 4;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int k = ks * 4 + t;
      double bv[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) bv[j] = bx[k * XS + j * 8 + g];
#pragma unroll
      for (int i = 0; i < kMTW; ++i) {
        if (val[i]) {
          const double av = sbz[k * RS + chiz[i]] * by[k * BS + iyv[i]];
#pragma unroll
          for (int j = 0; j < NT; ++j) dev::dmma(acc[i][j][0], acc[i][j][1], av, bv[j]);
        }
      }
    }
  }
  double* ob = out + (size_t)b * M * p;
#pragma unroll
  for (int i = 0; i < kMTW; ++i) {
    if (!val[i]) continue;
    const int m = (mt0 + warp + kAWarps * i) * 8 + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int cc = j * 8 + 2 * t;
      if (cc < p) ob[(size_t)m * p + cc] = acc[i][j][0];
      if (cc + 1 < p) ob[(size_t)m * p + cc + 1] = acc[i][j][1];
    }
  }
}

// K3, second form: C[(ch,iz), (iy,ix)] = sum_a S[a, (ch,iz)] (by[a,iy] bx[a,ix])
// with S = s_ch bz formed once per chunk in shared memory (the A operand,
// fragment loads only) and the B values by * bx formed per fragment, each
// feeding all MT m-tiles of the (ch, iz) rows: 1 multiply per MT DMMAs
// instead of one per n-tile.  A warp owns NTW column tiles of the (iy, ix)
// plane; a CTA covers 8 NTW of them, so a leaf takes ceil(p^2 / 64 NTW) CTAs.
#ifndef SDMK_A2S_MT
#define SDMK_A2S_MT 17
#define SDMK_A2S_NTW 2
#endif
// warps per CTA and n-tiles per warp are template parameters (A/B measured per
// kernel: the Stokeslet runs 12 x 3 -- two CTAs per leaf --, the stresslet's
// 17 m-tiles need the registers of 12 x 2)
#ifndef SDMK_A2_KC
#define SDMK_A2_KC 32
#endif
// points per shared chunk (k_anterp2's last template parameter): 64 for the
// Stokeslet (fewer chunk barriers), 32 for the stresslet (A/B measured)
constexpr int kA2Chunk = SDMK_A2_KC;
template <int MT, int NTW, int PC, int KC, int DC, int W, int kKC2>
__global__ void __launch_bounds__(W * 32, 1) k_anterp2(ChebDev cb, const DBox* __restrict__ boxes,
                                                            const int* __restrict__ leaves,
                                                            const double* __restrict__ basis,
                                                            const double* __restrict__ str, int n,
                                                            double* __restrict__ out) {
  extern __shared__ double sm[];
  constexpr int p = PC, dim = DC, pz = dim == 3 ? p : 1, kernel = KC;
  constexpr int sc = kernel == 0 ? dim : (kernel == 1 ? 2 * dim : (dim == 3 ? 3 : 1));
  constexpr int nch = kernel == 0 ? dim : (kernel == 1 ? dim * (dim + 1) / 2 : (dim == 3 ? 3 : 1));
  constexpr int MR = nch * pz, NN = p * p;
  constexpr int RS = (MT * 8) % 8 == 4 ? MT * 8 : MT * 8 + 4;  // point rows: == 4 mod 8 (fragment loads)
  constexpr int XS = (p + 3) / 4 * 4 % 8 == 4 ? (p + 3) / 4 * 4 : (p + 3) / 4 * 4 + 4;  // == 4 mod 8
  constexpr int RAW = kKC2 * (3 * XS + 8);
  double* sbz = sm;                 // [kKC2][RS]
  double* raw = sbz + kKC2 * RS;     // 2 x { bx[kKC2][XS], by[kKC2][XS], bz[kKC2][XS], str[kKC2][8] }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  const int nt0 = blockIdx.y * W * NTW;
  __shared__ int rcode[MT * 8];  // (ch, iz) of each S row
  __shared__ double s_chv[kKC2][8];
  // rows [rb0, rb0 + 8 MT) of the MR (ch, iz) rows: blockIdx.z splits tall
  // problems (the stresslet's 6 channels) into row blocks of the same shape
  const int rb0 = blockIdx.z * MT * 8, nrow = min(MT * 8, MR - rb0);
  for (int r = tid; r < MT * 8; r += blockDim.x)
    rcode[r] = r < nrow ? (((rb0 + r) / pz) | (((rb0 + r) % pz) << 8)) : -1;
  int iyv[NTW], ixv[NTW];
#pragma unroll
  for (int j = 0; j < NTW; ++j) {
    const int col = (nt0 + warp + W * j) * 8 + g;
    iyv[j] = col < NN ? col / p : 0;
    ixv[j] = col < NN ? col % p : 0;
  }
  double acc[MT][NTW][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int e = tid; e < kKC2 * RS; e += blockDim.x) sbz[e] = 0.0;  // row padding stays zero
  const double* bxg = basis;
  const double* byg = basis + (size_t)n * p;
  const double* bzg = basis + (size_t)2 * n * p;
  const int nchunks = (box.se - box.sb + kKC2 - 1) / kKC2;
  auto issue = [&](int c, int buf) {
    const int a0 = box.sb + c * kKC2, kc = min(kKC2, box.se - a0);
    double* rb = raw + buf * RAW;
    for (int e = tid; e < kKC2 * p; e += blockDim.x) {
      const int pt = e / p, i = e % p;
      const bool v = pt < kc;
      const size_t o = (size_t)(a0 + (v ? pt : 0)) * p + i;
      dev::cp_async8(rb + pt * XS + i, bxg + o, v);
      dev::cp_async8(rb + kKC2 * XS + pt * XS + i, byg + o, v);
      if (dim == 3) dev::cp_async8(rb + 2 * kKC2 * XS + pt * XS + i, bzg + o, v);
    }
    for (int e = tid; e < kKC2 * sc; e += blockDim.x) {
      const int pt = e / sc, j = e % sc;
      const bool v = pt < kc;
      dev::cp_async8(rb + 3 * kKC2 * XS + pt * 8 + j, v ? str + (size_t)j * n + a0 + pt : str, v);
    }
    dev::cp_commit();
  };
  if (nchunks > 0) issue(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1;
    __syncthreads();  // everyone is done with the buffer the next issue overwrites (and with sbz)
    if (c + 1 < nchunks) {
      issue(c + 1, buf ^ 1);
      dev::cp_wait1();
    } else {
      dev::cp_wait0();
    }
    __syncthreads();
    const double* bx = raw + buf * RAW;
    const double* by = bx + kKC2 * XS;
    const double* bz = by + kKC2 * XS;
    const double* ss = bz + kKC2 * XS;
    // channel values once per point (build_source_channels, dmk.cpp:492-525) ...
    for (int e = tid; e < kKC2 * nch; e += blockDim.x) {
      const int pt = e / nch, ch = e % nch;
      const double* s = ss + pt * 8;
      double sv;
      if (kernel == 1) {
        double w = 0.0;
#pragma unroll
        for (int j = 0; j < dim; ++j) w += s[j] * s[dim + j];
        if (dim == 3) {
          sv = ch == 0 ? 2.0 * s[0] * s[3] + w
             : ch == 1 ? 2.0 * s[1] * s[4] + w
             : ch == 2 ? 2.0 * s[2] * s[5] + w
             : ch == 3 ? s[0] * s[4] + s[1] * s[3]
             : ch == 4 ? s[0] * s[5] + s[2] * s[3]
                       : s[1] * s[5] + s[2] * s[4];
        } else {
          sv = ch == 0 ? 2.0 * s[0] * s[2] + w : ch == 1 ? 2.0 * s[1] * s[3] + w : s[0] * s[3] + s[1] * s[2];
        }
      } else {
        sv = s[ch];
      }
      s_chv[pt][ch] = sv;
    }
    __syncthreads();
    // ... then S[pt][(ch, iz)] = s_ch * bz over all threads
    // (a warp per point row, lanes along the (ch, iz) rows: no integer division)
    for (int pt = warp; pt < kKC2; pt += W)
      for (int r = lane; r < nrow; r += 32) {
        const int code = rcode[r];
        sbz[pt * RS + r] = s_chv[pt][code & 255] * (dim == 3 ? bz[pt * XS + (code >> 8)] : 1.0);
      }
    __syncthreads();
    // k-steps of 4 points up to the chunk's last point (the rest of a partial
    // last chunk is zero padding)
    const int nks = (min(kKC2, box.se - box.sb - c * kKC2) + 3) / 4;
#pragma unroll 2
    for (int ks = 0; ks < nks; ++ks) {
      const int k = ks * 4 + t;
      double bv[NTW];
#pragma unroll
      for (int j = 0; j < NTW; ++j) bv[j] = by[k * XS + iyv[j]] * bx[k * XS + ixv[j]];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double av = sbz[k * RS + i * 8 + g];
#pragma unroll
        for (int j = 0; j < NTW; ++j) dev::dmma(acc[i][j][0], acc[i][j][1], av, bv[j]);
      }
    }
  }
  double* ob = out + (size_t)b * MR * NN;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int ml = i * 8 + g, m = rb0 + ml;
    if (ml >= nrow) continue;
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int cc = (nt0 + warp + W * j) * 8 + 2 * t;
      if (cc < NN) ob[(size_t)m * NN + cc] = acc[i][j][0];
      if (cc + 1 < NN) ob[(size_t)m * NN + cc + 1] = acc[i][j][1];
    }
  }
}

// ------------------------------------------------------------------- K11 --
#ifndef SDMK_I_ROWS
#define SDMK_I_ROWS 256  // W rows staged per chunk (rounded down to whole (j, iz) row groups)
#endif
// doubles per flat W buffer (even: 16-byte aligned buffers): the copy (RG
// row groups of p x p plus one leading alignment double, rounded to 16 bytes)
// and the furthest padded fragment read (row PY - 1, column PY - 1 of the
// last group, past the leading double)
__host__ __device__ constexpr int interp_flat(int RG, int PY, int p) {
  return ((RG * p * p + 2 > (RG - 1) * p * p + (PY - 1) * p + PY + 1 ? RG * p * p + 2
                                                                     : (RG - 1) * p * p + (PY - 1) * p + PY + 1) +
          1) & ~1;
}
// (j, iz) row groups per chunk: SDMK_I_ROWS / PY rows, cut down until the two
// flat buffers and the bz rows of one pass fit the 227 KB of shared memory at
// the widest p of the instantiation (PC, or 8 TY; 64 bytes kept for the barriers)
__host__ __device__ constexpr int interp_rg(int TY, int PC) {
  const int PY = 8 * TY, tb = TY <= 3 ? 8 * 5 * 8 : 12 * 4 * 8, pw = PC > 0 ? PC : PY;
  int rg = PY >= SDMK_I_ROWS ? 1 : SDMK_I_ROWS / PY;
  while (rg > 1 && 16 * (long)interp_flat(rg, PY, pw) + 8 * (long)tb * (pw | 1) + 64 > 232448) --rg;
  return rg;
}
// warps per CTA (IW) and m-tiles per warp (ITW) are template parameters:
// 8 x 5 for TY <= 3 (p <= 24; measured 4 % faster than 12 x 4 at p = 23),
// 12 x 4 above (the 8 x 5 accumulators would spill); one pass per leaf covers
// IW * ITW * 8 targets

// u_j(t) = sum_{iz,iy,ix} W[j,iz,iy,ix] bz[t,iz] by[t,iy] bx[t,ix]  (dmk.cpp:861-915)
//  * x contraction on the FP64 tensor cores: C[t, (j,iz,iy)] = bx[t,:] . W[(j,iz,iy),:]
//    with the (j,iz) rows padded to PY = 8 TY in iy, so every 8-column tile
//    has one (j, iz) and a fixed iy block;
//  * y contraction in the epilogue: a lane's C columns are always
//    iy = 8q + 2t + {0,1}, so its 2 TY by values per target live in registers;
//  * z contraction as one running FMA per (j, iz) row with bz from shared
//    memory, handed to component j when its last iz row is done.
// The leaf's W streams once through shared memory while every target of the
// leaf is resident: RG (j, iz) row groups per chunk are one contiguous range
// of the incoming array, moved by one 1D TMA bulk copy (cp.async.bulk, issued
// by one thread, completion on an mbarrier; double buffered) into a flat
// [rows][p] copy.  Fragment reads of the padding (iy >= p or ix >= p) are
// predicated to zero, so the flat copy needs no padded rows.  Warp w owns
// m-tiles w, w + kIW, ..., and each B fragment feeds its kITW tiles (TY x kITW
// independent DMMA chains per k-step).
template <int TY, int PC, int DC, int kIW = (TY <= 3 ? 8 : 12), int kITW = (TY <= 3 ? 5 : 4)>
__global__ void __launch_bounds__(kIW * 32, 1) k_interp_mma(ChebDev cb, const DBox* __restrict__ boxes,
                                                           const int* __restrict__ leaves,
                                                           const double* __restrict__ tbasis, int nt,
                                                           const int* __restrict__ tperm,
                                                           const double* __restrict__ incoming,
                                                           double* __restrict__ ufar) {
  constexpr int PY = 8 * TY, KS = 2 * TY;
  constexpr int kTB = kIW * kITW * 8;  // targets per pass
  constexpr int RG = interp_rg(TY, PC);  // (j, iz) rows per chunk
  extern __shared__ double sm[];
  __shared__ uint64_t bar[2];
  const int p = PC > 0 ? PC : cb.p, dim = DC > 0 ? DC : cb.dim, pz = dim == 3 ? p : 1;
  const int NG = dim * pz;          // (j, iz) rows
  const int P2 = p * p;
  const int FL = interp_flat(RG, PY, p);  // doubles per buffer
  const int BZ = p | 1;             // odd row stride: the 8 target rows of a fragment hit distinct banks
  double* Ws = sm;                  // [2][FL]
  double* bzs = Ws + 2 * FL;        // [kTB][BZ]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  if (tid == 0) {
    dev::mbar_init(&bar[0], 1);
    dev::mbar_init(&bar[1], 1);
    dev::mbar_fence_init();
  }
  const double* W = incoming + (size_t)b * NG * P2;
  const double* bxg = tbasis;
  const double* byg = tbasis + (size_t)nt * p;
  const double* bzg = tbasis + (size_t)2 * nt * p;
  const int nchunk = (NG + RG - 1) / RG;
  // chunk c: rows [c RG, c RG + ng) = W[c RG P2, (c RG + ng) P2), copied from
  // the 16-byte boundary at or below its start (sh = 1 extra leading double)
  auto shift = [&](int c) { return (int)((reinterpret_cast<uintptr_t>(W + (size_t)c * RG * P2) >> 3) & 1); };
  auto issue = [&](int c, int buf) {  // one thread
    const int ng = min(RG, NG - c * RG), sh = shift(c);
    const uint32_t bytes = (uint32_t)(((ng * P2 + sh) * 8 + 15) & ~15);
    dev::mbar_expect_tx(&bar[buf], bytes);
    dev::bulk_g2s(Ws + buf * FL, W + (size_t)c * RG * P2 - sh, bytes, &bar[buf]);
  };
  // per-lane validity of the padded fragment rows (iy) and columns (ix)
  bool vq[TY], vk[KS];
#pragma unroll
  for (int q = 0; q < TY; ++q) vq[q] = q * 8 + g < p;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) vk[ks] = ks * 4 + t < p;
  int seq = 0;  // chunks issued so far (buffer seq & 1, mbarrier phase seq >> 1)
  __syncthreads();  // barriers initialised
  for (int t0 = box.tb; t0 < box.te; t0 += kTB) {
    const int tc = min(kTB, box.te - t0);
    const int ntm = (tc + 7) / 8;
    if (tid == 0) issue(0, seq & 1);
    for (int e = tid; e < kTB * p; e += blockDim.x) {
      const int a = e / p, k = e % p;
      bzs[a * BZ + k] = a < tc ? (dim == 3 ? bzg[(size_t)(t0 + a) * p + k] : (k == 0 ? 1.0 : 0.0)) : 0.0;
    }
    double af[kITW][KS], byv[kITW][TY][2], v[kITW][3], vz[kITW];
#pragma unroll
    for (int i = 0; i < kITW; ++i) {
      const int r = (warp + kIW * i) * 8 + g;
      const bool ok = r < tc;
      const double* bxr = bxg + (size_t)(t0 + (ok ? r : 0)) * p;
      const double* byr = byg + (size_t)(t0 + (ok ? r : 0)) * p;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) af[i][ks] = (ok && ks * 4 + t < p) ? bxr[ks * 4 + t] : 0.0;
#pragma unroll
      for (int q = 0; q < TY; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) byv[i][q][e] = (ok && 8 * q + 2 * t + e < p) ? byr[8 * q + 2 * t + e] : 0.0;
      v[i][0] = v[i][1] = v[i][2] = vz[i] = 0.0;
    }
    const int nmine = warp < ntm ? (ntm - warp + kIW - 1) / kIW : 0;  // m-tiles this warp owns
    const bool full = nmine == kITW;
    __syncthreads();  // bz rows staged
    for (int c = 0; c < nchunk; ++c, ++seq) {
      const int buf = seq & 1;
      if (tid == 0 && c + 1 < nchunk) issue(c + 1, buf ^ 1);  // its buffer was released at the end of c - 1
      dev::mbar_wait(&bar[buf], (uint32_t)((seq >> 1) & 1));
      const double* Wc = Ws + buf * FL + shift(c);
      if (nmine > 0) {
        const int ng = min(RG, NG - c * RG);
        for (int gl = 0; gl < ng; ++gl) {
          const int gi = c * RG + gl, j = gi / pz, iz = gi - j * pz;
          double cc[kITW][TY][2];
#pragma unroll
          for (int i = 0; i < kITW; ++i)
#pragma unroll
            for (int q = 0; q < TY; ++q) cc[i][q][0] = cc[i][q][1] = 0.0;
          const double* Wg = Wc + gl * P2 + g * p + t;
          if (full) {
            // every m-tile: no per-DMMA predicate (each predicated DMMA costs a
            // WARPSYNC + NOP)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
              for (int q = 0; q < TY; ++q) {
                double bv = Wg[q * 8 * p + ks * 4];
                if ((PC == 0 || (q == TY - 1 && PC % 8 != 0) || (ks == KS - 1 && PC % 4 != 0)) && !(vq[q] && vk[ks]))
                  bv = 0.0;
#pragma unroll
                for (int i = 0; i < kITW; ++i) dev::dmma(cc[i][q][0], cc[i][q][1], af[i][ks], bv);
              }
          } else {
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
              for (int q = 0; q < TY; ++q) {
                double bv = Wg[q * 8 * p + ks * 4];
                if ((PC == 0 || (q == TY - 1 && PC % 8 != 0) || (ks == KS - 1 && PC % 4 != 0)) && !(vq[q] && vk[ks]))
                  bv = 0.0;
#pragma unroll
                for (int i = 0; i < kITW; ++i)
                  if (i < nmine) dev::dmma(cc[i][q][0], cc[i][q][1], af[i][ks], bv);
              }
          }
#pragma unroll
          for (int i = 0; i < kITW; ++i) {
            if (!full && i >= nmine) continue;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < TY; ++q) s = fma(byv[i][q][0], cc[i][q][0], fma(byv[i][q][1], cc[i][q][1], s));
            vz[i] = fma(s, bzs[((warp + kIW * i) * 8 + g) * BZ + iz], vz[i]);
          }
          if (iz == pz - 1) {  // the z sum of component j is complete (warp-uniform)
#pragma unroll
            for (int i = 0; i < kITW; ++i) {
#pragma unroll
              for (int jj = 0; jj < 3; ++jj)
                if (jj == j) v[i][jj] = vz[i];
              vz[i] = 0.0;
            }
          }
        }
      }
      __syncthreads();  // buffer released: the next issue overwrites it
    }
#pragma unroll
    for (int i = 0; i < kITW; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        v[i][j] += __shfl_xor_sync(0xffffffffu, v[i][j], 1);
        v[i][j] += __shfl_xor_sync(0xffffffffu, v[i][j], 2);
      }
      const int r = (warp + kIW * i) * 8 + g;
      if (t == 0 && r < tc) {
        double* ut = ufar + (size_t)tperm[t0 + r] * dim;
        ut[0] = v[i][0];
        ut[1] = v[i][1];
        if (dim == 3) ut[2] = v[i][2];
      }
    }
  }
}

void smem_attr(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

bool mma_anterp_supported(int p) { return p <= 48; }

void launch_basis(const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* pts, int n,
                  int use_targets, double* basis, cudaStream_t st) {
  if (nleaf <= 0) return;
  const size_t sm = sizeof(double) * kBasisW * 32 * (cb.p | 1);
#define KB(PC_)                                                                                              \
  do {                                                                                                       \
    smem_attr((const void*)k_basis<PC_>, sm);                                                                \
    k_basis<PC_><<<nleaf, kBasisW * 32, sm, st>>>(cb, boxes, leaves, pts, n, use_targets, basis);           \
  } while (0)
  if (cb.p == 23) KB(23);
  else if (cb.p == 22) KB(22);
  else if (cb.p == 30) KB(30);
  else KB(0);
#undef KB
}

void launch_anterp_mma(int kernel, const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf,
                       const double* basis, const double* str, int n, double* out, int nch, cudaStream_t st) {
  if (nleaf <= 0) return;
  const int p = cb.p, pz = cb.pz;
  const int M = nch * pz * p, total_mt = (M + 7) / 8;
  const int NTv = (p + 7) / 8;
  const int mtw = NTv <= 2 ? 8 : (NTv == 3 ? 6 : (NTv == 4 ? 4 : 3));
  const int per_cta_max = kAWarps * mtw;
  const int nct = (total_mt + per_cta_max - 1) / per_cta_max;
  const int mt_per = (total_mt + nct - 1) / nct;
  const size_t smem =
      sizeof(double) * (size_t)kKC * (cstride(nch * pz) + 2 * (cstride(NTv * 8) + 2 * cstride(p) + 8));
  dim3 grid(nleaf, nct);
#define AMS(NTT, MW, PC_, KC_, DC_)                                                                    \
  do {                                                                                                 \
    smem_attr((const void*)k_anterp_mma<NTT, MW, PC_, KC_, DC_>, smem);                                \
    k_anterp_mma<NTT, MW, PC_, KC_, DC_><<<grid, kAWarps * 32, smem, st>>>(kernel, cb, boxes, leaves, basis, \
                                                                           str, n, out, nch, mt_per);   \
  } while (0)
#define AM(NTT, MW) AMS(NTT, MW, 0, -1, 0)
#define A2(MT_, NTW_, PC_, KC_, W_, CH_)                                                                      \
  do {                                                                                                  \
    constexpr int RS_ = MT_ * 8 + 4;                                                                    \
    constexpr int XS_ = (PC_ + 3) / 4 * 4 % 8 == 4 ? (PC_ + 3) / 4 * 4 : (PC_ + 3) / 4 * 4 + 4;         \
    const size_t sm2 = sizeof(double) * (size_t)CH_ * (RS_ + 2 * (3 * XS_ + 8));                      \
    const int ntt = (PC_ * PC_ + 7) / 8, per = W_ * NTW_;                                             \
    smem_attr((const void*)k_anterp2<MT_, NTW_, PC_, KC_, 3, W_, CH_>, sm2);                                     \
    const int nrb = ((KC_ == 1 ? 6 : 3) * PC_ + MT_ * 8 - 1) / (MT_ * 8);                               \
    k_anterp2<MT_, NTW_, PC_, KC_, 3, W_, CH_><<<dim3(nleaf, (ntt + per - 1) / per, nrb), W_ * 32, sm2, st>>>( \
        cb, boxes, leaves, basis, str, n, out);                                                         \
  } while (0)
#ifndef SDMK_A2K_NTW
#define SDMK_A2K_NTW 3
#define SDMK_A2K_W 12
#endif
  if (cb.dim == 3 && p == 23 && kernel == 0) A2(9, SDMK_A2K_NTW, 23, 0, SDMK_A2K_W, 64);
  else if (cb.dim == 3 && p == 22 && kernel == 1) A2(SDMK_A2S_MT, SDMK_A2S_NTW, 22, 1, 12, kA2Chunk);
  else if (cb.dim == 3 && p == 30 && kernel == 0) A2(12, 2, 30, 0, 12, kA2Chunk);
  else if (NTv <= 1) AM(1, 8);
  else if (NTv == 2) AM(2, 8);
  else if (NTv == 3) AM(3, 6);
  else if (NTv == 4) AM(4, 4);
  else if (NTv == 5) AM(5, 3);
  else AM(6, 3);
#undef AM
#undef AMS
#undef A2
}

void launch_interp_mma(const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* tbasis,
                       int nt, const int* tperm, const double* incoming, double* ufar, cudaStream_t st) {
  if (nleaf <= 0) return;
  const int p = cb.p;
  const int TYv = (p + 7) / 8;
  auto smem_for = [&](int TY, int PC) {
    const int PY = 8 * TY, RG = interp_rg(TY, PC);
    const int tb = TY <= 3 ? 8 * 5 * 8 : 12 * 4 * 8;  // the kernel's IW * ITW * 8
    return sizeof(double) * (2 * (size_t)interp_flat(RG, PY, p) + (size_t)tb * (p | 1));
  };
#define IMS(TY_, PC_, DC_)                                                                                \
  do {                                                                                                    \
    size_t sm = smem_for(TY_, PC_);                                                                            \
    smem_attr((const void*)k_interp_mma<TY_, PC_, DC_>, sm);                                              \
    k_interp_mma<TY_, PC_, DC_><<<nleaf, (TY_ <= 3 ? 8 : 12) * 32, sm, st>>>(cb, boxes, leaves, tbasis, nt, tperm, incoming, ufar); \
  } while (0)
  if (cb.dim == 3 && p == 23) IMS(3, 23, 3);
  else if (cb.dim == 3 && p == 22) IMS(3, 22, 3);
  else if (cb.dim == 3 && p == 30) IMS(4, 30, 3);
  else if (TYv <= 1) IMS(1, 0, 0);
  else if (TYv == 2) IMS(2, 0, 0);
  else if (TYv == 3) IMS(3, 0, 0);
  else if (TYv == 4) IMS(4, 0, 0);
  else if (TYv == 5) IMS(5, 0, 0);
  else IMS(6, 0, 0);
#undef IMS
}

}  // namespace sdmkb
