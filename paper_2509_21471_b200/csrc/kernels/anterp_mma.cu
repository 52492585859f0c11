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
__global__ void __launch_bounds__(256) k_basis(ChebDev cb, const DBox* __restrict__ boxes,
                                               const int* __restrict__ leaves, const double* __restrict__ pts, int n,
                                               int use_targets, double* __restrict__ basis) {
  __shared__ double nodes[64], wts[64];
  const int p = cb.p, dim = cb.dim;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    nodes[i] = cb.nodes[i];
    wts[i] = cb.wts[i];
  }
  __syncthreads();
  const DBox box = boxes[leaves[blockIdx.x]];
  const int b0 = use_targets ? box.tb : box.sb, b1 = use_targets ? box.te : box.se;
  const double hinv = 1.0 / box.half;
  const int cnt = b1 - b0;
  for (int task = threadIdx.x; task < cnt * dim; task += blockDim.x) {
    const int ax = task / cnt, i = b0 + task % cnt;
    const double x = __dmul_rn(__dsub_rn(pts[(size_t)ax * n + i], box.c[ax]), hinv);
    dev::cheb_basis(p, nodes, wts, x, basis + ((size_t)ax * n + i) * p, 1);
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

// ------------------------------------------------------------------- K11 --
constexpr int kTB = 128;     // targets per block (two m-tiles per warp)

// W chunks arrive by cp.async, double buffered; each warp keeps the A
// fragments of its two 8-target m-tiles in registers and runs their DMMA
// chains interleaved.
template <int KS, int kNC, int PC, int DC>  // kNC: W rows per shared chunk; PC/DC: compile-time p, dim
__global__ void __launch_bounds__(256, 1) k_interp_mma(ChebDev cb, const DBox* __restrict__ boxes,
                                                      const int* __restrict__ leaves,
                                                      const double* __restrict__ tbasis, int nt,
                                                      const int* __restrict__ tperm,
                                                      const double* __restrict__ incoming,
                                                      double* __restrict__ ufar) {
  extern __shared__ double sm[];
  constexpr int KP = KS * 4, WS = KP + 4;
  const int p = PC > 0 ? PC : cb.p, dim = DC > 0 ? DC : cb.dim, pz = dim == 3 ? p : 1;
  const int N = dim * pz * p, BS = p + 1;
  double* Ws = sm;                    // [2][kNC][WS]
  double* bxs = Ws + 2 * kNC * WS;    // [kTB][WS]
  double* bys = bxs + kTB * WS;       // [kTB][BS]
  double* bzs = bys + kTB * BS;       // [kTB][BS]
  int* ntab = reinterpret_cast<int*>(bzs + kTB * BS);  // [N]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int b = leaves[blockIdx.x];
  const DBox box = boxes[b];
  for (int e = tid; e < N; e += blockDim.x) {
    const int j = e / (pz * p), r = e % (pz * p);
    ntab[e] = (j << 16) | ((r / p) << 8) | (r % p);
  }
  for (int e = tid; e < 2 * kNC * WS; e += blockDim.x) Ws[e] = 0.0;  // k padding stays zero
  const double* W = incoming + (size_t)b * N * p;
  const double* bxg = tbasis;
  const double* byg = tbasis + (size_t)nt * p;
  const double* bzg = tbasis + (size_t)2 * nt * p;
  const int nchunk = (N + kNC - 1) / kNC;
  auto issue = [&](int c, int buf) {
    const int n0 = c * kNC, nc = min(kNC, N - n0);
    double* dstb = Ws + buf * kNC * WS;
    for (int e = tid; e < kNC * p; e += blockDim.x) {
      const int r = e / p, k = e % p;
      const bool v = r < nc;
      dev::cp_async8(dstb + r * WS + k, v ? W + (size_t)(n0 + r) * p + k : W, v);
    }
    dev::cp_commit();
  };
  for (int t0 = box.tb; t0 < box.te; t0 += kTB) {
    const int tc = min(kTB, box.te - t0);
    __syncthreads();
    issue(0, 0);
    for (int e = tid; e < kTB * KP; e += blockDim.x) {
      const int a = e / KP, k = e % KP;
      bxs[a * WS + k] = (a < tc && k < p) ? bxg[(size_t)(t0 + a) * p + k] : 0.0;
    }
    for (int e = tid; e < kTB * p; e += blockDim.x) {
      const int a = e / p, k = e % p;
      bys[a * BS + k] = a < tc ? byg[(size_t)(t0 + a) * p + k] : 0.0;
      bzs[a * BS + k] = a < tc ? (dim == 3 ? bzg[(size_t)(t0 + a) * p + k] : (k == 0 ? 1.0 : 0.0)) : 0.0;
    }
    __syncthreads();
    const int r0 = warp * 16 + g, r1 = r0 + 8;  // this lane's two targets (A / C rows)
    double a0[KS], a1[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      a0[ks] = bxs[r0 * WS + ks * 4 + t];
      a1[ks] = bxs[r1 * WS + ks * 4 + t];
    }
    double v[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    const bool active = warp * 16 < tc;
    for (int c = 0; c < nchunk; ++c) {
      const int buf = c & 1;
      if (c + 1 < nchunk) {
        issue(c + 1, buf ^ 1);
        dev::cp_wait1();
      } else {
        dev::cp_wait0();
      }
      __syncthreads();
      const double* Wc = Ws + buf * kNC * WS;
      const int n0 = c * kNC, nc = min(kNC, N - n0);
      if (active) {
        const int ntiles = (nc + 7) / 8;
        for (int nt_ = 0; nt_ < ntiles; ++nt_) {
          double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const double bv = Wc[(nt_ * 8 + g) * WS + ks * 4 + t];
            dev::dmma(c00, c01, a0[ks], bv);
            dev::dmma(c10, c11, a1[ks], bv);
          }
          const int na = n0 + nt_ * 8 + 2 * t;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = na + e;
            if (nn < N) {
              const int code = ntab[nn];
              const int j = code >> 16, iz = (code >> 8) & 255, iy = code & 255;
              const double w0 = bzs[r0 * BS + iz] * bys[r0 * BS + iy] * (e ? c01 : c00);
              const double w1 = bzs[r1 * BS + iz] * bys[r1 * BS + iy] * (e ? c11 : c10);
              v[0][j] += w0;
              v[1][j] += w1;
            }
          }
        }
      }
      __syncthreads();  // the next issue overwrites this buffer
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        v[h][j] += __shfl_xor_sync(0xffffffffu, v[h][j], 1);
        v[h][j] += __shfl_xor_sync(0xffffffffu, v[h][j], 2);
      }
    if (t == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = h ? r1 : r0;
        if (r < tc) {
          double* ut = ufar + (size_t)tperm[t0 + r] * dim;
          ut[0] = v[h][0];
          ut[1] = v[h][1];
          if (dim == 3) ut[2] = v[h][2];
        }
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
  k_basis<<<nleaf, 256, 0, st>>>(cb, boxes, leaves, pts, n, use_targets, basis);
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
  if (cb.dim == 3 && p == 23 && kernel == 0) AMS(3, 6, 23, 0, 3);
  else if (cb.dim == 3 && p == 22 && kernel == 1) AMS(3, 6, 22, 1, 3);
  else if (cb.dim == 3 && p == 30 && kernel == 0) AMS(4, 4, 30, 0, 3);
  else if (NTv <= 1) AM(1, 8);
  else if (NTv == 2) AM(2, 8);
  else if (NTv == 3) AM(3, 6);
  else if (NTv == 4) AM(4, 4);
  else if (NTv == 5) AM(5, 3);
  else AM(6, 3);
#undef AM
#undef AMS
}

void launch_interp_mma(const ChebDev& cb, const DBox* boxes, const int* leaves, int nleaf, const double* tbasis,
                       int nt, const int* tperm, const double* incoming, double* ufar, cudaStream_t st) {
  if (nleaf <= 0) return;
  const int p = cb.p, N = cb.dim * cb.pz * p;
  const int KSv = (p + 3) / 4;
  auto smem_for = [&](int KS, int NC) {
    const int WS = KS * 4 + 4;
    return sizeof(double) * (2 * (size_t)NC * WS + (size_t)kTB * WS + 2 * (size_t)kTB * (p + 1)) + sizeof(int) * N;
  };
#define IMS(KSS, NCC, PC_, DC_)                                                                           \
  do {                                                                                                    \
    size_t sm = smem_for(KSS, NCC);                                                                       \
    smem_attr((const void*)k_interp_mma<KSS, NCC, PC_, DC_>, sm);                                         \
    k_interp_mma<KSS, NCC, PC_, DC_><<<nleaf, 256, sm, st>>>(cb, boxes, leaves, tbasis, nt, tperm, incoming, \
                                                              ufar);                                      \
  } while (0)
#define IM(KSS, NCC) IMS(KSS, NCC, 0, 0)
  if (cb.dim == 3 && p == 23) IMS(6, 256, 23, 3);
  else if (cb.dim == 3 && p == 22) IMS(6, 256, 22, 3);
  else if (cb.dim == 3 && p == 30) IMS(8, 128, 30, 3);
  else if (KSv <= 2) IM(2, 256);
  else if (KSv <= 4) IM(4, 256);
  else if (KSv <= 6) IM(6, 256);
  else if (KSv <= 8) IM(8, 128);
  else IM(12, 64);
#undef IM
#undef IMS
}

}  // namespace sdmkb
