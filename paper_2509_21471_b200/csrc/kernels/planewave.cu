// Plane-wave stage of the downward pass (K5-K8) and the root far field (K10):
// dmk.cpp:166-243 (forward / inverse separable DFT), 339-383 (phased
// colleague accumulation), 387-469 (kernel symbol), 671-701 and 705-833.
//
// B200 restructuring (same sums, different order):
//  * Hermitian half spectrum.  Proxy data are real, so G(-m) = conj G(m) and
//    every symbol keeps F Hermitian; only modes with m0 >= 0 are formed and
//    the inverse weights m0 > 0 by 2 (the reference forms all N^3 modes and
//    keeps Re of the full sum).
//  * Band compression.  Only modes inside the prolate band are produced
//    (the reference transforms the full cube and zeroes outside the band).
//    xy-columns (my, m0) are ordered by their z half-length lz, so the
//    in-band columns of every z-slab form a prefix: mode (mz, c) lives at
//    slab_off[mz] + c and each slab is a contiguous, coalesced run.
//  * One forward transform per (box, channel) (the reference recomputes a
//    colleague's transform once per sibling group, 5-7x per box).
//  * Phases are cube roots of unity: sum_e w^{r(m,tau_e)} G_e is formed as
//    S0 + w S1 + w^2 S2 with complex adds only.
// Stages: fwd_xy (x then y, per z-slab, in shared memory) -> fwd_z (thread
// per column) -> acc_sym (per target box, mode-chunked so colleague G stay
// L2-resident) -> inv_z -> inv_xy (adds pf * Re into the incoming proxies).
#include "common.cuh"
#include "launch.hpp"

#include <algorithm>
#include <cstdlib>

namespace sdmkb {

namespace {

constexpr int kPWBlock = 256;
constexpr int kModeChunk = 2048;
constexpr int kMaxEntries = 64;

// ---------------------------------------------------------------- forward --
__global__ void __launch_bounds__(kPWBlock) k_fwd_xy(PWGrid g, const int* __restrict__ boxes, int nch,
                                                     const double* __restrict__ outgoing, double2* __restrict__ B) {
  extern __shared__ double2 smc[];
  const int p = g.p, N = g.N, M = g.M, M1 = g.M + 1, pp = p * p, ncol = g.ncol;
  double2* EsT = smc;              // [p][N]: EsT[i][m+M] = E[m][i]
  double2* as = EsT + p * N;       // [p][M+1]
  double* ws = reinterpret_cast<double*>(as + p * M1);  // [p][p]
  const int tid = threadIdx.x;
  for (int e = tid; e < N * p; e += blockDim.x) {
    int m = e / p, i = e % p;
    EsT[i * N + m] = g.E[e];
  }
  const int slot = blockIdx.x, ch = blockIdx.y;
  const int b = boxes[slot];
  const double* w = outgoing + ((size_t)b * nch + ch) * (size_t)(g.pz * pp);
  double2* Bo = B + ((size_t)slot * nch + ch) * (size_t)g.pz * ncol;
  for (int iz = 0; iz < g.pz; ++iz) {
    __syncthreads();
    for (int e = tid; e < pp; e += blockDim.x) ws[e] = w[(size_t)iz * pp + e];
    __syncthreads();
    for (int e = tid; e < p * M1; e += blockDim.x) {  // x: a[iy][m0] = sum_ix E[m0][ix] w[iy][ix]
      int iy = e / M1, m0 = e % M1;
      const double* wr = ws + iy * p;
      double2 acc = make_double2(0.0, 0.0);
      for (int ix = 0; ix < p; ++ix) {
        double2 ev = EsT[ix * N + m0 + M];
        acc.x = fma(ev.x, wr[ix], acc.x);
        acc.y = fma(ev.y, wr[ix], acc.y);
      }
      as[e] = acc;
    }
    __syncthreads();
    for (int c = tid; c < ncol; c += blockDim.x) {  // y: b[c] = sum_iy E[my][iy] a[iy][m0]
      int my = g.col_my[c] + M, m0 = g.col_m0[c];
      double2 acc = make_double2(0.0, 0.0);
      for (int iy = 0; iy < p; ++iy) dev::cfma(acc, EsT[iy * N + my], as[iy * M1 + m0]);
      Bo[(size_t)iz * ncol + c] = acc;
    }
  }
}

template <int PZM>
__global__ void __launch_bounds__(kPWBlock) k_fwd_z(PWGrid g, int nch, const double2* __restrict__ B,
                                                    double2* __restrict__ G) {
  extern __shared__ double2 Ez[];  // [Nz][pz]
  const int pz = g.pz, Nz = g.Nz, Mz = g.Mz, ncol = g.ncol;
  const int tid = threadIdx.x;
  for (int e = tid; e < Nz * pz; e += blockDim.x) Ez[e] = g.Ez[e];  // [mz][iz]
  __syncthreads();
  const int slot = blockIdx.x, ch = blockIdx.y;
  const double2* Bi = B + ((size_t)slot * nch + ch) * (size_t)pz * ncol;
  double2* Go = G + ((size_t)slot * nch + ch) * (size_t)g.nhalf;
  const int lane = tid & 31;
  for (int c0 = (tid & ~31); c0 < ncol; c0 += blockDim.x) {
    const int c = c0 + lane;
    const bool act = c < ncol;
    double2 bv[PZM];
#pragma unroll
    for (int iz = 0; iz < PZM; ++iz) bv[iz] = (act && iz < pz) ? Bi[(size_t)iz * ncol + c] : make_double2(0.0, 0.0);
    const int lz = act ? g.col_lz[c] : -1;
    const int L = g.col_lz[c0];  // columns sorted by lz descending: lane 0 has the warp max
    for (int mz = -L; mz <= L; ++mz) {
      const double2* er = Ez + (mz + Mz) * pz;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int iz = 0; iz < PZM; ++iz)
        if (iz < pz) dev::cfma(acc, er[iz], bv[iz]);
      if (mz >= -lz && mz <= lz) Go[g.slab_off[mz + Mz] + c] = acc;
    }
  }
}

// ------------------------------------------------- accumulate + symbol --
// Kernel symbol applied to the phased colleague sum Ph (dmk.cpp:387-469):
// out[j] = F_j(k) for k = h m; A[|m|^2] is the level's radial symbol table.
template <int KERNEL, int DIM, int NCH>
__device__ __forceinline__ void apply_symbol(const double2 (&Ph)[NCH], int m0, int my, int mz,
                                             const double* __restrict__ A, double h, double2 (&out)[DIM]) {
#pragma unroll
  for (int j = 0; j < DIM; ++j) out[j] = make_double2(0.0, 0.0);
  const int s2 = m0 * m0 + my * my + mz * mz;
  const double av = A[s2];
  const double k0 = h * m0, k1 = h * my, k2 = DIM == 3 ? h * mz : 0.0;
  const double kk = k0 * k0 + k1 * k1 + k2 * k2;
  if (av != 0.0) {
    if (KERNEL == 0) {  // Stokeslet: A (k^2 f - k (k.f))
      double2 kf;
      kf.x = k0 * Ph[0].x + k1 * Ph[1].x + (DIM == 3 ? k2 * Ph[DIM - 1].x : 0.0);
      kf.y = k0 * Ph[0].y + k1 * Ph[1].y + (DIM == 3 ? k2 * Ph[DIM - 1].y : 0.0);
      const double kv[3] = {k0, k1, k2};
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        out[j].x = av * (kk * Ph[j].x - kv[j] * kf.x);
        out[j].y = av * (kk * Ph[j].y - kv[j] * kf.y);
      }
    } else if (KERNEL == 1) {  // stresslet: i A (k^2 Sk - k (kSk) + k tr(S) k^2 / (d+2))
      const double kv[3] = {k0, k1, k2};
      double2 Sk[3], kSk, wtr;
      if (DIM == 3) {
        const double2 S00 = Ph[0], S11 = Ph[1], S22 = Ph[2], S01 = Ph[3], S02 = Ph[4], S12 = Ph[5];
        Sk[0] = make_double2(S00.x * k0 + S01.x * k1 + S02.x * k2, S00.y * k0 + S01.y * k1 + S02.y * k2);
        Sk[1] = make_double2(S01.x * k0 + S11.x * k1 + S12.x * k2, S01.y * k0 + S11.y * k1 + S12.y * k2);
        Sk[2] = make_double2(S02.x * k0 + S12.x * k1 + S22.x * k2, S02.y * k0 + S12.y * k1 + S22.y * k2);
        kSk = make_double2(k0 * Sk[0].x + k1 * Sk[1].x + k2 * Sk[2].x, k0 * Sk[0].y + k1 * Sk[1].y + k2 * Sk[2].y);
        const double q = kk / 5.0;
        wtr = make_double2((S00.x + S11.x + S22.x) * q, (S00.y + S11.y + S22.y) * q);
      } else {
        const double2 S00 = Ph[0], S11 = Ph[1], S01 = Ph[2];
        Sk[0] = make_double2(S00.x * k0 + S01.x * k1, S00.y * k0 + S01.y * k1);
        Sk[1] = make_double2(S01.x * k0 + S11.x * k1, S01.y * k0 + S11.y * k1);
        Sk[2] = make_double2(0.0, 0.0);
        kSk = make_double2(k0 * Sk[0].x + k1 * Sk[1].x, k0 * Sk[0].y + k1 * Sk[1].y);
        const double q = kk / 4.0;
        wtr = make_double2((S00.x + S11.x) * q, (S00.y + S11.y) * q);
      }
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        double2 v = make_double2(av * (kk * Sk[j].x - kv[j] * kSk.x + kv[j] * wtr.x),
                                 av * (kk * Sk[j].y - kv[j] * kSk.y + kv[j] * wtr.y));
        out[j] = make_double2(-v.y, v.x);  // times i
      }
    } else {  // rotlet: -(i/2) A (g x k)
      const double ha = -0.5 * av;
      if (DIM == 3) {
        const double2 g0 = Ph[0], g1 = Ph[1], g2 = Ph[2];
        double2 c0 = make_double2(g1.x * k2 - g2.x * k1, g1.y * k2 - g2.y * k1);
        double2 c1 = make_double2(g2.x * k0 - g0.x * k2, g2.y * k0 - g0.y * k2);
        double2 c2 = make_double2(g0.x * k1 - g1.x * k0, g0.y * k1 - g1.y * k0);
        out[0] = make_double2(-ha * c0.y, ha * c0.x);
        out[1] = make_double2(-ha * c1.y, ha * c1.x);
        out[DIM - 1] = make_double2(-ha * c2.y, ha * c2.x);
      } else {
        const double2 g0 = Ph[0];
        double2 a = make_double2(k1 * g0.x, k1 * g0.y);
        double2 b = make_double2(k0 * g0.x, k0 * g0.y);
        out[0] = make_double2(-ha * a.y, ha * a.x);
        out[1] = make_double2(ha * b.y, -ha * b.x);
      }
    }
  }
}

template <int KERNEL, int DIM>
__global__ void __launch_bounds__(kPWBlock) k_acc_sym(PWGrid g, const int* __restrict__ ent_start,
                                                      const int* __restrict__ ent_slot,
                                                      const int* __restrict__ ent_tau,
                                                      const double2* __restrict__ G, int nch,
                                                      const double* __restrict__ A, double h,
                                                      double2* __restrict__ F) {
  __shared__ int s_slot[kMaxEntries], s_t0[kMaxEntries], s_t1[kMaxEntries], s_t2[kMaxEntries];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int e0 = ent_start[t], ne = ent_start[t + 1] - e0;
  for (int e = tid; e < ne; e += blockDim.x) {
    int code = ent_tau[e0 + e];
    s_slot[e] = ent_slot[e0 + e];
    s_t0[e] = code % 3 - 1;
    s_t1[e] = (code / 3) % 3 - 1;
    s_t2[e] = code / 9 - 1;
  }
  __syncthreads();
  constexpr int NCH = KERNEL == 0 ? DIM : (KERNEL == 1 ? (DIM == 3 ? 6 : 3) : (DIM == 3 ? 3 : 1));
  const int nhalf = g.nhalf;
  const int m_begin = blockIdx.y * kModeChunk, m_end = min(nhalf, m_begin + kModeChunk);
  const double w1r = -0.5, w1i = -0.8660254037844386467637232;  // exp(-2 pi i / 3)
  double2* Fo = F + (size_t)t * DIM * nhalf;
  for (int idx = m_begin + tid; idx < m_end; idx += blockDim.x) {
    const int code = g.mode_code[idx];
    const int c = code & 0xffff, mz = (code >> 16) - g.Mz;
    const int m0 = g.col_m0[c], my = g.col_my[c];
    double2 S0[NCH], S1[NCH], S2[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) S0[k] = S1[k] = S2[k] = make_double2(0.0, 0.0);
    for (int e = 0; e < ne; ++e) {
      int r = (m0 * s_t0[e] + my * s_t1[e] + mz * s_t2[e]) % 3;
      r = r < 0 ? r + 3 : r;
      const double2* ge = G + (size_t)s_slot[e] * nch * nhalf + idx;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        double2 v = ge[(size_t)k * nhalf];
        if (r == 0) { S0[k].x += v.x; S0[k].y += v.y; }
        else if (r == 1) { S1[k].x += v.x; S1[k].y += v.y; }
        else { S2[k].x += v.x; S2[k].y += v.y; }
      }
    }
    // Phi = S0 + w S1 + conj(w) S2
    double2 Ph[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      Ph[k].x = S0[k].x + w1r * (S1[k].x + S2[k].x) - w1i * (S1[k].y - S2[k].y);
      Ph[k].y = S0[k].y + w1r * (S1[k].y + S2[k].y) + w1i * (S1[k].x - S2[k].x);
    }
    double2 out[DIM];
    apply_symbol<KERNEL, DIM, NCH>(Ph, m0, my, mz, A, h, out);
#pragma unroll
    for (int j = 0; j < DIM; ++j) Fo[(size_t)j * nhalf + idx] = out[j];
  }
}

// Sibling-group accumulation: the same sums as k_acc_sym, grouped so that
// each colleague transform is read once per parent instead of once per
// target.  The 2^d children of one parent only see colleagues inside the
// parent's 4^d neighbourhood, positions pos in {-1..2}^d relative to the
// parent's anchor; child c sees the boxes at pos in c + {-1,0,1}^d, with
// phase w^{m.(pos - c)} = w^{-m.c} w^{m.pos}.  So every colleague is phased
// once per group, H(pos) = w^{m.pos} G(pos); the 3^d window sums of H are
// formed separably (two windows per axis sharing one pair sum); child c
// takes w^{-m.c} window_c, without its own H when it is a leaf (the
// reference skips a leaf's self entry, dmk.cpp:775).  The host verifies
// that the windows reproduce each target's reference entry list
// (dmk.cpp:760-797) and keeps levels where they would not (the periodic top
// levels) on k_acc_sym.
//
// Data movement: one CTA streams a group through mode chunks of kGM modes;
// each neighbourhood row (yi, zi) of a chunk is 4 positions x NCH channels
// of contiguous kGM-mode segments, fetched by the TMA engine (1D bulk
// copies, mbarrier byte count) into a kGS-stage shared ring, so the loads of
// the next rows are in flight while this row is summed (thread per mode).
constexpr int kGroupPos = 64;
constexpr int kGM = 128;  // modes per chunk = threads per CTA

__device__ __forceinline__ double2 phase3(int r, double2 v) {  // w^r v, w = exp(-2 pi i / 3)
  const double ci = r == 0 ? 0.0 : (r == 1 ? -0.8660254037844386467637232 : 0.8660254037844386467637232);
  const double cr = r == 0 ? 1.0 : -0.5;
  return make_double2(cr * v.x - ci * v.y, cr * v.y + ci * v.x);
}

// Shape per (kernel, dim, passes): ring stages and resident CTAs per SM,
// sized so registers (one pass keeps 8 or 4 windows x channels live) and
// the shared ring both fit; the stage count divides the rows per chunk so
// every row's stage is a compile-time constant.
template <int KERNEL, int DIM, int ZH>
struct GroupCfg {
  static constexpr int kNch = KERNEL == 0 ? DIM : (KERNEL == 1 ? (DIM == 3 ? 6 : 3) : (DIM == 3 ? 3 : 1));
  static constexpr int kRowBytes = 4 * kNch * kGM * 16;
  static constexpr int kRows = ZH * 4 * (DIM == 3 ? (ZH == 1 ? 4 : 3) : 1);  // rows per chunk
  static constexpr int kMinBlocks = (DIM == 3 && ZH == 1) || kNch > 3 ? 2 : 3;
  static constexpr int kZeroBytes = kNch * kGM * 16;  // stands in for absent positions
  static constexpr int kMaxStages = (227 * 1024 / kMinBlocks - 4096 - kZeroBytes) / kRowBytes;
  static constexpr int stages(int n) { return n <= 1 ? 1 : (kRows % n == 0 ? n : stages(n - 1)); }
  static constexpr int kStages = stages(kMaxStages);
  static constexpr int kBytes = kStages * kRowBytes;
};
constexpr int kGroupThreads = kGM + 32;  // 4 consumer warps + 1 TMA producer warp

template <int KERNEL, int DIM, int ZH>
__global__ void __launch_bounds__(kGroupThreads, GroupCfg<KERNEL, DIM, ZH>::kMinBlocks)
    k_acc_group(PWGrid g, const int* __restrict__ grp_tstart, const int* __restrict__ grp_slot,
                const int* __restrict__ t_meta, int t_base, const double2* __restrict__ G,
                const double* __restrict__ A, double h, double2* __restrict__ F) {
  using Cfg = GroupCfg<KERNEL, DIM, ZH>;
  constexpr int NCH = Cfg::kNch;
  constexpr int NCZ = DIM == 3 ? 2 : 1;  // z windows (children along z)
  constexpr int CZP = NCZ / ZH;          // z windows per pass
  constexpr int NW = 4 * CZP;            // windows per pass
  constexpr int NL = DIM == 3 ? (ZH == 1 ? 4 : 3) : 1;  // z layers per pass
  constexpr int RP = 4 * NL;                             // rows per pass
  constexpr int RC = Cfg::kRows;                         // rows per chunk
  constexpr int NS = Cfg::kStages;
  static_assert(NS >= 2 && RC % NS == 0, "ring shape");
  constexpr double kS3 = 0.8660254037844386467637232;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* ring = reinterpret_cast<double2*>(smraw);  // [NS][4][NCH][kGM]
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ int s_slot[kGroupPos];
  __shared__ int s_tgt[8];  // child code -> target index in the group | leaf << 8, or -1
  __shared__ __align__(16) double2 zero[NCH * kGM];
  const int grp = blockIdx.x, tid = threadIdx.x;
  const int ta = grp_tstart[grp], nt = grp_tstart[grp + 1] - ta;
  if (tid < kGroupPos) s_slot[tid] = grp_slot[(size_t)grp * kGroupPos + tid];
  if (tid < 8) s_tgt[tid] = -1;
  for (int e = tid; e < NCH * kGM; e += kGroupThreads) zero[e] = make_double2(0.0, 0.0);
  if (tid < NS) {
    dev::mbar_init(&full[tid], 1);
    dev::mbar_init(&empty[tid], kGM / 32);
  }
  if (tid == 0) dev::mbar_fence_init();
  __syncthreads();
  if (tid < nt) {
    const int meta = t_meta[ta + tid];
    s_tgt[meta & 7] = tid | ((meta & 8) << 5);
  }
  __syncthreads();
  const int nhalf = g.nhalf;
  const size_t bstride = (size_t)NCH * nhalf;
  const int nchunk = (nhalf + kGM - 1) / kGM;
  const int my_chunks = (nchunk - (int)blockIdx.y + (int)gridDim.y - 1) / (int)gridDim.y;
  if (tid >= kGM) {  // producer warp: refill each stage once the 4 consumer warps released it;
                     // lane l < 4 NCH issues the bulk copy of (position l / NCH, channel l % NCH),
                     // so the row's copies are issued in parallel
    const int lane = tid - kGM;
    const int xl = lane / NCH, kl = lane % NCH;
    const int nrows = my_chunks * RC;
    for (int i = 0; i < nrows; ++i) {
      if (i >= NS) dev::mbar_wait(&empty[i % NS], (uint32_t)((i / NS - 1) & 1));
      const int ck = (int)blockIdx.y + (i / RC) * (int)gridDim.y, r = i % RC;
      const int zh = r / RP, rr = r % RP;
      const int yi = rr & 3, zi = DIM == 3 ? zh + (rr >> 2) : 1;
      const int m_begin = ck * kGM, nm = min(kGM, nhalf - m_begin);
      const uint32_t seg = (uint32_t)nm * 16u;
      const int* srow = s_slot + 4 * yi + 16 * zi;
      uint64_t* bar = &full[i % NS];
      if (lane == 0) {
        uint32_t tx = 0;
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) tx += srow[xi] >= 0 ? NCH * seg : 0u;
        dev::mbar_expect_tx(bar, tx);
      }
      __syncwarp();  // the byte count is registered before any copy can complete
      double2* st = ring + (size_t)(i % NS) * 4 * NCH * kGM;
      if (lane < 4 * NCH) {
        const int sl = srow[xl];
        if (sl >= 0)
          dev::bulk_g2s(st + (xl * NCH + kl) * kGM, G + (size_t)sl * bstride + (size_t)kl * nhalf + m_begin, seg,
                        bar);
      }
    }
    return;
  }
  for (int it = 0; it < my_chunks; ++it) {
    const int ck = (int)blockIdx.y + it * (int)gridDim.y;
    const int idx = ck * kGM + tid;
    const bool act = idx < nhalf;
    int m0 = 0, my = 0, mz = 0;
    if (act) {
      const int code = g.mode_code[idx];
      const int c = code & 0xffff;
      mz = (code >> 16) - g.Mz;
      m0 = g.col_m0[c];
      my = g.col_my[c];
    }
    const int a0 = ((m0 % 3) + 3) % 3, a1 = ((my % 3) + 3) % 3, a2 = ((mz % 3) + 3) % 3;
    // x phases w^{m0 (xi - 1)} as coefficients (xi = 1 is 1); y/z phases per row
    const double pxr = a0 == 0 ? 1.0 : -0.5;
    const double pxi = a0 == 0 ? 0.0 : (a0 == 1 ? -kS3 : kS3);  // w^{a0}
    const double2 px2 = make_double2(pxr, pxi), px0 = make_double2(pxr, -pxi);  // w^{m0}, w^{-m0}
    const double2 px3 = make_double2(pxr * pxr - pxi * pxi, 2.0 * pxr * pxi);   // w^{2 m0}
    const int ry[4] = {(3 - a1) % 3, 0, a1, (2 * a1) % 3};
    const int rz[4] = {(3 - a2) % 3, 0, a2, (2 * a2) % 3};
#pragma unroll
    for (int zh = 0; zh < ZH; ++zh) {
      double2 W[NW][NCH];
#pragma unroll
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int k = 0; k < NCH; ++k) W[w][k] = make_double2(0.0, 0.0);
#pragma unroll
      for (int rr = 0; rr < RP; ++rr) {
        const int r = zh * RP + rr;
        const int yi = rr & 3, zi = DIM == 3 ? zh + (rr >> 2) : 1;
        const int stage = r % NS;
        dev::mbar_wait(&full[stage], (uint32_t)((it * (RC / NS) + r / NS) & 1));
        const double2* st = ring + (size_t)stage * 4 * NCH * kGM + tid;
        const double2* q[4];
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) q[xi] = s_slot[xi + 4 * yi + 16 * zi] >= 0 ? st + xi * NCH * kGM : zero + tid;
        int ryz = ry[yi] + (DIM == 3 ? rz[zi] : 0);
        ryz = ryz >= 3 ? ryz - 3 : ryz;
        const double rr_ = ryz == 0 ? 1.0 : -0.5;
        const double ri_ = ryz == 0 ? 0.0 : (ryz == 1 ? -kS3 : kS3);
        const double2 prow = make_double2(rr_, ri_);
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const double2 v0 = dev::cmul(px0, q[0][k * kGM]);
          const double2 v1 = q[1][k * kGM];
          const double2 v2 = dev::cmul(px2, q[2][k * kGM]);
          const double2 v3 = dev::cmul(px3, q[3][k * kGM]);
          const double2 mid = make_double2(v1.x + v2.x, v1.y + v2.y);
          const double2 X[2] = {dev::cmul(prow, make_double2(v0.x + mid.x, v0.y + mid.y)),
                                dev::cmul(prow, make_double2(mid.x + v3.x, mid.y + v3.y))};
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const int cx = w & 1, cy = (w >> 1) & 1, czg = DIM == 3 ? zh + (w >> 2) : 0;
            const bool in = yi >= cy && yi <= cy + 2 && (DIM == 2 || (zi >= czg && zi <= czg + 2));
            if (!in) continue;
            W[w][k].x += X[cx].x;
            W[w][k].y += X[cx].y;
            if (yi == cy + 1 && (DIM == 2 || zi == czg + 1)) {  // the window's own position
              const int tg = s_tgt[cx + 2 * cy + 4 * czg];
              if (tg >= 0 && (tg >> 8)) {  // a leaf child leaves its own H out
                const double2 sv = dev::cmul(prow, cx ? v2 : v1);
                W[w][k].x -= sv.x;
                W[w][k].y -= sv.y;
              }
            }
          }
        }
        __syncwarp();
        if ((tid & 31) == 0) dev::mbar_arrive(&empty[stage]);  // stage consumed by this warp
      }
      if (act) {  // pass complete: phase, symbol, store
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int cx = w & 1, cy = (w >> 1) & 1, cz = DIM == 3 ? zh + (w >> 2) : 0;
          const int tg = s_tgt[cx + 2 * cy + 4 * cz];
          if (tg < 0) continue;
          int rv = (a0 * cx + a1 * cy + a2 * cz) % 3;  // w^{-m.c}
          rv = rv == 0 ? 0 : 3 - rv;
          double2 Ph[NCH];
#pragma unroll
          for (int k = 0; k < NCH; ++k) Ph[k] = phase3(rv, W[w][k]);
          double2 out[DIM];
          apply_symbol<KERNEL, DIM, NCH>(Ph, m0, my, mz, A, h, out);
          double2* Fo = F + (size_t)(ta + (tg & 0xff) - t_base) * DIM * nhalf + idx;
#pragma unroll
          for (int j = 0; j < DIM; ++j) Fo[(size_t)j * nhalf] = out[j];
        }
      }
    }
  }
}

// ---------------------------------------------------------------- inverse --
template <int PZM>
__global__ void __launch_bounds__(kPWBlock) k_inv_z(PWGrid g, int d, const double2* __restrict__ F,
                                                    double2* __restrict__ C) {
  extern __shared__ double2 Ez[];  // [Nz][pz]
  const int pz = g.pz, Nz = g.Nz, Mz = g.Mz, ncol = g.ncol;
  const int tid = threadIdx.x;
  for (int e = tid; e < Nz * pz; e += blockDim.x) Ez[e] = g.Ez[e];
  __syncthreads();
  const int t = blockIdx.x, j = blockIdx.y;
  const double2* Fi = F + ((size_t)t * d + j) * (size_t)g.nhalf;
  double2* Co = C + ((size_t)t * d + j) * (size_t)pz * ncol;
  const int lane = tid & 31;
  for (int c0 = (tid & ~31); c0 < ncol; c0 += blockDim.x) {
    const int c = c0 + lane;
    const bool act = c < ncol;
    const int lz = act ? g.col_lz[c] : -1;
    const int L = g.col_lz[c0];
    double2 acc[PZM];
#pragma unroll
    for (int iz = 0; iz < PZM; ++iz) acc[iz] = make_double2(0.0, 0.0);
    for (int mz = -L; mz <= L; ++mz) {
      if (mz < -lz || mz > lz) continue;
      const double2 fv = Fi[g.slab_off[mz + Mz] + c];
      const double2* er = Ez + (mz + Mz) * pz;
#pragma unroll
      for (int iz = 0; iz < PZM; ++iz)
        if (iz < pz) dev::cfma_conj(acc[iz], er[iz], fv);
    }
    if (act) {
#pragma unroll
      for (int iz = 0; iz < PZM; ++iz)
        if (iz < pz) Co[(size_t)iz * ncol + c] = acc[iz];
    }
  }
}

// stage = 0: the row of C is read in place (global memory) instead of from a
// shared copy -- the same sums in the same order; used when E, the row and
// the y-stage result together pass the 227 KB of shared memory (p = 60, N1 = 107)
__global__ void __launch_bounds__(kPWBlock) k_inv_xy(PWGrid g, const int* __restrict__ tboxes, int d,
                                                     const double2* __restrict__ C, double pf,
                                                     double* __restrict__ incoming, int stage) {
  extern __shared__ double2 smc[];
  const int p = g.p, N = g.N, M = g.M, M1 = g.M + 1, pp = p * p, ncol = g.ncol;
  double2* EsT = smc;         // [p][N]
  double2* csm = EsT + p * N;                // [ncol] (stage)
  double2* ds = csm + (stage ? ncol : 0);    // [p][M+1]
  const int tid = threadIdx.x;
  for (int e = tid; e < N * p; e += blockDim.x) {
    int m = e / p, i = e % p;
    EsT[i * N + m] = g.E[e];
  }
  const int t = blockIdx.x, j = blockIdx.y;
  const int b = tboxes[t];
  const double2* Ci = C + ((size_t)t * d + j) * (size_t)g.pz * ncol;
  double* out = incoming + ((size_t)b * d + j) * (size_t)(g.pz * pp);
  for (int iz = 0; iz < g.pz; ++iz) {
    __syncthreads();
    const double2* cs = Ci + (size_t)iz * ncol;
    if (stage) {
      for (int c = tid; c < ncol; c += blockDim.x) csm[c] = cs[c];
      cs = csm;
      __syncthreads();
    }
    for (int e = tid; e < p * M1; e += blockDim.x) {  // y: d[iy][m0] = sum_my conj(E[my][iy]) c[(my,m0)]
      int iy = e / M1, m0 = e % M1;
      double2 acc = make_double2(0.0, 0.0);
      for (int k = g.m0_start[m0]; k < g.m0_start[m0 + 1]; ++k) {
        int c = g.m0_cols[k];
        dev::cfma_conj(acc, EsT[iy * N + g.col_my[c] + M], cs[c]);
      }
      ds[e] = acc;
    }
    __syncthreads();
    for (int e = tid; e < pp; e += blockDim.x) {  // x: out += pf Re(sum_m0 wt conj(E[m0][ix]) d[iy][m0])
      int iy = e / p, ix = e % p;
      const double2* dr = ds + iy * M1;
      const double2 e0 = EsT[ix * N + M];
      double s0 = e0.x * dr[0].x + e0.y * dr[0].y;
      double s = 0.0;
      for (int m0 = 1; m0 <= M; ++m0) {
        double2 ev = EsT[ix * N + m0 + M];
        s = fma(ev.x, dr[m0].x, s);
        s = fma(ev.y, dr[m0].y, s);
      }
      out[(size_t)iz * pp + e] += pf * (s0 + 2.0 * s);
    }
  }
}

void set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

void launch_forward(const PWGrid& g, const int* boxes, int nbox, int nch, const double* outgoing, double2* B,
                    double2* G, cudaStream_t st) {
  if (nbox <= 0) return;
  dim3 grid(nbox, nch);
  size_t smem = sizeof(double2) * (g.p * g.N + g.p * (g.M + 1)) + sizeof(double) * g.p * g.p;
  set_smem((const void*)k_fwd_xy, smem);
  k_fwd_xy<<<grid, kPWBlock, smem, st>>>(g, boxes, nch, outgoing, B);
  size_t zs = sizeof(double2) * g.Nz * g.pz;
  set_smem((const void*)k_fwd_z<64>, zs);  // only pz > 32 can pass 48 KB
  if (g.pz <= 1) k_fwd_z<1><<<grid, kPWBlock, zs, st>>>(g, nch, B, G);
  else if (g.pz <= 16) k_fwd_z<16><<<grid, kPWBlock, zs, st>>>(g, nch, B, G);
  else if (g.pz <= 24) k_fwd_z<24><<<grid, kPWBlock, zs, st>>>(g, nch, B, G);
  else if (g.pz <= 32) k_fwd_z<32><<<grid, kPWBlock, zs, st>>>(g, nch, B, G);
  else k_fwd_z<64><<<grid, kPWBlock, zs, st>>>(g, nch, B, G);
}

void launch_accumulate_symbol(const PWGrid& g, int kernel, int ntb, const int* ent_start,
                                   const int* ent_slot, const int* ent_tau, const double2* G, int nch,
                                   const double* A, double h, double2* F, cudaStream_t st) {
  if (ntb <= 0) return;
  dim3 grid(ntb, (g.nhalf + kModeChunk - 1) / kModeChunk);
#define ACC(K, D) k_acc_sym<K, D><<<grid, kPWBlock, 0, st>>>(g, ent_start, ent_slot, ent_tau, G, nch, A, h, F)
  if (g.dim == 3) {
    if (kernel == 0) ACC(0, 3);
    else if (kernel == 1) ACC(1, 3);
    else ACC(2, 3);
  } else {
    if (kernel == 0) ACC(0, 2);
    else if (kernel == 1) ACC(1, 2);
    else ACC(2, 2);
  }
#undef ACC
}

void launch_accumulate_group(const PWGrid& g, int kernel, int ngroups, const int* grp_tstart, const int* grp_slot,
                             const int* t_meta, int t_base, const double2* G, const double* A, double h,
                             double2* F, cudaStream_t st) {
  if (ngroups <= 0) return;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // enough CTAs for ~4 waves at 2 per SM; big levels stream whole groups
  const int nchunk = (g.nhalf + kGM - 1) / kGM;
  const int want = 8 * num_sms;
  const int gy = std::max(1, std::min(nchunk, (want + ngroups - 1) / ngroups));
  dim3 grid(ngroups, gy);
#define ACC(K, D, Z)                                                                                         \
  do {                                                                                                       \
    const int sm_ = GroupCfg<K, D, Z>::kBytes;                                                               \
    cudaFuncSetAttribute(k_acc_group<K, D, Z>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_);            \
    k_acc_group<K, D, Z><<<grid, kGroupThreads, sm_, st>>>(g, grp_tstart, grp_slot, t_meta, t_base, G, A, h, F); \
  } while (0)
  if (g.dim == 3) {
    if (kernel == 0) ACC(0, 3, 1);
    else if (kernel == 1) ACC(1, 3, 2);
    else ACC(2, 3, 1);
  } else {
    if (kernel == 0) ACC(0, 2, 1);
    else if (kernel == 1) ACC(1, 2, 1);
    else ACC(2, 2, 1);
  }
#undef ACC
}

void launch_inverse(const PWGrid& g, const int* tboxes, int ntb, int d, const double2* F, double2* C, double pf,
                    double* incoming, cudaStream_t st) {
  if (ntb <= 0) return;
  dim3 grid(ntb, d);
  size_t zs = sizeof(double2) * g.Nz * g.pz;
  set_smem((const void*)k_inv_z<64>, zs);  // only pz > 32 can pass 48 KB
  if (g.pz <= 1) k_inv_z<1><<<grid, kPWBlock, zs, st>>>(g, d, F, C);
  else if (g.pz <= 16) k_inv_z<16><<<grid, kPWBlock, zs, st>>>(g, d, F, C);
  else if (g.pz <= 24) k_inv_z<24><<<grid, kPWBlock, zs, st>>>(g, d, F, C);
  else if (g.pz <= 32) k_inv_z<32><<<grid, kPWBlock, zs, st>>>(g, d, F, C);
  else k_inv_z<64><<<grid, kPWBlock, zs, st>>>(g, d, F, C);
  size_t smem = sizeof(double2) * (g.p * g.N + g.ncol + g.p * (g.M + 1));
  const int stage = smem <= 227 * 1024;
  if (!stage) smem -= sizeof(double2) * g.ncol;
  set_smem((const void*)k_inv_xy, smem);
  k_inv_xy<<<grid, kPWBlock, smem, st>>>(g, tboxes, d, C, pf, incoming, stage);
}

}  // namespace sdmkb
