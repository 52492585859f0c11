// K12: near-field residual pass (dmk.cpp:919-1032) with the fused residual
// apply (split.cpp:258-317).
//
// Persistent kernel: one 16-warp CTA per SM; each warp takes 32-target
// chunks of one leaf from an atomic counter, one target per lane, so each
// target's pairs are summed by one lane in a fixed order (own box first, then
// the near ranges and their sources in the reference's order).
//  1. Intervals: the lanes build the chunk's source intervals in parallel, one
//     near range per lane (own box nu = r_l, colleague leaves and fine
//     neighbours nu = r_l/2, coarse neighbours nu = r_l; dmk.cpp:966-990):
//     the range box and then its Morton child sub-cells are culled against
//     the warp's target bounding box with a conservative margin (no pair with
//     r^2 < (nu*support)^2 is dropped); survivors in (range, sub-cell) order.
//  2. Own box (dense): rounds of 32 packed source records are staged in the
//     warp's list storage and broadcast to every lane; the exact test masks
//     out-of-support pairs.
//  3. Other intervals (lists): sources stream in coalesced rounds of 32 and
//     are broadcast by shuffles; each lane runs a conservative single-
//     precision pre-test and appends candidates to a short lane-private list
//     in shared memory, spilled to the lane's list in global scratch
//     (L2-resident) whenever one lane's fills up; the chunk's lists are
//     evaluated once at its end, in lockstep, two entries per step, with
//     the reference's exact double-precision support test (x = xt - (xs +
//     shift), unfused r2).  (Evaluating each shared list when it filled cost
//     2.6 lockstep slots per candidate: the lanes fill unevenly during the
//     scan, but per chunk their totals are similar.)
//  4. Radial tables: a piecewise degree-6 re-expansion of the reference's
//     Chebyshev tables in the local coordinate w = y - floor(y), scaled by
//     the kernel's constant factors, in shared memory (8 bank-interleaved
//     copies), within 2e-15 of them; pairs in the first interval (s < 1/128,
//     where the kernels' 1/r^2..1/r^5 factors amplify absolute table errors)
//     are re-evaluated after their round / list block with the reference's
//     own coefficients and Clenshaw recurrence, unfused.  1/r from rsqrt;
//     contributions enter by predicated FMAs; support and zero tests on the
//     bit patterns of r2 (integer pipe).
// No atomics on the data and a fixed per-target order: bitwise reproducible.
#include "common.cuh"
#include "launch.hpp"

#include <algorithm>
#include <type_traits>

namespace sdmkb {

namespace {

using dev::DBox;

// One 16-warp CTA per SM (persistent): the SM's single copy of the radial
// table can then hold 128 intervals at degree 6 -- 7 coefficient loads per
// pair, values within 1e-15 of the reference's Clenshaw tables.
constexpr int kRBlock = 512;
constexpr int kWarps = kRBlock / 32;
#ifndef SDMK_RES_LIST
#define SDMK_RES_LIST 40
#endif
constexpr int kList = SDMK_RES_LIST;  // per-lane list capacity (entries): longer lists, less lockstep padding
constexpr int kMaxRanges = 160;
constexpr int kMaxIvl = kMaxRanges * 8;  // source intervals per chunk: ranges x Morton sub-cells
constexpr int kResBlocksPerSM = 1;       // persistent grid (registers and shared memory: 1 per SM)
constexpr int kGCap = 1024;              // per-lane global candidate list (entries; even)
constexpr int kMaxPW = 896;      // ni * (deg + 1) <= 896 (d, o) coefficient pairs (8 copies: 112 KB)
constexpr int kCopies = 8;       // table copies, one per 16-byte bank group

// Packed source record (coordinates, then strengths), padded to an even
// number of doubles: the pair evaluation gathers one record with 16-byte loads
// instead of d + sc scattered 8-byte loads.
template <int KERNEL, int DIM>
struct Rec {
  static constexpr int kSc = KERNEL == 0 ? DIM : (KERNEL == 1 ? 2 * DIM : (DIM == 3 ? 3 : 1));
  static constexpr int kW = (DIM + kSc + 1) / 2 * 2;
};

__global__ void k_pack_sources(const double* __restrict__ spts, const double* __restrict__ sstr, int n, int dim,
                               int sc, int rw, double* __restrict__ rec) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double* r = rec + (size_t)i * rw;
    for (int k = 0; k < dim; ++k) r[k] = spts[(size_t)k * n + i];
    for (int k = 0; k < sc; ++k) r[dim + k] = sstr[(size_t)k * n + i];
    for (int k = dim + sc; k < rw; ++k) r[k] = 0.0;
  }
}

// 1/sqrt(x) from the hardware double-precision estimate (MUFU.RSQ64H, ~23
// good bits, no f32 round trip) and two Newton steps (~1 ulp; the CUDA
// double rsqrt spends ~20 instructions on range handling).  Branch-free:
// x = 0 or subnormal gives NaN, and the callers send a NaN s to the exact
// path (s < s_exact is tested as !(s >= s_exact)), which uses rsqrt.
// Newton in the form y + y (1/2 - (x/2) y y): the same roundings as
// y + (y/2)(1 - x y y), one multiply fewer.
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  double r = fma(-hx * y, y, 0.5);
  y = fma(y, r, y);
  r = fma(-hx * y, y, 0.5);
  return fma(y, r, y);
}

// list appends through 32-bit shared addresses (a generic pointer would
// carry 64-bit arithmetic into the scan loop)
__device__ __forceinline__ void sts_u32(unsigned a, int v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void sts_u8(unsigned a, int v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}

// u += c where p (one predicated DADD; a select would cost two more)
__device__ __forceinline__ void add_if(double& u, double c, bool p) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}"
      : "+d"(u)
      : "d"(c), "r"((unsigned)p));
}

// r2 < b for r2 >= 0, b > 0: the bit patterns of non-negative doubles order
// as unsigned integers (integer pipe instead of a DSETP on the FP64 pipe)
__device__ __forceinline__ bool lt_nonneg(double r2, double b) {
  return (unsigned long long)__double_as_longlong(r2) < (unsigned long long)__double_as_longlong(b);
}
__device__ __forceinline__ bool is_zero_nonneg(double r2) { return __double_as_longlong(r2) == 0; }

// u += a b where p (one predicated DFMA instead of zeroing a factor by selects)
__device__ __forceinline__ void fma_if(double& u, double a, double b, bool p) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q fma.rn.f64 %0, %1, %2, %0;\n\t}"
      : "+d"(u)
      : "d"(a), "d"(b), "r"((unsigned)p));
}

struct RangeS {
  double sh[3];
  double lo[3], hi[3];
  double nu, inu, sup2, cull, half;
  int sb, se, self, zero_shift;
  int code;  // packed image shift (x+1 | y+1 << 2 | z+1 << 4) | fine-scale flag << 6
};

// Radial table values at table coordinate y = (s - lo) ni / (hi - lo) from
// the piecewise monomial form held in shared memory as (diag, offdiag) pairs,
// one 16-byte load per degree: interval i = floor(y), local w = y - i in [0, 1),
// Horner at a compile-time degree (the host pads the table with leading zero
// coefficients, which leave Horner's value unchanged).  The host scales both
// tables by the kernel's constant factor (ResidTables::scale_d / scale_o), so
// the assembly multiplies by powers of 1/r only.  Returns false at/after the
// support (y >= ni: the reference's value there is 0, split.cpp:147-179).
// Returns floor(y) (0xffffffff for NaN y, the canonical NaN's low word):
// fl >= ni is past the support, fl + 1 <= 1 the first interval or NaN.
// The table is stored kCopies times interleaved, copy c in 16-byte bank group
// c: lane L reads copy L % 8, so the 8 lanes of a 128-bit load phase always
// hit 8 distinct bank groups whatever intervals they need (no conflicts).
// The reference's Clenshaw (chebyshev.cpp:9-19) in its own operation order,
// every product and sum rounded separately (the reference is built without
// FMA contraction).
__device__ __forceinline__ double clenshaw_ref1(const double* __restrict__ c, int n, double lo, double hi, double x) {
  if (n == 0) return 0.0;
  const double t = __ddiv_rn(__dsub_rn(__dsub_rn(__dmul_rn(2.0, x), lo), hi), __dsub_rn(hi, lo));
  const double t2 = __dmul_rn(2.0, t);
  double b1 = 0.0, b2 = 0.0;
  for (int k = n - 1; k >= 1; --k) {
    const double b0 = __dadd_rn(__dsub_rn(__dmul_rn(t2, b1), b2), c[k]);
    b2 = b1;
    b1 = b0;
  }
  return __dadd_rn(__dsub_rn(__dmul_rn(t, b1), b2), c[0]);
}

// EXACT: the reference's tables and recurrence (pairs with s < s_exact, rare;
// re-evaluated after the fast pass so the hot path keeps its registers),
// scaled as the piecewise tables are
template <int KERNEL, int DEG, bool EXACT>
__device__ __forceinline__ unsigned radial_tables(const ResidTables& rt, const double2* __restrict__ pw, double y,
                                              double& fd, double& fo, const double* __restrict__ cheb, double r2,
                                              double inu) {
  if (EXACT) {
    const double se = __dmul_rn(__dsqrt_rn(r2), inu);  // s = sqrt(r2) / nu as the reference forms it
    fd = KERNEL != 2 ? rt.scale_d * clenshaw_ref1(cheb, rt.n_d, rt.lo, rt.hi, se) : 0.0;
    fo = rt.scale_o * clenshaw_ref1(cheb + kResidMaxCheb, rt.n_o, rt.lo, rt.hi, se);
    return 1u;  // inside the table, not in the first interval
  }
  // interval = floor(y) without FP64 conversions: y + 2^52 rounded down holds
  // floor(y) in its low word (y in [0, 2^31); NaN only for coincident
  // points, which are never kept); past the last interval the pair is dropped
  // (the clamped evaluation below is finite and discarded)
  const double t = __dadd_rd(y, 0x1p52);
  const unsigned fl = (unsigned)__double2loint(t);
  const int iv = (int)min(fl, (unsigned)(rt.ni - 1));
  const double u = y - (t - 0x1p52);  // exact
  const double2* c = pw + iv * (DEG + 1) * kCopies;  // pw already offset by this lane's copy
  double2 v = c[DEG * kCopies];
#pragma unroll
  for (int k = DEG - 1; k >= 0; --k) {
    const double2 ck = c[k * kCopies];
    if (KERNEL != 2) v.x = fma(v.x, u, ck.x);
    v.y = fma(v.y, u, ck.y);
  }
  fd = KERNEL != 2 ? v.x : 0.0;
  fo = v.y;
  return fl;
}

// residual_apply assembly (split.cpp:258-317) given the radial table values
// (already scaled by the kernel constants, except the 2D Stokeslet's), added
// into u when keep by predicated FMAs; rinv = 1/r from rsqrt, so 1/r, 1/r^2,
// 1/r^3, 1/r^5 are products.
template <int KERNEL, int DIM>
__device__ __forceinline__ void assemble(double fd, double fo, const double* x, double rinv, double s,
                                         double support, double nu, const double* sv, double* u, bool keep) {
  constexpr double k8pi = 1.0 / (8.0 * dev::kPI);
  const double rinv2 = rinv * rinv;
  if (KERNEL == 0) {  // Stokeslet
    double f[DIM], xf = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      f[i] = sv[i];
      xf += x[i] * f[i];
    }
    double cd, cf;
    if (DIM == 2) {  // fd = -2 s log s - table (split.cpp:147-155); amp = nu; unscaled tables
      fd = s < support ? (s > 0.0 ? -2.0 * s * log(s) : 0.0) - fd : 0.0;
      const double c0 = k8pi * rinv;
      cd = nu * fd * c0;
      cf = nu * fo * c0 * xf * rinv2;
    } else {
      cd = fd * rinv;
      cf = (fo * rinv) * (xf * rinv2);
    }
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      fma_if(u[j], cf, x[j], keep);
      fma_if(u[j], cd, f[j], keep);
    }
  } else if (KERNEL == 1) {  // stresslet
    const double amp = DIM == 2 ? nu : 1.0;
    double f[DIM], nn[DIM], xf = 0.0, xn = 0.0, fn = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      f[i] = sv[i];
      nn[i] = sv[DIM + i];
      xf += x[i] * f[i];
      xn += x[i] * nn[i];
      fn += f[i] * nn[i];
    }
    const double rinv3 = rinv2 * rinv;
    const double cd = amp * fd * rinv3;
    const double co = amp * fo * xf * xn * rinv3 * rinv2;
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      fma_if(u[j], co, x[j], keep);
      fma_if(u[j], cd, f[j] * xn + x[j] * fn + nn[j] * xf, keep);
    }
  } else {  // rotlet
    double c[3];
    if (DIM == 2) {
      const double c0 = fo * sv[0] * rinv2;
      c[0] = c0 * x[1];
      c[1] = -(c0 * x[0]);
    } else {
      const double c0 = fo * rinv2 * rinv;
      const double g0 = sv[0], g1 = sv[1], g2 = sv[2];
      c[0] = c0 * (g1 * x[2] - g2 * x[1]);
      c[1] = c0 * (g2 * x[0] - g0 * x[2]);
      c[DIM - 1] = c0 * (g0 * x[1] - g1 * x[0]);
    }
#pragma unroll
    for (int j = 0; j < DIM; ++j) add_if(u[j], c[j], keep);
  }
}

template <int KERNEL, int DIM, int DEG, int PER>
__global__ void __launch_bounds__(kRBlock) k_residual(ResidTables rt, const DBox* __restrict__ boxes,
                                                      const int* __restrict__ leaves, const int2* __restrict__ chunks, int nchunks,
                                                      const int* __restrict__ rng_start,
                                                      const int* __restrict__ rng_box,
                                                      const int* __restrict__ rng_info,
                                                      const int* __restrict__ subrange,
                                                      const double* __restrict__ spts, int ns,
                                                      const double* __restrict__ sstr,
                                                      const double2* __restrict__ srec,
                                                      const double* __restrict__ tpts, int nt,
                                                      const int* __restrict__ tperm, int alias, double self_const,
                                                      double* __restrict__ ures, int* flags,
                                                      unsigned long long* stats, int4* __restrict__ ivl_all,
                                                      int* __restrict__ glist, unsigned char* __restrict__ glcode,
                                                      int* __restrict__ next_chunk) {
  extern __shared__ __align__(16) double2 dyn2[];  // [npw][kCopies] table, then the lists
  double2* s_pw = dyn2;
  const int npw = rt.ni * (rt.deg + 1);
  double* s_cheb = reinterpret_cast<double*>(dyn2 + npw * kCopies);  // [2][kResidMaxCheb] reference tables
  int* dyn = reinterpret_cast<int*>(s_cheb + 2 * kResidMaxCheb);  // lane-interleaved lists: [kWarps][kList][32] ints then bytes
  int (*lsrc)[kList][32] = reinterpret_cast<int (*)[kList][32]>(dyn);
  unsigned char (*lrng)[kList][32] = reinterpret_cast<unsigned char (*)[kList][32]>(dyn + kWarps * kList * 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < npw * kCopies; e += blockDim.x) {
    const int k = e / kCopies;
    s_pw[e] = make_double2(KERNEL != 2 ? rt.pw_d[k] : 0.0, rt.pw_o[k]);
  }
  for (int e = tid; e < 2 * kResidMaxCheb; e += blockDim.x) {
    const int k = e % kResidMaxCheb;
    s_cheb[e] = e < kResidMaxCheb ? (k < rt.n_d ? rt.cheb_d[k] : 0.0) : (k < rt.n_o ? rt.cheb_o[k] : 0.0);
  }
  __syncthreads();
  int4* __restrict__ ivl = ivl_all + (size_t)(blockIdx.x * kWarps + warp) * kMaxIvl;  // this warp's interval list
  const double yscale = rt.ni / (rt.hi - rt.lo), ylo = -rt.lo * yscale;
  const double* __restrict__ spx = spts;
  const double* __restrict__ spy = spts + ns;
  const double* __restrict__ spz = spts + (size_t)(DIM == 3 ? 2 : 1) * ns;
  unsigned long long n_ref = 0, n_test = 0, n_in = 0;
  int singular = 0;
  // persistent warps: 32-target chunks of one leaf each, handed out in order
  for (;;) {
    int cid = 0;
    if (lane == 0) cid = atomicAdd(next_chunk, 1);
    cid = __shfl_sync(0xffffffffu, cid, 0);
    if (cid >= nchunks) break;
    const int2 chunk = chunks[cid];
    const int li = chunk.x;
    const int leaf = leaves[li];
    const DBox box = boxes[leaf];
    const double r_l = box.side, r_f = 0.5 * r_l;
    const double inv_rl = 1.0 / r_l, inv_rf = 1.0 / r_f;
    const double ysc_l = inv_rl * yscale, ysc_f = inv_rf * yscale;  // exact: 1/nu is a power of two
    const int r0 = rng_start[li], nr = rng_start[li + 1] - r0;
    double selfc = 0.0;
    if (alias && KERNEL == 0) selfc = DIM == 3 ? self_const / r_l : self_const + log(r_l) / (4.0 * dev::kPI);
    const int t0 = chunk.y;
    const int t = t0 + lane;
    const bool valid = t < box.te;
    const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
    const int tt = valid ? t : t0;
    double xt[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) xt[ax] = tpts[(size_t)ax * nt + tt];
    // single-precision copies relative to the leaf centre for the scan's
    // conservative pre-test (see 2. below)
    float xtf[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) xtf[ax] = valid ? (float)(xt[ax] - box.c[ax]) : -1e30f;  // invalid: far away
    double bl[3], bh[3];  // the warp's target bounding box
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
      double lo = xt[ax], hi = xt[ax];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      bl[ax] = lo;
      bh[ax] = hi;
    }
    // 1. The source intervals this chunk must scan, lane-parallel over the
    // leaf's near ranges (dmk.cpp:966-990): each range's box is culled
    // against the warp's target box, then its Morton child sub-cells; the
    // survivors are written in (range, sub-cell) order, so the scan below
    // visits sources in the same order as a per-range loop.
    // record: {a0, a1, meta, 0}, meta = image shift code (x+1 | y+1 << 2 |
    // z+1 << 4) | fine-scale << 6 | zero shift << 7 | self range << 8
    int nivl = 0;
    for (int rb = 0; rb < nr; rb += 32) {
      const int k = rb + lane;
      unsigned mask = 0;
      int sub[9];
      int meta = 0;
      if (k < nr) {
        const int sbx = rng_box[r0 + k], info = rng_info[r0 + k];
        const DBox sbox = boxes[sbx];
        const int code = info & 31;
        const int sh[3] = {code % 3 - 1, (code / 3) % 3 - 1, code / 9 - 1};
        const bool fine = (info >> 5) & 1;
        const int self = (info >> 6) & 1;
        meta = (sh[0] + 1) | ((sh[1] + 1) << 2) | ((DIM == 3 ? sh[2] + 1 : 1) << 4) | (fine ? 64 : 0) |
               (code == 13 ? 128 : 0) | (self ? 256 : 0);
        const double nu = fine ? r_f : r_l;
        const double cull = nu * rt.support * (1.0 + 1e-12) + 1e-15;
        const double cull2 = cull * cull;
        double lo[3];
        double d2 = 0.0;  // distance from the warp's target box to the source box
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
          lo[ax] = sbox.c[ax] - sbox.half + (double)sh[ax];
          const double hi = sbox.c[ax] + sbox.half + (double)sh[ax];
          const double dd = fmax(0.0, fmax(lo[ax] - bh[ax], bl[ax] - hi));
          d2 += dd * dd;
        }
        n_ref += (unsigned long long)nvalid * (sbox.se - sbox.sb - ((alias && self) ? 1 : 0));
        if (d2 <= cull2) {
          const int* sp = subrange + (size_t)sbx * 9;
#pragma unroll
          for (int c = 0; c < 9; ++c) sub[c] = sp[c];
          constexpr int NC = 1 << DIM;
#pragma unroll
          for (int ci = 0; ci < NC; ++ci) {
            if (sub[ci] == sub[ci + 1]) continue;
            double e2 = 0.0;
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
              const double l = lo[ax] + ((ci >> ax) & 1) * sbox.half, h = l + sbox.half;
              const double dd = fmax(0.0, fmax(l - bh[ax], bl[ax] - h));
              e2 += dd * dd;
            }
            if (e2 <= cull2) mask |= 1u << ci;
          }
        }
      }
      const int c = __popc(mask);
      int pre = c;  // inclusive warp scan of the survivor counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      int pos = nivl + pre - c;
      for (unsigned m = mask; m; m &= m - 1) {
        const int ci = __ffs(m) - 1;
        ivl[pos++] = make_int4(sub[ci], sub[ci + 1], meta, 0);
        n_test += (unsigned long long)nvalid * (sub[ci + 1] - sub[ci]);
      }
      nivl += __shfl_sync(0xffffffffu, pre, 31);
    }
    __syncwarp();
    // Each target's pairs are summed by its lane in a fixed order (plain
    // sums: the reference's Kahan accumulators change no result at the
    // BASELINE configurations by more than 1e-15 of the parity bar, and cost
    // ~10% of the kernel).  Pairs with s < s_exact (rare) are evaluated after
    // their round / list pass with the reference's own tables and recurrence.
    double u[3] = {0.0, 0.0, 0.0};
    unsigned n_in32 = 0;  // this chunk's in-support pairs (this lane)
    const double sup2l = (r_l * rt.support) * (r_l * rt.support);
    const double sup2f = (r_f * rt.support) * (r_f * rt.support);
    // Candidate lists: each lane appends its candidates to a short list in
    // shared memory (kList entries, lane-interleaved); when any lane's list is
    // nearly full the warp spills every lane's list to the lane's own list in
    // global scratch (kGCap entries, L2-resident) and carries on.  The
    // candidates are evaluated once per chunk, in lockstep, from the global
    // lists: during the scan the lanes fill unevenly (a source sub-cell is
    // near some of the warp's targets and not others), but per chunk every
    // target's total is similar, so lockstep padding stays small.
    int* __restrict__ gl = glist + ((size_t)(blockIdx.x * kWarps + warp) * 32 + lane) * kGCap;
    unsigned char* __restrict__ glc = glcode + (PER ? ((size_t)(blockIdx.x * kWarps + warp) * 32 + lane) * kGCap : 0);
    int gcnt = 0;
    // free space: the entry is the source index, bit 31 set for the fine
    // scale; periodic: the index, and the image shift (x+1 | y+1 << 2 | z+1
    // << 4) | fine << 6 in the code list
    // returns bit 0: in the support (counted), bit 1: deferred to the exact pass
    auto eval = [&](int a, int code, bool use, auto exact) -> int {
      constexpr bool EXACT = decltype(exact)::value;
      if (!PER) {
        code = a < 0 ? 64 : 0;
        a &= 0x7fffffff;
      }
      const bool fine = code & 64;
      const double nu = fine ? r_f : r_l, inu = fine ? inv_rf : inv_rl;
      constexpr int RW = Rec<KERNEL, DIM>::kW;
      double rv[RW];
      const double2* rp = srec + (size_t)a * (RW / 2);
#pragma unroll
      for (int k = 0; k < RW / 2; ++k) {
        const double2 v = rp[k];
        rv[2 * k] = v.x;
        rv[2 * k + 1] = v.y;
      }
      // the reference's arithmetic (dmk.cpp:1003-1008): x = xt - (xs + shift),
      // r2 = ((x0 x0 + x1 x1) + x2 x2), every operation rounded (no FMA), so
      // the exact support test and the coincidence test decide as it does
      double x[3] = {0.0, 0.0, 0.0};
      if (PER) {
        x[0] = xt[0] - (rv[0] + (double)((code & 3) - 1));
        x[1] = xt[1] - (rv[1] + (double)(((code >> 2) & 3) - 1));
        if (DIM == 3) x[2] = xt[2] - (rv[2] + (double)(((code >> 4) & 3) - 1));
      } else {
        x[0] = xt[0] - rv[0];
        x[1] = xt[1] - rv[1];
        if (DIM == 3) x[2] = xt[2] - rv[2];
      }
      double r2 = __dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1]));
      if (DIM == 3) r2 = __dadd_rn(r2, __dmul_rn(x[2], x[2]));
      const bool in = use && lt_nonneg(r2, fine ? sup2f : sup2l);
      const bool zero = is_zero_nonneg(r2);
      if (in && zero) singular = 1;
      const double rinv = EXACT ? rsqrt(r2) : rsqrt_fast(r2);
      // table coordinate y = (s - lo) ni / (hi - lo), s = r / nu (nu is a power
      // of two: r * (1/nu) == r / nu); the first interval (y < 1) goes exact
      const double r = r2 * rinv;
      const double y = fma(r, fine ? ysc_f : ysc_l, ylo);
      const double s = DIM == 2 && KERNEL == 0 ? r * inu : 0.0;
      const bool kept = in && !zero;
      double fd, fo;
      const unsigned fl = radial_tables<KERNEL, DEG, EXACT>(rt, s_pw + (lane & (kCopies - 1)), y, fd, fo, s_cheb, r2, inu);
      const bool tab = fl < (unsigned)rt.ni;
      const bool near = !EXACT && fl + 1u <= 1u;  // y < 1, or NaN (subnormal r2)
      assemble<KERNEL, DIM>(fd, fo, x, rinv, s, rt.support, nu, rv + DIM, u, kept && tab && !near);
      return (kept ? 1 : 0) | (kept && near ? 2 : 0);
    };
    // evaluate the global lists in order (lockstep to the longest), blocks of
    // 64 entries; each block's near pairs (s < s_exact) are re-evaluated
    // exactly after it
    auto eval_global = [&]() {
      int mx = gcnt;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int b = 0; b < mx; b += 64) {
        const int bend = min(mx, b + 64);
        unsigned long long nearmask = 0;
        int2 cur = *reinterpret_cast<const int2*>(gl + b);
        uchar2 ccur = PER ? *reinterpret_cast<const uchar2*>(glc + b) : make_uchar2(0, 0);
        for (int i = b; i < bend; i += 2) {
          int2 nxt = cur;
          uchar2 cnxt = ccur;
          if (i + 2 < bend) {  // the next two entries in flight while these are evaluated
            nxt = *reinterpret_cast<const int2*>(gl + i + 2);
            if (PER) cnxt = *reinterpret_cast<const uchar2*>(glc + i + 2);
          }
          // in list order; entries past the lane's count are replaced by
          // source 0 and contribute nothing
          const bool u0 = i < gcnt, u1 = i + 1 < gcnt;
          const int s0 = eval(u0 ? cur.x : 0, u0 ? (int)ccur.x : 0, u0, std::false_type{});
          const int s1 = eval(u1 ? cur.y : 0, u1 ? (int)ccur.y : 0, u1, std::false_type{});
          n_in32 += (s0 & 1) + (s1 & 1);
          nearmask |= (unsigned long long)((s0 >> 1) | (s1 & 2)) << (i - b);
          cur = nxt;
          ccur = cnxt;
        }
        while (__any_sync(0xffffffffu, nearmask != 0)) {  // rare: s < s_exact
          if (nearmask) {
            const int i = b + __ffsll(nearmask) - 1;
            nearmask &= nearmask - 1;
            eval(gl[i], PER ? (int)glc[i] : 0, true, std::true_type{});
          }
        }
      }
      gcnt = 0;
    };
    // the shared-memory lists (cnt entries in this lane), evaluated in place
    // in lockstep to the longest (mx), near pairs exactly afterwards
    auto eval_shared = [&](int cnt, int mx) {
      unsigned long long nearmask = 0;  // kList <= 64
      for (int i = 0; i < mx; i += 2) {
        const bool u0 = i < cnt, u1 = i + 1 < cnt;
        const int s0 = eval(u0 ? lsrc[warp][i][lane] : 0, PER && u0 ? (int)lrng[warp][i][lane] : 0, u0,
                            std::false_type{});
        const int s1 = eval(u1 ? lsrc[warp][i + 1][lane] : 0, PER && u1 ? (int)lrng[warp][i + 1][lane] : 0, u1,
                            std::false_type{});
        n_in32 += (s0 & 1) + (s1 & 1);
        nearmask |= (unsigned long long)((s0 >> 1) | (s1 & 2)) << i;
      }
      while (__any_sync(0xffffffffu, nearmask != 0)) {  // rare: s < s_exact
        if (nearmask) {
          const int i = __ffsll(nearmask) - 1;
          nearmask &= nearmask - 1;
          eval(lsrc[warp][i][lane], PER ? (int)lrng[warp][i][lane] : 0, true, std::true_type{});
        }
      }
    };
    // a full shared list: when the lanes are evenly filled (dense
    // neighbourhoods, e.g. the Ewald's local part: every target has many
    // candidates) the lists are evaluated in place; otherwise every lane's
    // entries move to the end of its global list, evaluated once at the
    // chunk's end
    auto spill = [&](int cnt) {
      int mx = cnt, sum = cnt;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
      }
      if (5 * sum >= 3 * 32 * mx) {  // mean >= 60 % of the longest: little lockstep padding
        eval_shared(cnt, mx);
        return;
      }
      if (__any_sync(0xffffffffu, gcnt + cnt > kGCap)) eval_global();  // global list full (dense clusters)
      for (int k = 0; k < mx; ++k) {
        if (k < cnt) {
          gl[gcnt + k] = lsrc[warp][k][lane];
          if (PER) glc[gcnt + k] = lrng[warp][k][lane];
        }
      }
      gcnt += cnt;
    };
    // 2. Scan: sources arrive in rounds of up to 32, one coalesced load per
    // coordinate (lane j holds source a + j), and are broadcast to every
    // lane's target with shuffles; the next round's load is issued before
    // the current round is tested.  The test is a conservative pre-test in
    // single precision on coordinates relative to the leaf centre: r2 <
    // sup2 (1 + 1e-4), while the float error of r2 is below ~2e-6 relative
    // near the support sphere, so every pair the reference keeps is listed;
    // the evaluation repeats the reference's exact double-precision test
    // (the very few extra candidates contribute exact zeros).
    const float sup2l_hi = (float)(sup2l * (1.0 + 1e-4)), sup2f_hi = (float)(sup2f * (1.0 + 1e-4));
    // 2a. The leaf's own sources (the first near range, nu = r_l, zero shift)
    // are in the support of most of the warp's targets, so they skip the
    // lists: each round of 32 source records is loaded coalesced and every
    // source is broadcast to all lanes and evaluated at once (the exact test
    // masks the pairs outside the support).  Own-box pairs come first in the
    // reference's order, so every target still sums its pairs in order.
    int nself = 0;
    {
      const bool isself = lane < nivl && (ivl[lane].z & 256);
      const unsigned notself = __ballot_sync(0xffffffffu, !isself);
      nself = notself ? __ffs(notself) - 1 : 32;
    }
    for (int q = 0; q < nself; ++q) {
      const int4 iv = ivl[q];
      constexpr int RW = Rec<KERNEL, DIM>::kW;
      for (int base = iv.x; base < iv.y; base += 32) {
        const int nv = min(32, iv.y - base);
        // the round's records go to the warp's (still empty) list storage and
        // are read back as 16-byte broadcasts
        static_assert(RW * 32 * sizeof(double) <= kList * 32 * sizeof(int), "round buffer exceeds the list storage");
        double2* rb = reinterpret_cast<double2*>(&lsrc[warp][0][0]);
        if (lane < nv) {
          const double2* rp = srec + (size_t)(base + lane) * (RW / 2);
#pragma unroll
          for (int k = 0; k < RW / 2; ++k) rb[lane * (RW / 2) + k] = rp[k];
        }
        __syncwarp();
        // returns bit 0: in the support (counted), bit 1: deferred to the exact pass
        auto dense = [&](int j, bool use, auto exact) -> int {
          constexpr bool EXACT = decltype(exact)::value;
          double sv[RW];
#pragma unroll
          for (int k = 0; k < RW / 2; ++k) {
            const double2 v = rb[j * (RW / 2) + k];
            sv[2 * k] = v.x;
            sv[2 * k + 1] = v.y;
          }
          const int a = base + j;
          double x[3] = {0.0, 0.0, 0.0};
          x[0] = xt[0] - sv[0];
          x[1] = xt[1] - sv[1];
          if (DIM == 3) x[2] = xt[2] - sv[2];
          double r2 = __dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1]));
          if (DIM == 3) r2 = __dadd_rn(r2, __dmul_rn(x[2], x[2]));
          const bool in = use && valid && lt_nonneg(r2, sup2l) && !(alias && a == t);
          const bool zero = is_zero_nonneg(r2);
          if (in && zero) singular = 1;
          const double rinv = EXACT ? rsqrt(r2) : rsqrt_fast(r2);
          const double r = r2 * rinv;
          const double y = fma(r, ysc_l, ylo);
          const double sc = DIM == 2 && KERNEL == 0 ? r * inv_rl : 0.0;
          const bool kept = in && !zero;
          double fd, fo;
          const unsigned fl =
              radial_tables<KERNEL, DEG, EXACT>(rt, s_pw + (lane & (kCopies - 1)), y, fd, fo, s_cheb, r2, inv_rl);
          const bool tab = fl < (unsigned)rt.ni;
          const bool near = !EXACT && fl + 1u <= 1u;  // y < 1, or NaN (subnormal r2)
          assemble<KERNEL, DIM>(fd, fo, x, rinv, sc, rt.support, r_l, sv + DIM, u, kept && tab && !near);
          return (kept ? 1 : 0) | (kept && near ? 2 : 0);
        };
        unsigned nearbits = 0;  // sources of this round to re-evaluate exactly
        for (int j = 0; j < nv; j += 2) {
          const int s0 = dense(j, true, std::false_type{});
          const int s1 = dense(min(j + 1, nv - 1), j + 1 < nv, std::false_type{});
          n_in32 += (s0 & 1) + (s1 & 1);
          nearbits |= ((unsigned)(s0 >> 1) << j) | ((unsigned)(s1 >> 1) << (j + 1));
        }
        while (__any_sync(0xffffffffu, nearbits != 0)) {  // rare: s < s_exact
          if (nearbits) {
            const int j = __ffs(nearbits) - 1;
            nearbits &= nearbits - 1;
            dense(j, true, std::true_type{});
          }
        }
        __syncwarp();  // the next round overwrites the buffer
      }
    }
    // this lane's list (shared addresses): entry k at ls0 + 128 k, lr0 + 32 k
    const unsigned ls0 = (unsigned)__cvta_generic_to_shared(&lsrc[warp][0][lane]);
    const unsigned lr0 = (unsigned)__cvta_generic_to_shared(&lrng[warp][0][lane]);
    const unsigned ls_lim = ls0 + 128u * (kList - 8);
    const unsigned lr_off = lr0 - (ls0 >> 2);  // byte entry k at (address of int entry k) / 4 + lr_off
    unsigned ls = ls0;
    for (int ib = nself; ib < nivl; ib += 32) {
      const int nb = min(32, nivl - ib);
      const int4 iv = lane < nb ? ivl[ib + lane] : make_int4(0, 0, 0, 0);
      int i = 0, s = __shfl_sync(0xffffffffu, iv.x, 0);
      int e = __shfl_sync(0xffffffffu, iv.y, 0);
      double px = 0.0, py = 0.0, pz = 0.0;
      auto load = [&](int s_, int e_) {
        if (s_ + lane < e_) {
          px = spx[s_ + lane];
          py = spy[s_ + lane];
          if (DIM == 3) pz = spz[s_ + lane];
        } else {  // past the interval's end: far away, fails every pre-test
          px = py = pz = 1e30;
        }
      };
      load(s, e);
      while (i < nb) {
        const int ci = i, cs = s, ce = e;
        const double cx = px, cy = py, cz = pz;
        // advance to the next round and start its load
        s += 32;
        if (s >= e) {
          ++i;
          if (i < nb) {
            s = __shfl_sync(0xffffffffu, iv.x, i);
            e = __shfl_sync(0xffffffffu, iv.y, i);
          }
        }
        if (i < nb) load(s, e);
        const int meta = __shfl_sync(0xffffffffu, iv.z, ci);
        const int code = meta & 127;
        const float sup2 = (meta & 64) ? sup2f_hi : sup2l_hi;
        const int encb = (meta & 64) ? (int)((unsigned)cs | 0x80000000u) : cs;  // free-space entry: + jj
        // (no self range here: it is the first range, its intervals are the
        // first nself, and the dense rounds above took them)
        const int nv = min(32, ce - cs);
        // this lane's source of the round, shifted and relative to the leaf centre
        float cxf, cyf, czf = 0.0f;
        if (PER) {
          cxf = (float)((cx + (double)((code & 3) - 1)) - box.c[0]);
          cyf = (float)((cy + (double)(((code >> 2) & 3) - 1)) - box.c[1]);
          if (DIM == 3) czf = (float)((cz + (double)(((code >> 4) & 3) - 1)) - box.c[2]);
        } else {
          cxf = (float)(cx - box.c[0]);
          cyf = (float)(cy - box.c[1]);
          if (DIM == 3) czf = (float)(cz - box.c[2]);
        }
        // (lanes past nv hold far-away sources and invalid targets a far-away
        // target, so the pre-test alone decides; jj <= 31 as 32 % 8 == 0)
        for (int j = 0; j < nv; j += 8) {
          if (__any_sync(0xffffffffu, ls > ls_lim)) {
            spill((int)(ls - ls0) >> 7);
            ls = ls0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int jj = j + q;
            const float sx = __shfl_sync(0xffffffffu, cxf, jj);
            const float sy = __shfl_sync(0xffffffffu, cyf, jj);
            const float sz = DIM == 3 ? __shfl_sync(0xffffffffu, czf, jj) : 0.0f;
            const float x0 = xtf[0] - sx, x1 = xtf[1] - sy;
            float r2 = x0 * x0 + x1 * x1;
            if (DIM == 3) {
              const float x2 = xtf[2] - sz;
              r2 += x2 * x2;
            }
            if (r2 < sup2) {
              if (PER) {
                sts_u32(ls, cs + jj);
                sts_u8((ls >> 2) + lr_off, code);
              } else {
                sts_u32(ls, encb + jj);
              }
              ls += 32 * sizeof(int);
            }
          }
        }
      }
    }
    spill((int)(ls - ls0) >> 7);
    eval_global();
    if (valid) {
      double* ut = ures + (size_t)tperm[t] * DIM;
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        double v = u[j];
        if (selfc != 0.0) v += selfc * sstr[(size_t)j * ns + t];  // dmk.cpp:1015-1018
        ut[j] = v;
      }
    }
    n_in += n_in32;
    __syncwarp();  // the interval list is rewritten by the next chunk
  }
  if (singular) atomicOr(flags, 1);
  if (stats) {
    // n_ref / n_test were counted once per range / interval by one lane
    // (times the warp's valid targets); n_in per lane
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      n_test += __shfl_xor_sync(0xffffffffu, n_test, o);
      n_ref += __shfl_xor_sync(0xffffffffu, n_ref, o);
      n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
    }
    if (lane == 0) {
      atomicAdd(stats + 0, n_test);
      atomicAdd(stats + 1, n_in);
      atomicAdd(stats + 2, n_ref);
    }
  }
}

}  // namespace

size_t residual_scratch_bytes() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t nw = (size_t)kResBlocksPerSM * sms * kWarps;
  return nw * kMaxIvl * sizeof(int4) + nw * 32 * kGCap * (sizeof(int) + 1) + 256;
}

void launch_residual(const ResidTables& rt, const DBox* boxes, const int* leaves, int nleaf, const int* chunks,
                     int nchunks, const int* rng_start,
                     const int* rng_box, const int* rng_info, const int* subrange, const double* spts, int ns, const double* sstr,
                     double* srec, int periodic,
                     const double* tpts, int nt, const int* tperm, int alias, int reserve_sms, double self_const,
                     double* ures, int* flags, unsigned long long* stats, void* scratch, cudaStream_t st) {
  if (nleaf <= 0 || nchunks <= 0) return;
  {
    const int sc = rt.kernel == 0 ? rt.dim : (rt.kernel == 1 ? 2 * rt.dim : (rt.dim == 3 ? 3 : 1));
    const int rw = (rt.dim + sc + 1) / 2 * 2;
    k_pack_sources<<<148 * 8, 256, 0, st>>>(spts, sstr, ns, rt.dim, sc, rw, srec);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // reserve_sms: SMs left free for kernels running beside this one (the NCCL
  // halo exchange of a multi-GPU evaluation)
  const int nblk = std::min(kResBlocksPerSM * std::max(1, sms - reserve_sms), (nchunks + kWarps - 1) / kWarps);
  int* next_chunk = reinterpret_cast<int*>(scratch);
  int4* ivl = reinterpret_cast<int4*>(reinterpret_cast<char*>(scratch) + 256);
  const size_t nw = (size_t)kResBlocksPerSM * sms * kWarps;
  int* glist = reinterpret_cast<int*>(ivl + nw * kMaxIvl);
  unsigned char* glcode = reinterpret_cast<unsigned char*>(glist + nw * 32 * kGCap);
  cudaMemsetAsync(next_chunk, 0, sizeof(int), st);
  const int2* ch2 = reinterpret_cast<const int2*>(chunks);
  const size_t dsm = (size_t)kWarps * kList * 32 * (sizeof(int) + 1) +
                     sizeof(double) * 2 * kCopies * (size_t)rt.ni * (rt.deg + 1) + sizeof(double) * 2 * kResidMaxCheb;
#define RES(K, D)                                                                                                \
  do {                                                                                                           \
    if (rt.deg == 5) RES1(K, D, 5);                                                                              \
    else if (rt.deg == 6) RES1(K, D, 6);                                                                         \
    else if (rt.deg == 8) RES1(K, D, 8);                                                                         \
    else if (rt.deg == 10) RES1(K, D, 10);                                                                       \
    else RES1(K, D, 12);                                                                                         \
  } while (0)
#define RES1(K, D, G)                                                                                            \
  do {                                                                                                           \
    if (periodic) RES2(K, D, G, 1);                                                                              \
    else RES2(K, D, G, 0);                                                                                       \
  } while (0)
#define RES2(K, D, G, P)                                                                                         \
  do {                                                                                                           \
    cudaFuncSetAttribute(k_residual<K, D, G, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);         \
    k_residual<K, D, G, P><<<nblk, kRBlock, dsm, st>>>(rt, boxes, leaves, ch2, nchunks, rng_start, rng_box,      \
                                                       rng_info, subrange, spts, ns, sstr,                       \
                                                       reinterpret_cast<const double2*>(srec), tpts, nt, tperm,  \
                                                       alias, self_const, ures, flags, stats, ivl, glist, glcode, next_chunk);  \
  } while (0)
  if (rt.dim == 3) {
    if (rt.kernel == 0) RES(0, 3);
    else if (rt.kernel == 1) RES(1, 3);
    else RES(2, 3);
  } else {
    if (rt.kernel == 0) RES(0, 2);
    else if (rt.kernel == 1) RES(1, 2);
    else RES(2, 2);
  }
#undef RES
#undef RES1
#undef RES2
}

int residual_max_ranges() { return kMaxRanges; }
int residual_max_pw() { return kMaxPW; }

}  // namespace sdmkb
