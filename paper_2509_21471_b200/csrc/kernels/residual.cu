// K12: near-field residual pass (dmk.cpp:919-1032) with the fused residual
// apply (split.cpp:258-317) and Clenshaw table lookups (chebyshev.cpp:9-19).
//
// One CTA per target leaf, one warp per target at a time.
//  1. The leaf's near ranges (own box nu = r_l, colleague leaves and fine
//     neighbours nu = r_l/2, coarse neighbours nu = r_l; dmk.cpp:980-990) are
//     staged in shared memory with their (shifted) bounding boxes.
//  2. A range whose box lies entirely outside the target's support sphere is
//     skipped warp-uniformly (conservative margin, so no pair with
//     r^2 < (nu*support)^2 is ever dropped).
//  3. Lanes test 32 sources at a time (coalesced SoA loads); in-support pairs
//     are compacted with a ballot into a per-warp list in shared memory.
//  4. When the list fills, all 32 lanes evaluate list entries (two Clenshaw
//     tables + tensor assembly), so the expensive path runs at full SIMT
//     width even though only a few percent of candidates are in support.
//  5. Lane partial sums are combined by a fixed xor-shuffle tree
//     (deterministic run to run), then the alias self term is added.
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

using dev::DBox;

constexpr int kRBlock = 256;
constexpr int kWarps = kRBlock / 32;
constexpr int kCap = 128;
constexpr int kMaxRanges = 160;
constexpr int kMaxPW = 32 * 25;  // ni * (deg + 1) <= 800 doubles per table

struct RangeS {
  double sh[3];
  double lo[3], hi[3];
  double nu, inu, sup2, cull2;
  int sb, se, self;
};

// Radial table values at s (unit scale) from the piecewise monomial form held
// in shared memory: interval i = floor((s - lo) ni / (hi - lo)), local
// u = 2 (frac) - 1, Horner.  Zero at/after the support (split.cpp:147-179).
template <int KERNEL>
__device__ __forceinline__ void radial_tables(const ResidTables& rt, const double* __restrict__ pd,
                                              const double* __restrict__ po, double s, double& fd, double& fo) {
  const bool in = s < rt.support;
  const double y = (s - rt.lo) * (rt.ni / (rt.hi - rt.lo));
  int iv = (int)y;
  iv = iv < 0 ? 0 : (iv >= rt.ni ? rt.ni - 1 : iv);
  const double u = 2.0 * (y - iv) - 1.0;
  const int n1 = rt.deg + 1;
  const double* cd = pd + iv * n1;
  const double* co = po + iv * n1;
  double vd = KERNEL != 2 ? cd[rt.deg] : 0.0, vo = co[rt.deg];
  for (int k = rt.deg - 1; k >= 0; --k) {
    if (KERNEL != 2) vd = fma(vd, u, cd[k]);
    vo = fma(vo, u, co[k]);
  }
  fd = (KERNEL != 2 && in) ? vd : 0.0;
  fo = in ? vo : 0.0;
}

// residual_apply assembly (split.cpp:258-317) given the radial table values;
// rinv = 1/r from rsqrt, so 1/r, 1/r^2, 1/r^3, 1/r^5 are products.
template <int KERNEL, int DIM>
__device__ __forceinline__ void assemble(double fd, double fo, const double* x, double rinv, double s,
                                         double support, double nu, const double* __restrict__ sstr, int ns, int a,
                                         double* u) {
  constexpr double k8pi = 1.0 / (8.0 * dev::kPI), k4pi = 1.0 / (4.0 * dev::kPI);
  const double rinv2 = rinv * rinv;
  if (KERNEL == 0) {  // Stokeslet
    if (DIM == 2) fd = s < support ? (s > 0.0 ? -2.0 * s * log(s) : 0.0) - fd : 0.0;  // split.cpp:147-155
    const double amp = DIM == 2 ? nu : 1.0;
    const double c0 = k8pi * rinv;
    double f[DIM], xf = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      f[i] = sstr[(size_t)i * ns + a];
      xf += x[i] * f[i];
    }
    const double cd = amp * fd * c0, cf = amp * fo * c0 * xf * rinv2;
#pragma unroll
    for (int j = 0; j < DIM; ++j) u[j] += cd * f[j] + cf * x[j];
  } else if (KERNEL == 1) {  // stresslet
    const double amp = DIM == 2 ? nu : 1.0;
    double f[DIM], nn[DIM], xf = 0.0, xn = 0.0, fn = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      f[i] = sstr[(size_t)i * ns + a];
      nn[i] = sstr[(size_t)(DIM + i) * ns + a];
      xf += x[i] * f[i];
      xn += x[i] * nn[i];
      fn += f[i] * nn[i];
    }
    const double rinv3 = rinv2 * rinv;
    const double cd = amp * fd * k8pi * rinv3;
    const double co = -3.0 * k4pi * amp * fo * xf * xn * rinv3 * rinv2;
#pragma unroll
    for (int j = 0; j < DIM; ++j) u[j] += cd * (f[j] * xn + x[j] * fn + nn[j] * xf) + co * x[j];
  } else {  // rotlet
    if (DIM == 2) {
      const double c0 = fo * sstr[a] * k4pi * rinv2;
      u[0] += c0 * x[1];
      u[1] -= c0 * x[0];
    } else {
      const double c0 = fo * k8pi * rinv2 * rinv;
      const double g0 = sstr[a], g1 = sstr[(size_t)ns + a], g2 = sstr[(size_t)2 * ns + a];
      u[0] += c0 * (g1 * x[2] - g2 * x[1]);
      u[1] += c0 * (g2 * x[0] - g0 * x[2]);
      u[DIM - 1] += c0 * (g0 * x[1] - g1 * x[0]);
    }
  }
}

template <int KERNEL, int DIM>
__global__ void __launch_bounds__(kRBlock) k_residual(ResidTables rt, const DBox* __restrict__ boxes,
                                                      const int* __restrict__ leaves,
                                                      const int* __restrict__ rng_start,
                                                      const int* __restrict__ rng_box,
                                                      const int* __restrict__ rng_info,
                                                      const double* __restrict__ spts, int ns,
                                                      const double* __restrict__ sstr,
                                                      const double* __restrict__ tpts, int nt,
                                                      const int* __restrict__ tperm, int alias, double self_const,
                                                      double* __restrict__ ures, int* flags,
                                                      unsigned long long* stats) {
  __shared__ RangeS rs[kMaxRanges];
  __shared__ int lsrc[kWarps][kCap];
  __shared__ unsigned char lrng[kWarps][kCap];
  __shared__ double s_pd[kMaxPW], s_po[kMaxPW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int leaf = leaves[blockIdx.x];
  const DBox box = boxes[leaf];
  const double r_l = box.side, r_f = 0.5 * r_l;
  const int r0 = rng_start[blockIdx.x], nr = rng_start[blockIdx.x + 1] - r0;
  {
    const int npw = rt.ni * (rt.deg + 1);
    for (int k = tid; k < npw; k += blockDim.x) {
      s_pd[k] = KERNEL != 2 ? rt.pw_d[k] : 0.0;
      s_po[k] = rt.pw_o[k];
    }
  }
  for (int k = tid; k < nr; k += blockDim.x) {
    const int sbx = rng_box[r0 + k], info = rng_info[r0 + k];
    const DBox sb = boxes[sbx];
    RangeS R;
    const int code = info & 31;
    const int sh[3] = {code % 3 - 1, (code / 3) % 3 - 1, code / 9 - 1};
    R.nu = (info >> 5) & 1 ? r_f : r_l;
    R.inu = 1.0 / R.nu;
    R.self = (info >> 6) & 1;
    const double sup = R.nu * rt.support;
    R.sup2 = sup * sup;
    const double cs = sup * (1.0 + 1e-12) + 1e-15;
    R.cull2 = cs * cs;
    for (int ax = 0; ax < 3; ++ax) {
      R.sh[ax] = ax < DIM ? (double)sh[ax] : 0.0;
      R.lo[ax] = sb.c[ax] - sb.half + R.sh[ax];
      R.hi[ax] = sb.c[ax] + sb.half + R.sh[ax];
    }
    R.sb = sb.sb;
    R.se = sb.se;
    rs[k] = R;
  }
  __syncthreads();
  double selfc = 0.0;
  if (alias && KERNEL == 0) selfc = DIM == 3 ? self_const / r_l : self_const + log(r_l) / (4.0 * dev::kPI);
  unsigned long long n_ref = 0, n_test = 0, n_in = 0;
  int singular = 0;
  int* ls = lsrc[warp];
  unsigned char* lr = lrng[warp];
  for (int t = box.tb + warp; t < box.te; t += kWarps) {
    double xt[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) xt[ax] = tpts[(size_t)ax * nt + t];
    double u[3] = {0.0, 0.0, 0.0};
    int cnt = 0;
    auto flush = [&]() {
      for (int k = lane; k < cnt; k += 32) {
        const int a = ls[k];
        const RangeS& R = rs[lr[k]];
        double x[3] = {0.0, 0.0, 0.0}, r2 = 0.0;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
          x[ax] = xt[ax] - (spts[(size_t)ax * ns + a] + R.sh[ax]);
          r2 += x[ax] * x[ax];
        }
        const double rinv = rsqrt(r2);
        const double s = (r2 * rinv) * R.inu;  // nu is a power of two: r * (1/nu) == r / nu
        double fd, fo;
        radial_tables<KERNEL>(rt, s_pd, s_po, s, fd, fo);
        assemble<KERNEL, DIM>(fd, fo, x, rinv, s, rt.support, R.nu, sstr, ns, a, u);
      }
      cnt = 0;
      __syncwarp();
    };
    for (int k = 0; k < nr; ++k) {
      const RangeS& R = rs[k];
      const int len = R.se - R.sb;
      n_ref += len - ((alias && R.self) ? 1 : 0);
      double d2 = 0.0;
#pragma unroll
      for (int ax = 0; ax < DIM; ++ax) {
        double dd = fmax(0.0, fmax(R.lo[ax] - xt[ax], xt[ax] - R.hi[ax]));
        d2 += dd * dd;
      }
      if (d2 > R.cull2) continue;  // whole range outside the support sphere
      n_test += len;
      for (int a0 = R.sb; a0 < R.se; a0 += 32) {
        const int a = a0 + lane;
        bool in = false;
        if (a < R.se && !(alias && R.self && a == t)) {
          double r2 = 0.0;
#pragma unroll
          for (int ax = 0; ax < DIM; ++ax) {
            double xv = xt[ax] - (spts[(size_t)ax * ns + a] + R.sh[ax]);
            r2 += xv * xv;
          }
          in = r2 < R.sup2;
          if (in && r2 == 0.0) {
            singular = 1;
            in = false;
          }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        if (in) {
          const int pos = cnt + __popc(mask & ((1u << lane) - 1u));
          ls[pos] = a;
          lr[pos] = (unsigned char)k;
        }
        cnt += __popc(mask);
        n_in += __popc(mask);
        __syncwarp();
        if (cnt > kCap - 32) flush();
      }
    }
    flush();
#pragma unroll
    for (int j = 0; j < DIM; ++j)
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) u[j] += __shfl_xor_sync(0xffffffffu, u[j], o);
    if (lane == 0) {
      double* ut = ures + (size_t)tperm[t] * DIM;
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        double v = u[j];
        if (selfc != 0.0) v += selfc * sstr[(size_t)j * ns + t];
        ut[j] = v;
      }
    }
  }
  if (singular) atomicOr(flags, 1);
  if (stats && lane == 0) {
    atomicAdd(stats + 0, n_test);
    atomicAdd(stats + 1, n_in);
    atomicAdd(stats + 2, n_ref);
  }
}

}  // namespace

void launch_residual(const ResidTables& rt, const DBox* boxes, const int* leaves, int nleaf, const int* rng_start,
                     const int* rng_box, const int* rng_info, const double* spts, int ns, const double* sstr,
                     const double* tpts, int nt, const int* tperm, int alias, double /*unused*/, double self_const,
                     double* ures, int* flags, unsigned long long* stats, cudaStream_t st) {
  if (nleaf <= 0) return;
#define RES(K, D)                                                                                              \
  k_residual<K, D><<<nleaf, kRBlock, 0, st>>>(rt, boxes, leaves, rng_start, rng_box, rng_info, spts, ns, sstr, \
                                              tpts, nt, tperm, alias, self_const, ures, flags, stats)
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
}

int residual_max_ranges() { return kMaxRanges; }
int residual_max_pw() { return kMaxPW; }

}  // namespace sdmkb
