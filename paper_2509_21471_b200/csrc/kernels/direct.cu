// O(N*M) reference sums on the GPU:
//   direct_sum           (oracle.cpp:143-179)  exact free-space kernels
//   direct_residual_sum  (oracle.cpp:181-241)  residual kernel at one scale,
//                        with the 3^d image shifts when periodic
// Each target's sources are summed by one thread in the reference's order
// (sources ascending; shifts i2, i1, i0 nested with i0 fastest) with the
// same Kahan accumulator and the same expression trees as accumulate_exact
// (oracle.cpp:32-94) and residual_apply (split.cpp:258-317), and this file
// is compiled with -fmad=false (Makefile), so no product is fused into an
// add.  IEEE division and sqrt are correctly rounded on both sides, so the
// results are bitwise equal to the reference's, except where a kernel needs
// log (2D Stokeslet): CUDA's log is within 1 ulp of glibc's.
//
// Layout: sources are staged in shared memory as point-major records
// (coordinates then strengths, the caller's AoS order), a tile of kTile
// sources per step; every thread reads the same record (broadcast).
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

constexpr int kDBlock = 128;
constexpr int kTPT = 2;      // targets per thread (two independent Kahan chains)
constexpr int kTile = 256;   // sources per shared-memory tile
constexpr double kPi = 3.141592653589793238462643383279502884;

struct Kahan {  // oracle.cpp:20-30
  double sum = 0.0, comp = 0.0;
  __device__ __forceinline__ void add(double x) {
    double y = x - comp;
    double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
};

// accumulate_exact (oracle.cpp:32-94), x = target - source
template <int KERNEL, int DIM>
__device__ __forceinline__ void acc_exact(const double* x, double r2, const double* s, Kahan* u) {
  if (DIM == 3) {
    const double r = sqrt(r2);
    if (KERNEL == 0) {
      const double xf = x[0] * s[0] + x[1] * s[1] + x[2] * s[2];
      const double c1 = 1.0 / (8.0 * kPi * r);
      const double c2 = xf / (8.0 * kPi * r2 * r);
      for (int j = 0; j < 3; ++j) u[j].add(c1 * s[j] + c2 * x[j]);
    } else if (KERNEL == 1) {
      const double* f = s;
      const double* n = s + 3;
      const double xf = x[0] * f[0] + x[1] * f[1] + x[2] * f[2];
      const double xn = x[0] * n[0] + x[1] * n[1] + x[2] * n[2];
      const double c = -3.0 / (4.0 * kPi) * xf * xn / (r2 * r2 * r);
      for (int j = 0; j < 3; ++j) u[j].add(c * x[j]);
    } else {
      const double c = 1.0 / (8.0 * kPi * r2 * r);
      u[0].add(c * (s[1] * x[2] - s[2] * x[1]));
      u[1].add(c * (s[2] * x[0] - s[0] * x[2]));
      u[2].add(c * (s[0] * x[1] - s[1] * x[0]));
    }
  } else {
    if (KERNEL == 0) {
      const double xf = x[0] * s[0] + x[1] * s[1];
      const double c1 = -0.5 * log(r2) / (4.0 * kPi);
      const double c2 = xf / (4.0 * kPi * r2);
      for (int j = 0; j < 2; ++j) u[j].add(c1 * s[j] + c2 * x[j]);
    } else if (KERNEL == 1) {
      const double* f = s;
      const double* n = s + 2;
      const double xf = x[0] * f[0] + x[1] * f[1];
      const double xn = x[0] * n[0] + x[1] * n[1];
      const double c = -xf * xn / (kPi * r2 * r2);
      for (int j = 0; j < 2; ++j) u[j].add(c * x[j]);
    } else {
      const double c = s[0] / (4.0 * kPi * r2);
      u[0].add(c * x[1]);
      u[1].add(-c * x[0]);
    }
  }
}

// ChebTable::eval (chebyshev.cpp:9-19), coefficients in shared memory
__device__ __forceinline__ double cheb_eval(const double* a, int n, double lo, double hi, double x) {
  if (n == 0) return 0.0;
  double t = (2.0 * x - lo - hi) / (hi - lo);
  double b1 = 0.0, b2 = 0.0;
  for (int k = n - 1; k >= 1; --k) {
    double b0 = 2.0 * t * b1 - b2 + a[k];
    b2 = b1;
    b1 = b0;
  }
  return t * b1 - b2 + a[0];
}

struct ChebS {
  const double* a;
  int n;
  double lo, hi;
};

// residual_apply (split.cpp:258-317) into u (u starts at zero per pair, as
// the reference's tmp[3])
template <int KERNEL, int DIM>
__device__ __forceinline__ void res_apply(const DirectTables& T, const ChebS& td, const ChebS& to, const double* x,
                                          double nu, const double* s, double* u) {
  double r2 = 0.0;
  for (int i = 0; i < DIM; ++i) r2 += x[i] * x[i];  // norm2
  const double cut = nu * T.support;
  if (r2 >= cut * cut || r2 == 0.0) return;
  const double r = sqrt(r2), sc = r / nu;
  // *_residual_diag / _offd (split.cpp:181-227): |s| >= support -> 0
  const double sa = fabs(sc);
  auto diag = [&]() -> double {
    if (sa >= T.support) return 0.0;
    if (KERNEL == 0 && DIM == 2) {
      const double exact = sa > 0.0 ? -2.0 * sa * log(sa) : 0.0;
      return exact - cheb_eval(td.a, td.n, td.lo, td.hi, sa);
    }
    return cheb_eval(td.a, td.n, td.lo, td.hi, sa);
  };
  auto offd = [&]() -> double { return sa >= T.support ? 0.0 : cheb_eval(to.a, to.n, to.lo, to.hi, sa); };
  if (KERNEL == 0) {
    const double amp = DIM == 2 ? nu : 1.0;
    const double fd = amp * diag();
    const double fo = amp * offd();
    const double c0 = 1.0 / (8.0 * kPi * r);
    double xf = 0.0;
    for (int i = 0; i < DIM; ++i) xf += x[i] * s[i];
    const double cf = fo * c0 * xf / r2;
    for (int j = 0; j < DIM; ++j) u[j] += fd * c0 * s[j] + cf * x[j];
  } else if (KERNEL == 1) {
    const double* f = s;
    const double* nrm = s + DIM;
    const double amp = DIM == 2 ? nu : 1.0;
    const double fd = amp * diag();
    const double fo = amp * offd();
    double xf = 0.0, xn = 0.0, fn = 0.0;
    for (int i = 0; i < DIM; ++i) {
      xf += x[i] * f[i];
      xn += x[i] * nrm[i];
      fn += f[i] * nrm[i];
    }
    const double cd = fd / (8.0 * kPi * r2 * r);
    const double co = -3.0 * fo * xf * xn / (4.0 * kPi * r2 * r2 * r);
    for (int j = 0; j < DIM; ++j) u[j] += cd * (f[j] * xn + x[j] * fn + nrm[j] * xf) + co * x[j];
  } else {
    const double fo = offd();
    if (DIM == 2) {
      const double c0 = fo * s[0] / (4.0 * kPi * r2);
      u[0] += c0 * x[1];
      u[1] -= c0 * x[0];
    } else {
      const double c0 = fo / (8.0 * kPi * r2 * r);
      u[0] += c0 * (s[1] * x[2] - s[2] * x[1]);
      u[1] += c0 * (s[2] * x[0] - s[0] * x[2]);
      u[2] += c0 * (s[0] * x[1] - s[1] * x[0]);
    }
  }
}

template <int KERNEL, int DIM>
struct Width {
  static constexpr int kSc = KERNEL == 0 ? DIM : (KERNEL == 1 ? 2 * DIM : (DIM == 3 ? 3 : 1));
  static constexpr int kW = DIM + kSc;
};

// RES = false: direct_sum; RES = true: direct_residual_sum
template <int KERNEL, int DIM, bool RES>
__global__ void __launch_bounds__(kDBlock) k_direct(const double* __restrict__ src, int ns, const double* __restrict__ tgt,
                                                    int nt, const double* __restrict__ str, int alias, DirectTables T,
                                                    double* __restrict__ u, int* flags) {
  constexpr int SC = Width<KERNEL, DIM>::kSc, W = Width<KERNEL, DIM>::kW;
  __shared__ double s_rec[kTile * W];
  __shared__ double s_cheb[2 * kDirectMaxCheb];
  const int tid = threadIdx.x;
  ChebS td{s_cheb, 0, 0.0, 1.0}, to{s_cheb + kDirectMaxCheb, 0, 0.0, 1.0};
  if (RES) {
    for (int k = tid; k < T.nd; k += blockDim.x) s_cheb[k] = T.cd[k];
    for (int k = tid; k < T.no; k += blockDim.x) s_cheb[kDirectMaxCheb + k] = T.co[k];
    td.n = T.nd;
    td.lo = T.dlo;
    td.hi = T.dhi;
    to.n = T.no;
    to.lo = T.olo;
    to.hi = T.ohi;
  }
  const double sup2 = T.cutoff * T.support * T.cutoff * T.support;  // oracle.cpp:199
  int b[kTPT];
  double xb[kTPT][DIM];
  Kahan acc[kTPT][3];
#pragma unroll
  for (int q = 0; q < kTPT; ++q) {
    b[q] = blockIdx.x * kDBlock * kTPT + q * kDBlock + tid;
    const int bb = b[q] < nt ? b[q] : nt - 1;
#pragma unroll
    for (int i = 0; i < DIM; ++i) xb[q][i] = tgt[(size_t)bb * DIM + i];
  }
  int singular = 0;
  for (int a0 = 0; a0 < ns; a0 += kTile) {
    const int na = min(kTile, ns - a0);
    __syncthreads();
    for (int e = tid; e < na * W; e += blockDim.x) {
      const int a = e / W, k = e - a * W;
      s_rec[e] = k < DIM ? src[(size_t)(a0 + a) * DIM + k] : str[(size_t)(a0 + a) * SC + (k - DIM)];
    }
    __syncthreads();
    for (int ai = 0; ai < na; ++ai) {
      const double* rec = s_rec + ai * W;
      const int a = a0 + ai;
#pragma unroll
      for (int q = 0; q < kTPT; ++q) {
        if (!RES) {
          if (alias && a == b[q]) continue;
          double x[3], r2 = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            x[i] = xb[q][i] - rec[i];
            r2 += x[i] * x[i];
          }
          if (r2 == 0.0) {
            singular |= b[q] < nt;
            continue;
          }
          acc_exact<KERNEL, DIM>(x, r2, rec + DIM, acc[q]);
        } else {
          const int lo = T.periodic ? -1 : 0, hi = T.periodic ? 1 : 0;
          for (int i2 = (DIM == 3 ? lo : 0); i2 <= (DIM == 3 ? hi : 0); ++i2)
            for (int i1 = lo; i1 <= hi; ++i1)
              for (int i0 = lo; i0 <= hi; ++i0) {
                const double p[3] = {(double)i0, (double)i1, (double)i2};
                const bool zero_shift = p[0] == 0.0 && p[1] == 0.0 && (DIM == 2 || p[2] == 0.0);
                if (alias && a == b[q] && zero_shift) continue;
                double x[3], r2 = 0.0;
#pragma unroll
                for (int i = 0; i < DIM; ++i) {
                  x[i] = xb[q][i] - rec[i] - p[i];
                  r2 += x[i] * x[i];
                }
                if (r2 == 0.0) {
                  singular |= b[q] < nt;
                  continue;
                }
                if (r2 >= sup2) continue;
                double tmp[3] = {0.0, 0.0, 0.0};
                res_apply<KERNEL, DIM>(T, td, to, x, T.cutoff, rec + DIM, tmp);
#pragma unroll
                for (int j = 0; j < DIM; ++j) acc[q][j].add(tmp[j]);
              }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kTPT; ++q)
    if (b[q] < nt)
#pragma unroll
      for (int j = 0; j < DIM; ++j) u[(size_t)b[q] * DIM + j] = acc[q][j].sum;
  if (singular) atomicOr(flags, 1);
}

}  // namespace

void launch_direct(int kernel, int dim, const double* src, int ns, const double* tgt, int nt, const double* str,
                   int alias, const DirectTables& T, bool residual, double* u, int* flags, cudaStream_t st) {
  if (nt <= 0 || ns <= 0) return;
  const int nblk = (nt + kDBlock * kTPT - 1) / (kDBlock * kTPT);
#define DIR(K, D)                                                                                     \
  do {                                                                                                \
    if (residual) k_direct<K, D, true><<<nblk, kDBlock, 0, st>>>(src, ns, tgt, nt, str, alias, T, u, flags);  \
    else k_direct<K, D, false><<<nblk, kDBlock, 0, st>>>(src, ns, tgt, nt, str, alias, T, u, flags);          \
  } while (0)
  if (dim == 3) {
    if (kernel == 0) DIR(0, 3);
    else if (kernel == 1) DIR(1, 3);
    else DIR(2, 3);
  } else {
    if (kernel == 0) DIR(0, 2);
    else if (kernel == 1) DIR(1, 2);
    else DIR(2, 2);
  }
#undef DIR
}

}  // namespace sdmkb
