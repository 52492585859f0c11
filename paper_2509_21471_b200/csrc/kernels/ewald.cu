// FFT Ewald far field for the periodic 3D Stokeslet: the
// smooth part of the single-level split at scale nu (ewald.cpp:81-272 sums it
// mode by mode) through a type-1 / type-2 NUFFT pair on a uniform grid:
//   spread   g_j = sum_s f_s Phi(x_j - x_s),  Phi = phi(x/a) phi(y/a) phi(z/a)
//            (phi: a prolate spheroidal window on [-1, 1], a = w h / 2)
//   FFT      g^ (cuFFT, real -> half spectrum)
//   symbol   b = A(|k|) (k^2 g^ - k (k . g^)) D(k)^2, A = gamma^(k nu) / k^4,
//            D = h^3 / Phi^(k) (deconvolution, separable), k = 2 pi kappa != 0
//   inverse  b(x_j) (cuFFT, half spectrum -> real, unnormalized)
//   gather   u(x_t) = sum_j Phi(x_t - x_j) b(x_j)
// Coordinates are shifted to [0, 1) (the sum is translation invariant), so
// grid point j sits at j h with no phase factor.
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

// phi(|z|) on [0, 1): piecewise monomials of degree deg on ni intervals
__device__ __forceinline__ double ew_phi(const EwGrid& g, double az) {
  if (az >= 1.0) return 0.0;
  const double y = az * g.ni;
  int iv = (int)y;
  iv = iv >= g.ni ? g.ni - 1 : iv;
  const double u = 2.0 * (y - iv) - 1.0;
  const double* c = g.wpoly + iv * (g.deg + 1);
  double v = c[g.deg];
  for (int k = g.deg - 1; k >= 0; --k) v = fma(v, u, c[k]);
  return v;
}

// the w grid points of one axis whose support holds position x in [0, 1):
// first index (may be negative: wrapped by the caller) and the weights
__device__ __forceinline__ int ew_weights(const EwGrid& g, double x, double* wt) {
  const double s = x * g.inv_h;
  const int j0 = (int)ceil(s - 0.5 * g.w);
  for (int k = 0; k < g.w; ++k) wt[k] = ew_phi(g, fabs(((j0 + k) - s) * g.h * g.inv_alpha));
  return j0;
}

__device__ __forceinline__ int ew_wrap(int j, int n) { return j < 0 ? j + n : (j >= n ? j - n : j); }

constexpr int kEwMaxW = 16;

// one thread per source, sources in Morton order (neighbouring threads touch
// neighbouring grid lines); double atomics into the grid
__global__ void k_ew_spread(EwGrid g, int n, const double* __restrict__ spts, const double* __restrict__ sstr,
                            double* __restrict__ grid) {
  const int M = g.Mg;
  const size_t M3 = (size_t)M * M * M;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double wx[kEwMaxW], wy[kEwMaxW], wz[kEwMaxW];
    const int jx = ew_weights(g, spts[i] + 0.5, wx);
    const int jy = ew_weights(g, spts[(size_t)n + i] + 0.5, wy);
    const int jz = ew_weights(g, spts[2 * (size_t)n + i] + 0.5, wz);
    const double f0 = sstr[i], f1 = sstr[(size_t)n + i], f2 = sstr[2 * (size_t)n + i];
    for (int kz = 0; kz < g.w; ++kz) {
      const size_t oz = (size_t)ew_wrap(jz + kz, M) * M;
      for (int ky = 0; ky < g.w; ++ky) {
        const double wzy = wz[kz] * wy[ky];
        const size_t oy = (oz + ew_wrap(jy + ky, M)) * M;
        for (int kx = 0; kx < g.w; ++kx) {
          const double v = wzy * wx[kx];
          const size_t o = oy + ew_wrap(jx + kx, M);
          atomicAdd(grid + o, v * f0);
          atomicAdd(grid + M3 + o, v * f1);
          atomicAdd(grid + 2 * M3 + o, v * f2);
        }
      }
    }
  }
}

// half spectrum [3][M][M][M/2 + 1]: b = A (k^2 g - k (k.g)) D^2, zero outside the band and at kappa = 0
__global__ void k_ew_symbol(EwGrid g, double2* __restrict__ spec, const double* __restrict__ A,
                            const double* __restrict__ dfac) {
  const int M = g.Mg, MH = M / 2 + 1;
  const size_t S = (size_t)M * M * MH;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < S; e += (size_t)gridDim.x * blockDim.x) {
    const int ix = (int)(e % MH), iy = (int)((e / MH) % M), iz = (int)(e / ((size_t)MH * M));
    const int kx = ix, ky = iy <= M / 2 ? iy : iy - M, kz = iz <= M / 2 ? iz : iz - M;
    const int ax = kx, ay = ky < 0 ? -ky : ky, az = kz < 0 ? -kz : kz;
    const long s2 = (long)kx * kx + (long)ky * ky + (long)kz * kz;
    double2* p0 = spec + e;
    double2* p1 = spec + S + e;
    double2* p2 = spec + 2 * S + e;
    if (s2 == 0 || ax > g.kmax || ay > g.kmax || az > g.kmax || s2 > g.s2max) {
      *p0 = *p1 = *p2 = make_double2(0.0, 0.0);
      continue;
    }
    const double D = dfac[ax] * dfac[ay] * dfac[az];
    const double a = A[s2] * D * D;
    const double k0 = (2.0 * dev::kPI) * kx, k1 = (2.0 * dev::kPI) * ky, k2 = (2.0 * dev::kPI) * kz;
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    const double2 f0 = *p0, f1 = *p1, f2 = *p2;
    const double dr = k0 * f0.x + k1 * f1.x + k2 * f2.x, di = k0 * f0.y + k1 * f1.y + k2 * f2.y;
    *p0 = make_double2(a * (kk * f0.x - k0 * dr), a * (kk * f0.y - k0 * di));
    *p1 = make_double2(a * (kk * f1.x - k1 * dr), a * (kk * f1.y - k1 * di));
    *p2 = make_double2(a * (kk * f2.x - k2 * dr), a * (kk * f2.y - k2 * di));
  }
}

// one thread per target (Morton order), written to caller order
__global__ void k_ew_gather(EwGrid g, int n, const double* __restrict__ tpts, const int* __restrict__ tperm,
                            const double* __restrict__ grid, double* __restrict__ u) {
  const int M = g.Mg;
  const size_t M3 = (size_t)M * M * M;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double wx[kEwMaxW], wy[kEwMaxW], wz[kEwMaxW];
    const int jx = ew_weights(g, tpts[i] + 0.5, wx);
    const int jy = ew_weights(g, tpts[(size_t)n + i] + 0.5, wy);
    const int jz = ew_weights(g, tpts[2 * (size_t)n + i] + 0.5, wz);
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    for (int kz = 0; kz < g.w; ++kz) {
      const size_t oz = (size_t)ew_wrap(jz + kz, M) * M;
      for (int ky = 0; ky < g.w; ++ky) {
        const double wzy = wz[kz] * wy[ky];
        const size_t oy = (oz + ew_wrap(jy + ky, M)) * M;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int kx = 0; kx < g.w; ++kx) {
          const size_t o = oy + ew_wrap(jx + kx, M);
          s0 = fma(wx[kx], grid[o], s0);
          s1 = fma(wx[kx], grid[M3 + o], s1);
          s2 = fma(wx[kx], grid[2 * M3 + o], s2);
        }
        u0 = fma(wzy, s0, u0);
        u1 = fma(wzy, s1, u1);
        u2 = fma(wzy, s2, u2);
      }
    }
    double* ut = u + (size_t)tperm[i] * 3;
    ut[0] = u0;
    ut[1] = u1;
    ut[2] = u2;
  }
}

// cell boundaries of Morton-sorted quantized points at level L (3D):
// bnd[c] = first point with cell >= c, c = 0..8^L
__global__ void k_cell_bounds(int n, const int32_t* __restrict__ q, int L, int ncell, int* __restrict__ bnd) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncell; c += gridDim.x * blockDim.x) {
    int lo = 0, hi = n;  // first i with cell(i) >= c
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      int cm = 0;
      const int sh = 30 - L;
      const int x = q[mid] >> sh, y = q[(size_t)n + mid] >> sh, z = q[2 * (size_t)n + mid] >> sh;
      for (int b = L - 1; b >= 0; --b) cm = (cm << 3) | (((z >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((x >> b) & 1);
      if (cm < c) lo = mid + 1;
      else hi = mid;
    }
    bnd[c] = lo;
  }
}

int grid_for_n(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_ew_spread(const EwGrid& g, int n, const double* spts, const double* sstr, double* grid, cudaStream_t st) {
  if (n <= 0) return;
  k_ew_spread<<<grid_for_n(n, 128), 128, 0, st>>>(g, n, spts, sstr, grid);
}

void launch_ew_symbol(const EwGrid& g, double2* spec, const double* A, const double* dfac, cudaStream_t st) {
  const size_t S = (size_t)g.Mg * g.Mg * (g.Mg / 2 + 1);
  k_ew_symbol<<<grid_for_n(S, 256), 256, 0, st>>>(g, spec, A, dfac);
}

void launch_ew_gather(const EwGrid& g, int n, const double* tpts, const int* tperm, const double* grid, double* u,
                      cudaStream_t st) {
  if (n <= 0) return;
  k_ew_gather<<<grid_for_n(n, 128), 128, 0, st>>>(g, n, tpts, tperm, grid, u);
}

void launch_cell_bounds(int n, const int32_t* q, int L, int* bnd, cudaStream_t st) {
  const int ncell = 1 << (3 * L);
  k_cell_bounds<<<grid_for_n((size_t)ncell + 1, 256), 256, 0, st>>>(n, q, L, ncell, bnd);
}

}  // namespace sdmkb
