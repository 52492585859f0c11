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

// the three component grids interleaved per point, (g0, g1) | (g2, pad), so
// the gather reads one 16-byte and one 8-byte value per grid point instead
// of three 8-byte values from three arrays
__global__ void k_ew_interleave(size_t M3, const double* __restrict__ grid, double4* __restrict__ gi) {
  for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < M3; o += (size_t)gridDim.x * blockDim.x)
    gi[o] = make_double4(grid[o], grid[M3 + o], grid[2 * M3 + o], 0.0);
}

// one thread per target (Morton order: neighbouring threads share stencil
// lines in L1), written to caller order
__global__ void k_ew_gather(EwGrid g, int n, const double* __restrict__ tpts, const int* __restrict__ tperm,
                            const double4* __restrict__ gi, double* __restrict__ u) {
  const int M = g.Mg;
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
        const double4* row = gi + (oz + ew_wrap(jy + ky, M)) * M;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int kx = 0; kx < g.w; ++kx) {
          const double2* pv = reinterpret_cast<const double2*>(row + ew_wrap(jx + kx, M));
          const double2 a = __ldg(pv);
          const double c = __ldg(reinterpret_cast<const double*>(pv + 1));
          s0 = fma(wx[kx], a.x, s0);
          s1 = fma(wx[kx], a.y, s1);
          s2 = fma(wx[kx], c, s2);
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

// ---- deterministic spreading and interpolation (no atomics) ---------------
// The Morton-sorted points are binned by cells at level Lc (side cs ~ 8 grid
// points; bnd[c] = first point of cell c in Morton order).
__device__ __forceinline__ int ew_cell(int cx, int cy, int cz, int Lc) {  // Morton index, x fastest
  int c = 0;
  for (int b = 0; b < Lc; ++b) c |= (((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2)) << (3 * b);
  return c;
}
__device__ __forceinline__ int ew_mod(int a, int m) { a %= m; return a < 0 ? a + m : a; }

// Spreading, output-stationary: one CTA per 16^3 brick of the grid, one
// thread per (x, y) column of the brick holding its 16 z values.  The CTA
// walks the cells whose points can reach the brick (cell order, then Morton
// order), stages each batch of points that do (first grid index per axis,
// the w window weights per axis, the strength), and every thread adds the
// batch into its column in that order: each grid value is one thread's
// fixed-order sum, written once (no atomics, no zeroing of the grid,
// bitwise reproducible).  A stencil's z range is the same for every column,
// so the z loop is unrolled with one predicate per row.
constexpr int kEwTB = 16, kEwSB = 64;
__global__ void __launch_bounds__(256) k_ew_spread2(EwGrid g, int Lc, const int* __restrict__ bnd,
                                                    const double* __restrict__ spts, int n,
                                                    const double* __restrict__ sstr, double* __restrict__ grid) {
  __shared__ double s_w[kEwSB][3][kEwMaxW];
  __shared__ double s_f[kEwSB][3];
  __shared__ double s_d0[kEwSB][3];
  __shared__ int s_j0[kEwSB][3];
  __shared__ int s_wp[2], s_n, s_cell[64];
  const int M = g.Mg, w = g.w, nbk = (M + kEwTB - 1) / kEwTB;
  const size_t M3 = (size_t)M * M * M;
  const int b = blockIdx.x, bx = b % nbk, by = (b / nbk) % nbk, bz = b / (nbk * nbk);
  const int b0[3] = {bx * kEwTB, by * kEwTB, bz * kEwTB};
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int gx = b0[0] + tx, gy = b0[1] + ty;
  double acc[kEwTB][3];
#pragma unroll
  for (int k = 0; k < kEwTB; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
  // cells that can hold a point reaching the brick: x M in (b0 - w/2, b0 + 15 + w/2]
  const int nc = 1 << Lc;
  const double cs = (double)M / nc;
  int ncell = 0;
  if (tid == 0) {
    int clo[3], ccnt[3];
    for (int a = 0; a < 3; ++a) {
      clo[a] = (int)floor((b0[a] - 0.5 * w - 1e-6) / cs);  // (margin: a point on a cell boundary)
      const int chi = (int)floor((b0[a] + kEwTB - 1 + 0.5 * w + 1e-6) / cs);
      ccnt[a] = min(chi - clo[a] + 1, nc);
    }
    for (int kz = 0; kz < ccnt[2]; ++kz)
      for (int ky = 0; ky < ccnt[1]; ++ky)
        for (int kx = 0; kx < ccnt[0]; ++kx)
          s_cell[ncell++] = ew_cell(ew_mod(clo[0] + kx, nc), ew_mod(clo[1] + ky, nc), ew_mod(clo[2] + kz, nc), Lc);
    s_n = ncell;
  }
  __syncthreads();
  ncell = s_n;
  for (int ci = 0; ci < ncell; ++ci) {
    const int c = s_cell[ci];
    const int p0 = bnd[c], p1 = bnd[c + 1];
    for (int base = p0; base < p1; base += kEwSB) {
      __syncthreads();  // the previous batch is consumed
      // filter: the points of this batch whose stencil meets the brick, compacted in order
      bool keep = false;
      int j0[3] = {0, 0, 0};
      double d0[3] = {0.0, 0.0, 0.0};
      const int pi = base + tid;
      if (tid < kEwSB && pi < p1) {
        keep = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double sx = (spts[(size_t)a * n + pi] + 0.5) * g.inv_h;
          const int ju = (int)ceil(sx - 0.5 * w);  // first grid index of the stencil (unwrapped)
          d0[a] = ju - sx;
          j0[a] = ew_mod(ju, M);
          const int dd = ew_mod(b0[a] - j0[a], M);  // brick start relative to the stencil start
          keep = keep && (dd < w || dd > M - kEwTB);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);  // order-preserving compaction
      if ((tid & 31) == 0 && tid < kEwSB) s_wp[tid >> 5] = __popc(bal);
      __syncthreads();
      const int off = (tid >= 32 ? s_wp[0] : 0) + __popc(bal & ((1u << (tid & 31)) - 1u));
      const int np = s_wp[0] + s_wp[1];
      if (keep) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          s_j0[off][a] = j0[a];
          s_d0[off][a] = d0[a];
          s_f[off][a] = sstr[(size_t)a * n + pi];
        }
      }
      __syncthreads();
      if (np == 0) continue;
      for (int e = tid; e < np * 3 * kEwMaxW; e += blockDim.x) {  // weights: (point, axis, k)
        const int q = e / (3 * kEwMaxW), r = e - q * 3 * kEwMaxW, a = r / kEwMaxW, k = r - a * kEwMaxW;
        s_w[q][a][k] = k < w ? ew_phi(g, fabs((s_d0[q][a] + k) * g.h * g.inv_alpha)) : 0.0;
      }
      __syncthreads();
      for (int q = 0; q < np; ++q) {
        int ox = gx - s_j0[q][0], oy = gy - s_j0[q][1];
        ox += ox < 0 ? M : 0;
        oy += oy < 0 ? M : 0;
        if (ox >= w || oy >= w) continue;
        const double wxy = s_w[q][0][ox] * s_w[q][1][oy];
        const double f0 = wxy * s_f[q][0], f1 = wxy * s_f[q][1], f2 = wxy * s_f[q][2];
        // row k of the brick is stencil row k - dz (dz in (-w, 16) after unwrapping)
        int dz = s_j0[q][2] - b0[2];
        dz += dz <= -w ? M : 0;
        dz -= dz >= kEwTB ? M : 0;
        const double* wz = s_w[q][2];
#pragma unroll
        for (int k = 0; k < kEwTB; ++k) {
          const int oz = k - dz;
          if (oz >= 0 && oz < w) {
            const double v = wz[oz];
            acc[k][0] = fma(v, f0, acc[k][0]);
            acc[k][1] = fma(v, f1, acc[k][1]);
            acc[k][2] = fma(v, f2, acc[k][2]);
          }
        }
      }
    }
  }
  if (gx < M && gy < M) {
#pragma unroll
    for (int k = 0; k < kEwTB; ++k) {
      const int gz = b0[2] + k;
      if (gz < M) {
        const size_t o = ((size_t)gz * M + gy) * M + gx;
        grid[o] = acc[k][0];
        grid[M3 + o] = acc[k][1];
        grid[2 * M3 + o] = acc[k][2];
      }
    }
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

// a stencil meets a brick in one run of rows (no double wrap) when Mg >= 16 + w
bool ew_spread_tiled_ok(const EwGrid& g, int Lc) {
  return g.w <= kEwTB && g.w <= kEwMaxW && Lc <= 7 && g.Mg >= kEwTB + g.w;
}

void launch_ew_spread_tiled(const EwGrid& g, int Lc, const int* bnd, int n, const double* spts, const double* sstr,
                            double* grid, cudaStream_t st) {
  const int nbk = (g.Mg + kEwTB - 1) / kEwTB;
  k_ew_spread2<<<nbk * nbk * nbk, 256, 0, st>>>(g, Lc, bnd, spts, n, sstr, grid);
}

void launch_ew_symbol(const EwGrid& g, double2* spec, const double* A, const double* dfac, cudaStream_t st) {
  const size_t S = (size_t)g.Mg * g.Mg * (g.Mg / 2 + 1);
  k_ew_symbol<<<grid_for_n(S, 256), 256, 0, st>>>(g, spec, A, dfac);
}

void launch_ew_gather(const EwGrid& g, int n, const double* tpts, const int* tperm, const double* grid, void* gi,
                      double* u, cudaStream_t st) {
  if (n <= 0) return;
  const size_t M3 = (size_t)g.Mg * g.Mg * g.Mg;
  double4* g4 = reinterpret_cast<double4*>(gi);
  k_ew_interleave<<<grid_for_n(M3, 256), 256, 0, st>>>(M3, grid, g4);
  k_ew_gather<<<grid_for_n(n, 128), 128, 0, st>>>(g, n, tpts, tperm, g4, u);
}

void launch_cell_bounds(int n, const int32_t* q, int L, int* bnd, cudaStream_t st) {
  const int ncell = 1 << (3 * L);
  k_cell_bounds<<<grid_for_n((size_t)ncell + 1, 256), 256, 0, st>>>(n, q, L, ncell, bnd);
}

}  // namespace sdmkb
