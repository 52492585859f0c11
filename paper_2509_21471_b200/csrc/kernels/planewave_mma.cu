// Plane-wave transforms (K5 forward, K8 inverse; dmk.cpp:166-243) on the FP64
// tensor cores, 3D.  Same half-spectrum / band-compressed layout as
// planewave.cu; the four stages become dense DMMA GEMMs (complex products as
// real GEMMs with the K dimension doubled over (index, re/im)):
//
//  fwd_xy : per (box, ch), four z-slabs at a time (cp.async double buffered)
//           X  a[(s,iy), (m0,re|im)] = w[(s,iy), ix] * EX[ix, (m0,re|im)]
//           Y  b[s][my, m0]          = E[my, iy] a[s][iy, m0]   (complex)
//           -> B[box][ch][iz][col] for the in-band columns (my, m0)
//  fwd_z  : per (box, ch, 64-column block)
//           G[mz, col] = E[mz, iz] B[iz, col]                    (complex)
//  inv_z  : per (box, j, 64-column block)
//           C1[iz, col] = conj(E)[mz, iz]^T F[mz, col]           (complex)
//  inv_xy : per (box, j), four slabs at a time
//           Y  d[(s,iy), m0] = conj(E)[my, iy]^T C1[s][(my, m0)] (complex)
//           X  out[(s,iy), ix] += pf * sum_m0 wt(m0) Re(conj(E)[m0, ix] d)
//
// Fragment-load strides follow the bank rule in anterp_mma.cu (== 4 mod 8 for
// row-indexed operands; the interleaved (index, re|im) B operands use rows of
// stride == 8 mod 16).
#include "common.cuh"
#include "launch.hpp"

#include <algorithm>
#include <cstdlib>

namespace sdmkb {

namespace {

using dev::cp_async8;
using dev::cp_commit;
using dev::cp_wait0;
using dev::cp_wait1;
using dev::dmma;

constexpr int kW = 8;  // warps per CTA

__host__ __device__ constexpr int r4(int x) { return (x + 3) / 4 * 4 % 8 == 4 ? (x + 3) / 4 * 4 : (x + 3) / 4 * 4 + 4; }
__host__ __device__ constexpr int r8(int x) { return (x + 7) / 8 * 8 % 16 == 8 ? (x + 7) / 8 * 8 : (x + 7) / 8 * 8 + 8; }

// ------------------------------------------------------------------ fwd_xy --
// fwd_xy with the Hermitian split of the Y stage.  E[-m] = conj E[m] and
// E[0] = 1, so for m0 >= 1 (complex a = ar + i ai) and my >= 1
//   P = Er ar, Q = Ei ai, R = Er ai, S = Ei ar      (Er, Ei: rows my = 1..M)
//   b[+my] = (P - Q) + i (R + S),   b[-my] = (P + Q) + i (R - S),
// four real GEMMs over M rows instead of one complex GEMM over 2M + 1 rows
// with interleaved K (~3.7x fewer DMMAs).  The my = 0 row (column sums of a)
// and the m0 = 0 column (a real: b[+-my] = P0 +- i S0) are CUDA-core dot
// products.  X stage columns: n = 2 (m0 - 1) + part for m0 = 1..M, n = 2M for
// m0 = 0 (E = 1).
template <int PT, int PC, int NC>
__global__ void __launch_bounds__(kW * 32, 1) k_fwd_xy2(PWGrid g, const int* __restrict__ boxes, int nbox, int nch,
                                                       const double* __restrict__ outgoing,
                                                       double2* __restrict__ B) {
  constexpr int P8 = PT * 8;
  constexpr int SE = P8 + 4;  // == 4 mod 8 for P8 = 24, 32
  constexpr int SY = P8 + 4;
  const int p = PC > 0 ? PC : g.p, N = NC > 0 ? NC : g.N, M = (N - 1) / 2, ncol = g.ncol, pp = p * p;
  const int M1 = M + 1, MT = (M + 7) / 8, M8 = MT * 8, NX8 = (2 * M + 1 + 7) / 8 * 8;
  const int SAa = r8(NX8 > 2 * M8 ? NX8 : 2 * M8);  // Y reads columns up to 2 M8 - 1
  extern __shared__ double sm[];
  double* EXT = sm;                        // [NX8][SE]
  double* EYr = EXT + NX8 * SE;            // [M8][SY]  rows my - 1
  double* EYi = EYr + M8 * SY;             // [M8][SY]
  double* win = EYi + M8 * SY;             // [2][4*P8][SE]
  double* a = win + 2 * 4 * P8 * SE;       // [4*P8][SAa]
  int* colidx = reinterpret_cast<int*>(a + 4 * P8 * SAa);  // [N][M1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  for (int e = tid; e < NX8 * SE; e += blockDim.x) {
    const int n = e / SE, ix = e % SE;
    double v = 0.0;
    if (ix < p) {
      if (n < 2 * M) {
        const double2 ev = g.E[(size_t)(n / 2 + 1 + M) * p + ix];
        v = (n & 1) ? ev.y : ev.x;
      } else if (n == 2 * M) {
        v = 1.0;
      }
    }
    EXT[e] = v;
  }
  for (int e = tid; e < M8 * SY; e += blockDim.x) {
    const int r = e / SY, iy = e % SY;
    double vr = 0.0, vi = 0.0;
    if (r < M && iy < p) {
      const double2 ev = g.E[(size_t)(r + 1 + M) * p + iy];
      vr = ev.x;
      vi = ev.y;
    }
    EYr[e] = vr;
    EYi[e] = vi;
  }
  for (int e = tid; e < N * M1; e += blockDim.x) colidx[e] = -1;
  for (int e = tid; e < 2 * 4 * P8 * SE; e += blockDim.x) win[e] = 0.0;
  for (int e = tid; e < 4 * P8 * SAa; e += blockDim.x) a[e] = 0.0;
  __syncthreads();
  for (int c = tid; c < ncol; c += blockDim.x) colidx[(g.col_my[c] + M) * M1 + g.col_m0[c]] = c;
  // persistent: items (box, channel) with stride gridDim.x, the flattened
  // (item, slab group) sequence keeps the next group's input in flight
  const int ngroups = (p + 3) / 4, nitems = nbox * nch;
  const int nsteps = ((nitems - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * ngroups;
  auto issue = [&](int step, int buf) {
    const int wi = blockIdx.x + (step / ngroups) * gridDim.x, grp = step % ngroups;
    const double* w = outgoing + ((size_t)boxes[wi / nch] * nch + wi % nch) * (size_t)(p * pp);
    double* dst = win + buf * 4 * P8 * SE;
    const int jz0 = grp * 4;
    for (int row = warp; row < 4 * p; row += kW) {
      const int s = row / p, r = row % p;
      const bool v = jz0 + s < p;
      const double* srow = w + (size_t)(v ? jz0 + s : 0) * pp + r * p;
      for (int cc = lane; cc < p; cc += 32) cp_async8(dst + (s * P8 + r) * SE + cc, srow + cc, v);
    }
    cp_commit();
  };
  double2* Bo = B;
  auto put = [&](int iz, int my, int m0, double re, double im) {
    const int c = colidx[(my + M) * M1 + m0];
    if (c >= 0) Bo[(size_t)iz * ncol + c] = make_double2(re, im);
  };
  if (nsteps > 0) issue(0, 0);
  const int nnt = NX8 / 8;
  const int xtiles = 4 * PT * nnt;
  const int yunits = 4 * MT * MT;
  for (int step = 0; step < nsteps; ++step) {
    const int buf = step & 1, grp = step % ngroups;
    Bo = B + (size_t)(blockIdx.x + (step / ngroups) * gridDim.x) * g.pz * ncol;  // (slot, ch) = item
    __syncthreads();
    if (step + 1 < nsteps) {
      issue(step + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    const double* A = win + buf * 4 * P8 * SE;
    // X stage (two tiles per warp iteration: independent chains)
    for (int tile0 = warp; tile0 < xtiles; tile0 += 2 * kW) {
      const int tile1 = tile0 + kW;
      const bool two = tile1 < xtiles;
      const int mA = tile0 / nnt, nA = tile0 % nnt, mB = two ? tile1 / nnt : mA, nB = two ? tile1 % nnt : nA;
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks) {
        dmma(c0, c1, A[(mA * 8 + gq) * SE + ks * 4 + t], EXT[(nA * 8 + gq) * SE + ks * 4 + t]);
        if (two) dmma(d0, d1, A[(mB * 8 + gq) * SE + ks * 4 + t], EXT[(nB * 8 + gq) * SE + ks * 4 + t]);
      }
      a[(mA * 8 + gq) * SAa + nA * 8 + 2 * t] = c0;
      a[(mA * 8 + gq) * SAa + nA * 8 + 2 * t + 1] = c1;
      if (two) {
        a[(mB * 8 + gq) * SAa + nB * 8 + 2 * t] = d0;
        a[(mB * 8 + gq) * SAa + nB * 8 + 2 * t + 1] = d1;
      }
    }
    __syncthreads();
    // Y stage: units (s, my tile, m0 tile), four accumulators each
    for (int u = warp; u < yunits; u += kW) {
      const int s = u / (MT * MT), mt = (u / MT) % MT, nt = u % MT;
      double P0 = 0, P1 = 0, Q0 = 0, Q1 = 0, R0 = 0, R1 = 0, S0 = 0, S1 = 0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks) {
        const int k = ks * 4 + t;
        const double* ar = a + (s * P8 + k) * SAa + 2 * (nt * 8 + gq);
        const double br = ar[0], bi = ar[1];
        const double er = EYr[(mt * 8 + gq) * SY + k], ei = EYi[(mt * 8 + gq) * SY + k];
        dmma(P0, P1, er, br);
        dmma(Q0, Q1, ei, bi);
        dmma(R0, R1, er, bi);
        dmma(S0, S1, ei, br);
      }
      const int my = mt * 8 + gq + 1, iz = grp * 4 + s;
      if (my <= M && iz < p) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m0 = nt * 8 + 2 * t + e + 1;
          if (m0 <= M) {
            const double P = e ? P1 : P0, Q = e ? Q1 : Q0, R = e ? R1 : R0, S = e ? S1 : S0;
            put(iz, my, m0, P - Q, R + S);
            put(iz, -my, m0, P + Q, R - S);
          }
        }
      }
    }
    // remainders on the CUDA cores: the m0 = 0 column (my >= 1) and the my = 0 row
    for (int it = tid; it < 4 * (2 * M + 1); it += blockDim.x) {
      const int s = it / (2 * M + 1), r = it % (2 * M + 1), iz = grp * 4 + s;
      if (iz >= p) continue;
      const double* as = a + s * P8 * SAa;
      if (r < M) {  // my = r + 1, m0 = 0: a real
        double P = 0.0, S = 0.0;
        for (int iy = 0; iy < p; ++iy) {
          const double a0 = as[iy * SAa + 2 * M];
          P = fma(EYr[r * SY + iy], a0, P);
          S = fma(EYi[r * SY + iy], a0, S);
        }
        put(iz, r + 1, 0, P, S);
        put(iz, -(r + 1), 0, P, -S);
      } else {  // my = 0, m0 = r - M
        const int m0 = r - M;
        double re = 0.0, im = 0.0;
        if (m0 == 0) {
          for (int iy = 0; iy < p; ++iy) re += as[iy * SAa + 2 * M];
        } else {
          for (int iy = 0; iy < p; ++iy) {
            re += as[iy * SAa + 2 * (m0 - 1)];
            im += as[iy * SAa + 2 * (m0 - 1) + 1];
          }
        }
        put(iz, 0, m0, re, im);
      }
    }
  }
}

// ------------------------------------------------------------ z stages ----
constexpr int kCB = 64;  // columns per z-stage work item

// z stages with the Hermitian split (E[-m] = conj E[m], E[0] = 1):
//  forward  G[+-mz] = (P -+ Q) + i (R +- S), P = Er Br, Q = Ei Bi, R = Er Bi,
//           S = Ei Br over mz = 1..M; G[0] = sum_iz B (CUDA cores);
//  inverse  C1.re = F[0].re + [Er | Ei] [Ur ; Vi],  C1.im = F[0].im + [Er | -Ei] [Ui ; Vr]
//           with U = F[+mz] + F[-mz], V = F[+mz] - F[-mz] (zero outside the band).
// ~2.5x fewer DMMAs than the complex GEMMs over all 2M + 1 rows.
// Persistent forms: a CTA keeps its E matrices and walks work items
// (box, component, 64-column block) with stride gridDim.x, the next item's
// input arriving by cp.async while the current one is multiplied.
template <int PT>
__global__ void __launch_bounds__(kW * 32, 3) k_zf2(PWGrid g, int nc, int nbox, const double2* __restrict__ IN,
                                                   double2* __restrict__ OUT) {
  constexpr int P8 = PT * 8, SK = P8 + 4;
  constexpr int SI = (2 * kCB) % 16 == 8 ? 2 * kCB : 2 * kCB + 8;
  extern __shared__ double sm[];
  const int M = g.Mz, MT = (M + 7) / 8, M8 = MT * 8, pz = g.pz, ncol = g.ncol;
  double* Ar = sm;               // [M8][SK]  Er[mz = r + 1][iz]
  double* Ai = Ar + M8 * SK;     // [M8][SK]
  double* In = Ai + M8 * SK;     // [2][P8][SI]  (col, re|im) interleaved
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  for (int e = tid; e < M8 * SK; e += blockDim.x) {
    const int r = e / SK, k = e % SK;
    double vr = 0.0, vi = 0.0;
    if (r < M && k < pz) {
      const double2 ev = g.Ez[(size_t)(r + 1 + M) * pz + k];
      vr = ev.x;
      vi = ev.y;
    }
    Ar[e] = vr;
    Ai[e] = vi;
  }
  const int ncbk = (ncol + kCB - 1) / kCB, nitems = nbox * nc * ncbk;
  auto issue = [&](int w, int buf) {
    const int bc = w / ncbk, c0 = (w % ncbk) * kCB, ncb = min(kCB, ncol - c0);
    const double2* src = IN + (size_t)bc * pz * ncol + c0;
    double* dst = In + buf * P8 * SI;
    for (int e = tid; e < P8 * kCB; e += blockDim.x) {
      const int k = e / kCB, cc = e % kCB;
      const bool v = k < pz && cc < ncb;
      dev::cp_async16z(dst + k * SI + 2 * cc, v ? src + (size_t)k * ncol + cc : src, v);
    }
    cp_commit();
  };
  int w = blockIdx.x;
  if (w < nitems) issue(w, 0);
  for (int it = 0; w < nitems; ++it, w += gridDim.x) {
    const int buf = it & 1;
    if (w + (int)gridDim.x < nitems) {
      issue(w + gridDim.x, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    const double* Ib = In + buf * P8 * SI;
    const int bc = w / ncbk, c0 = (w % ncbk) * kCB, ncb = min(kCB, ncol - c0);
    double2* dst = OUT + (size_t)bc * g.nhalf;
    const int ntc = kCB / 8, ntile = MT * ntc;
    for (int tile = warp; tile < ntile; tile += kW) {
      const int rt = tile / ntc, ct = tile % ntc;
      double P0 = 0, P1 = 0, Q0 = 0, Q1 = 0, R0 = 0, R1 = 0, S0 = 0, S1 = 0;
#pragma unroll
      for (int ks = 0; ks < 2 * PT; ++ks) {
        const int k = ks * 4 + t;
        const double br = Ib[k * SI + 2 * (ct * 8 + gq)], bi = Ib[k * SI + 2 * (ct * 8 + gq) + 1];
        const double er = Ar[(rt * 8 + gq) * SK + k], ei = Ai[(rt * 8 + gq) * SK + k];
        dmma(P0, P1, er, br);
        dmma(Q0, Q1, ei, bi);
        dmma(R0, R1, er, bi);
        dmma(S0, S1, ei, br);
      }
      const int mz = rt * 8 + gq + 1;
      if (mz > M) continue;
      const int np = g.slab_ncol[mz + M], nm = g.slab_ncol[M - mz];
      const int op = g.slab_off[mz + M], om = g.slab_off[M - mz];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = ct * 8 + 2 * t + e, col = c0 + cc;
        if (cc >= ncb) continue;
        const double P = e ? P1 : P0, Q = e ? Q1 : Q0, R = e ? R1 : R0, S = e ? S1 : S0;
        if (col < np) dst[op + col] = make_double2(P - Q, R + S);
        if (col < nm) dst[om + col] = make_double2(P + Q, R - S);
      }
    }
    // mz = 0: column sums over iz
    for (int cc = tid; cc < ncb; cc += blockDim.x) {
      const int col = c0 + cc;
      if (col >= g.slab_ncol[M]) continue;
      double re = 0.0, im = 0.0;
      for (int k = 0; k < pz; ++k) {
        re += Ib[k * SI + 2 * cc];
        im += Ib[k * SI + 2 * cc + 1];
      }
      dst[g.slab_off[M] + col] = make_double2(re, im);
    }
    __syncthreads();  // this buffer is refilled by the issue two items ahead
  }
}

template <int PT>
__global__ void __launch_bounds__(kW * 32, 2) k_zi2(PWGrid g, int nc, int nbox, const double2* __restrict__ IN,
                                                   double2* __restrict__ OUT) {
  constexpr int P8 = PT * 8;
  extern __shared__ double sm[];
  const int M = g.Mz, MT = (M + 7) / 8, M8 = MT * 8, K2 = 2 * M8, SA = r4(K2), pz = g.pz, ncol = g.ncol;
  const int NZ = 2 * M + 1;
  double* Are = sm;                  // [P8][SA]  [Er | Ei]
  double* Aim = Are + P8 * SA;       // [P8][SA]  [Er | -Ei]
  constexpr int FR = kCB + 2;        // F row stride (double2): 16-byte fragment loads conflict-free
  double2* Fs = reinterpret_cast<double2*>(Aim + P8 * SA);  // [2][NZ][FR]  raw F rows (mz + M)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  for (int e = tid; e < P8 * SA; e += blockDim.x) {
    const int iz = e / SA, k = e % SA;
    double vr = 0.0, vi = 0.0;
    if (iz < pz && k < K2) {
      const int r = k < M8 ? k : k - M8;
      if (r < M) {
        const double2 ev = g.Ez[(size_t)(r + 1 + M) * pz + iz];
        vr = k < M8 ? ev.x : ev.y;
        vi = k < M8 ? ev.x : -ev.y;
      }
    }
    Are[e] = vr;
    Aim[e] = vi;
  }
  const int ncbk = (ncol + kCB - 1) / kCB, nitems = nbox * nc * ncbk;
  auto issue = [&](int w, int buf) {
    const int bc = w / ncbk, c0 = (w % ncbk) * kCB;
    const double2* src = IN + (size_t)bc * g.nhalf;
    double2* dst = Fs + buf * NZ * FR;
    for (int s = warp; s < NZ; s += kW) {  // a warp per mz row: one band lookup per row
      const int nvalid = g.slab_ncol[s] - c0;
      const double2* row = src + g.slab_off[s] + c0;
      for (int cc = lane; cc < kCB; cc += 32) dev::cp_async16z(dst + s * FR + cc, cc < nvalid ? row + cc : src, cc < nvalid);
    }
    cp_commit();
  };
  int w = blockIdx.x;
  if (w < nitems) issue(w, 0);
  for (int it = 0; w < nitems; ++it, w += gridDim.x) {
    const int buf = it & 1;
    if (w + (int)gridDim.x < nitems) {
      issue(w + gridDim.x, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    const double2* Fb = Fs + buf * NZ * FR;
    const int bc = w / ncbk, c0 = (w % ncbk) * kCB, ncb = min(kCB, ncol - c0);
    double2* dst = OUT + (size_t)bc * pz * ncol;
    // warp w: column tile w, all row (iz) tiles; B' = [U ; V] formed at fragment load
    const int ct = warp;
    double r0[PT], r1[PT], i0[PT], i1[PT];
#pragma unroll
    for (int m = 0; m < PT; ++m) r0[m] = r1[m] = i0[m] = i1[m] = 0.0;
    const int cc_b = ct * 8 + gq;
#pragma unroll 2
    for (int ks = 0; ks < K2 / 4; ++ks) {
      const int k = ks * 4 + t;
      const int r = k < M8 ? k : k - M8;  // mz - 1
      double br = 0.0, bi = 0.0;
      if (r < M) {
        const double2 fp = Fb[(M + 1 + r) * FR + cc_b], fm = Fb[(M - 1 - r) * FR + cc_b];
        if (k < M8) {
          br = fp.x + fm.x;  // Ur
          bi = fp.y + fm.y;  // Ui
        } else {
          br = fp.y - fm.y;  // Vi
          bi = fp.x - fm.x;  // Vr
        }
      }
#pragma unroll
      for (int m = 0; m < PT; ++m) {
        dmma(r0[m], r1[m], Are[(m * 8 + gq) * SA + k], br);
        dmma(i0[m], i1[m], Aim[(m * 8 + gq) * SA + k], bi);
      }
    }
#pragma unroll
    for (int m = 0; m < PT; ++m) {
      const int iz = m * 8 + gq;
      if (iz >= pz) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = ct * 8 + 2 * t + e;
        if (cc >= ncb) continue;
        const double2 f0 = Fb[M * FR + cc];
        dst[(size_t)iz * ncol + c0 + cc] = make_double2((e ? r1[m] : r0[m]) + f0.x, (e ? i1[m] : i0[m]) + f0.y);
      }
    }
    __syncthreads();  // this buffer is refilled by the issue two items ahead
  }
}

// z stages, warp-independent forms (PT = 3, Mz <= 16): the unit of work is
// one (box, channel, 16-column block); every warp walks units with a global
// stride, its input block arriving by cp.async (double buffered), and does
// all 2 x 2 (forward) / 3 x 2 (inverse) output tiles of the block at once,
// so each k-step's fragments feed 12-16 DMMAs.  Block rows have a stride
// == 2 mod 8 complex (16-byte fragment loads of a quarter warp hit distinct
// bank groups).
constexpr int kZB = 16;           // columns per unit
constexpr int kZR = kZB + 2;      // block row stride (complex)
constexpr int kWZF = 12, kWZI = 10;  // warps per CTA

__global__ void __launch_bounds__(kWZF * 32, 1) k_zf3(PWGrid g, int nc, int nbox, const double2* __restrict__ IN,
                                                     double2* __restrict__ OUT) {
  constexpr int PT = 3, P8 = PT * 8, SK = P8 + 4, MTC = 2;
  extern __shared__ double sm[];
  const int M = g.Mz, pz = g.pz, ncol = g.ncol;
  double* Ar = sm;                 // [16][SK]  Er[mz = r + 1][iz]
  double* Ai = Ar + 16 * SK;       // [16][SK]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  double2* Bs = reinterpret_cast<double2*>(Ai + 16 * SK) + (size_t)warp * 2 * P8 * kZR;  // [2][P8][kZR]
  for (int e = tid; e < 16 * SK; e += blockDim.x) {
    const int r = e / SK, k = e % SK;
    double vr = 0.0, vi = 0.0;
    if (r < M && k < pz) {
      const double2 ev = g.Ez[(size_t)(r + 1 + M) * pz + k];
      vr = ev.x;
      vi = ev.y;
    }
    Ar[e] = vr;
    Ai[e] = vi;
  }
  for (int e = lane; e < 2 * P8 * kZR; e += 32) Bs[e] = make_double2(0.0, 0.0);  // rows iz >= pz stay 0
  __shared__ int s_ncol[33], s_off[33];  // slab table (mz + M), read per output element
  __shared__ uint64_t zbar[2 * kWZF];    // per warp: one mbarrier per block buffer
  if (tid < 2 * M + 1) {
    s_ncol[tid] = g.slab_ncol[tid];
    s_off[tid] = g.slab_off[tid];
  }
  if (lane == 0) {
    dev::mbar_init(&zbar[2 * warp], 1);
    dev::mbar_init(&zbar[2 * warp + 1], 1);
    dev::mbar_fence_init();
  }
  dev::fence_proxy_async_smem();  // the zero fill precedes the bulk copies into the same bytes
  __syncthreads();
  const int ncbk = (ncol + kZB - 1) / kZB, total = nbox * nc * ncbk;
  const int nw = gridDim.x * kWZF;
  // a unit's block: pz rows of ncb contiguous complex (16-byte aligned), one
  // 1D TMA bulk copy per row, issued by lanes 0 .. pz - 1 (columns past ncb
  // keep finite stale values; their outputs are not stored)
  auto issue = [&](int u, int buf) {
    const int bc = u / ncbk, c0 = (u % ncbk) * kZB, ncb = min(kZB, ncol - c0);
    if (lane == 0) dev::mbar_expect_tx(&zbar[2 * warp + buf], (uint32_t)(pz * ncb * 16));
    __syncwarp();
    if (lane < pz)
      dev::bulk_g2s(Bs + buf * P8 * kZR + lane * kZR, IN + ((size_t)bc * pz + lane) * ncol + c0, (uint32_t)ncb * 16u,
                    &zbar[2 * warp + buf]);
  };
  int u = blockIdx.x * kWZF + warp;
  if (u < total) issue(u, 0);
  for (int it = 0; u < total; ++it, u += nw) {
    const int buf = it & 1;
    if (u + nw < total) issue(u + nw, buf ^ 1);  // that buffer was released by the previous unit
    dev::mbar_wait(&zbar[2 * warp + buf], (uint32_t)((it >> 1) & 1));
    const double2* Bb = Bs + buf * P8 * kZR;
    const int bc = u / ncbk, c0 = (u % ncbk) * kZB, ncb = min(kZB, ncol - c0);
    double2* dst = OUT + (size_t)bc * g.nhalf;
    double P[MTC][2][2], Q[MTC][2][2], R[MTC][2][2], S[MTC][2][2];
#pragma unroll
    for (int i = 0; i < MTC; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) P[i][j][e] = Q[i][j][e] = R[i][j][e] = S[i][j][e] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2 * PT; ++ks) {
      const int k = ks * 4 + t;
      double er[MTC], ei[MTC];
      double2 b[2];
#pragma unroll
      for (int i = 0; i < MTC; ++i) {
        er[i] = Ar[(i * 8 + gq) * SK + k];
        ei[i] = Ai[(i * 8 + gq) * SK + k];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bb[k * kZR + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < MTC; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(P[i][j][0], P[i][j][1], er[i], b[j].x);
          dmma(Q[i][j][0], Q[i][j][1], ei[i], b[j].y);
          dmma(R[i][j][0], R[i][j][1], er[i], b[j].y);
          dmma(S[i][j][0], S[i][j][1], ei[i], b[j].x);
        }
    }
#pragma unroll
    for (int i = 0; i < MTC; ++i) {
      const int mz = i * 8 + gq + 1;
      if (mz > M) continue;
      const int np = s_ncol[mz + M], nm = s_ncol[M - mz];
      const int op = s_off[mz + M], om = s_off[M - mz];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = j * 8 + 2 * t + e, col = c0 + cc;
          if (cc >= ncb) continue;
          const double p_ = P[i][j][e], q_ = Q[i][j][e], r_ = R[i][j][e], s_ = S[i][j][e];
          if (col < np) dst[op + col] = make_double2(p_ - q_, r_ + s_);
          if (col < nm) dst[om + col] = make_double2(p_ + q_, r_ - s_);
        }
    }
    if (lane < ncb && c0 + lane < s_ncol[M]) {  // mz = 0: column sums over iz
      double re = 0.0, im = 0.0;
      for (int k = 0; k < pz; ++k) {
        re += Bb[k * kZR + lane].x;
        im += Bb[k * kZR + lane].y;
      }
      dst[s_off[M] + c0 + lane] = make_double2(re, im);
    }
    __syncwarp();  // this buffer is refilled by the issue two units ahead
  }
}

__global__ void __launch_bounds__(kWZI * 32, 1) k_zi3(PWGrid g, int nc, int nbox, const double2* __restrict__ IN,
                                                     double2* __restrict__ OUT) {
  constexpr int PT = 3, P8 = PT * 8, M8 = 16, K2 = 2 * M8, SA = 36;  // SA = r4(K2)
  extern __shared__ double sm[];
  const int M = g.Mz, pz = g.pz, ncol = g.ncol, NZ = 2 * M + 1;
  double* Are = sm;              // [P8][SA]  [Er | Ei]
  double* Aim = Are + P8 * SA;   // [P8][SA]  [Er | -Ei]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  double2* Fs = reinterpret_cast<double2*>(Aim + P8 * SA) + (size_t)warp * 2 * 33 * kZR;  // [2][NZ <= 33][kZR]
  for (int e = tid; e < P8 * SA; e += blockDim.x) {
    const int iz = e / SA, k = e % SA;
    double vr = 0.0, vi = 0.0;
    if (iz < pz && k < K2) {
      const int r = k < M8 ? k : k - M8;
      if (r < M) {
        const double2 ev = g.Ez[(size_t)(r + 1 + M) * pz + iz];
        vr = k < M8 ? ev.x : ev.y;
        vi = k < M8 ? ev.x : -ev.y;
      }
    }
    Are[e] = vr;
    Aim[e] = vi;
  }
  __shared__ int s_ncol[33], s_off[33];  // slab table (mz + M), read per input element
  __shared__ uint64_t zbar[2 * kWZI];    // per warp: one mbarrier per block buffer
  if (tid < NZ) {
    s_ncol[tid] = g.slab_ncol[tid];
    s_off[tid] = g.slab_off[tid];
  }
  for (int e = lane; e < 2 * 33 * kZR; e += 32) Fs[e] = make_double2(0.0, 0.0);
  if (lane == 0) {
    dev::mbar_init(&zbar[2 * warp], 1);
    dev::mbar_init(&zbar[2 * warp + 1], 1);
    dev::mbar_fence_init();
  }
  dev::fence_proxy_async_smem();  // the zero fill precedes the bulk copies into the same bytes
  __syncthreads();
  const int ncbk = (ncol + kZB - 1) / kZB, total = nbox * nc * ncbk;
  const int nw = gridDim.x * kWZI;
  // a unit's block: F row (mz + M) holds a contiguous prefix of the columns,
  // so each row is one 1D TMA bulk copy of its in-band part (a lane per row);
  // reads of out-of-band entries are predicated to zero instead of zero-filled
  auto issue = [&](int u, int buf) {
    const int bc = u / ncbk, c0 = (u % ncbk) * kZB;
    const double2* src = IN + (size_t)bc * g.nhalf;
    for (int s = lane; s < NZ; s += 32) {
      const int nv = min(kZB, s_ncol[s] - c0);
      if (nv > 0) {
        dev::mbar_expect_tx_only(&zbar[2 * warp + buf], (uint32_t)nv * 16u);
        dev::bulk_g2s(Fs + buf * 33 * kZR + s * kZR, src + s_off[s] + c0, (uint32_t)nv * 16u, &zbar[2 * warp + buf]);
      }
    }
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(&zbar[2 * warp + buf]);
  };
  int u = blockIdx.x * kWZI + warp;
  if (u < total) issue(u, 0);
  for (int it = 0; u < total; ++it, u += nw) {
    const int buf = it & 1;
    if (u + nw < total) issue(u + nw, buf ^ 1);  // that buffer was released by the previous unit
    dev::mbar_wait(&zbar[2 * warp + buf], (uint32_t)((it >> 1) & 1));
    const double2* Fb = Fs + buf * 33 * kZR;
    const int bc = u / ncbk, c0 = (u % ncbk) * kZB, ncb = min(kZB, ncol - c0);
    double2* dst = OUT + (size_t)bc * pz * ncol;
    double re[PT][2][2], im[PT][2][2];
#pragma unroll
    for (int i = 0; i < PT; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) re[i][j][0] = re[i][j][1] = im[i][j][0] = im[i][j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < K2 / 4; ++ks) {
      const int k = ks * 4 + t;
      const bool vpart = k >= M8;
      const int r = vpart ? k - M8 : k;  // mz - 1
      double br[2], bi[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double2 fp = make_double2(0.0, 0.0), fm = fp;
        if (r < M) {
          const int col = c0 + j * 8 + gq;
          if (col < s_ncol[M + 1 + r]) fp = Fb[(M + 1 + r) * kZR + j * 8 + gq];
          if (col < s_ncol[M - 1 - r]) fm = Fb[(M - 1 - r) * kZR + j * 8 + gq];
        }
        br[j] = vpart ? fp.y - fm.y : fp.x + fm.x;  // Vi | Ur
        bi[j] = vpart ? fp.x - fm.x : fp.y + fm.y;  // Vr | Ui
      }
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const double ar = Are[(i * 8 + gq) * SA + k], ai = Aim[(i * 8 + gq) * SA + k];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma(re[i][j][0], re[i][j][1], ar, br[j]);
          dmma(im[i][j][0], im[i][j][1], ai, bi[j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      const int iz = i * 8 + gq;
      if (iz >= pz) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = j * 8 + 2 * t + e;
          if (cc >= ncb) continue;
          const double2 f0 = Fb[M * kZR + cc];
          dst[(size_t)iz * ncol + c0 + cc] = make_double2(re[i][j][e] + f0.x, im[i][j][e] + f0.y);
        }
    }
    __syncwarp();  // this buffer is refilled by the issue two units ahead
  }
}

// ------------------------------------------------------------------ inv_xy --
// 16 warps; the compressed C1 rows of the next four slabs arrive by cp.async
// (double buffered) and feed the Y-stage B fragments directly through the
// (my, m0) -> column table (zero outside the band); each warp's X-stage
// outputs are loaded from HBM at the start of the group so the read of the
// incoming proxies overlaps the Y stage.
constexpr int kWI = 16;

template <int PT, int PC, int NC>
__global__ void __launch_bounds__(kWI * 32, 1) k_inv_xy_mma(PWGrid g, const int* __restrict__ tboxes, int d,
                                                           const double2* __restrict__ C, double pf,
                                                           double* __restrict__ incoming) {
  constexpr int P8 = PT * 8;
  constexpr int XTW = (4 * PT * PT + kWI - 1) / kWI;  // X tiles per warp
  const int p = PC > 0 ? PC : g.p, N = NC > 0 ? NC : g.N, M = (N - 1) / 2, ncol = g.ncol, pp = p * p;
  const int M1 = M + 1, NY8 = (N + 7) / 8 * 8, M18 = (M1 + 7) / 8 * 8, NX = 2 * M1, NX8 = (NX + 7) / 8 * 8;
  const int SA = r4(2 * NY8);      // A' rows iy, k' = 2 my + part
  const int SX = r4(NX8 > 2 * M18 ? NX8 : 2 * M18);
  const int SC = 2 * ncol;         // staged C1 row (interleaved re, im)
  extern __shared__ double sm[];
  double* Ar = sm;                          // [P8][SA]  conj(E)^T re'
  double* Ai = Ar + P8 * SA;                // [P8][SA]  im'
  double* EXw = Ai + P8 * SA;               // [P8 (ix)][SX]  wt * E.re|im
  double* dd = EXw + P8 * SX;               // [4*P8][SX]
  double* stg = dd + 4 * P8 * SX;           // [2][4][SC]
  int* colidx = reinterpret_cast<int*>(stg + 2 * 4 * SC);  // [NY8][M18]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  for (int e = tid; e < P8 * SA; e += blockDim.x) {  // conj(E)^T: re' = [Er | Ei], im' = [-Ei | Er]
    const int iy = e / SA, kk = e % SA, my = kk >> 1, part = kk & 1;
    double vr = 0.0, vi = 0.0;
    if (iy < p && my < N && kk < 2 * NY8) {
      const double2 ev = g.E[(size_t)my * p + iy];
      vr = part ? ev.y : ev.x;
      vi = part ? ev.x : -ev.y;
    }
    Ar[e] = vr;
    Ai[e] = vi;
  }
  for (int e = tid; e < P8 * SX; e += blockDim.x) {  // Re(conj(E) d) = Er d.re + Ei d.im, weight 1 | 2
    const int ix = e / SX, k = e % SX, m0 = k >> 1, part = k & 1;
    double v = 0.0;
    if (ix < p && m0 < M1) {
      const double2 ev = g.E[(size_t)(m0 + M) * p + ix];
      v = (m0 ? 2.0 : 1.0) * (part ? ev.y : ev.x);
    }
    EXw[e] = v;
  }
  for (int e = tid; e < NY8 * M18; e += blockDim.x) colidx[e] = -1;
  __syncthreads();
  for (int c = tid; c < ncol; c += blockDim.x) colidx[(g.col_my[c] + M) * M18 + g.col_m0[c]] = c;
  const int tb = blockIdx.x, j = blockIdx.y;
  const double2* Ci = C + ((size_t)tb * d + j) * (size_t)g.pz * ncol;
  double* out = incoming + ((size_t)tboxes[tb] * d + j) * (size_t)(p * pp);
  const int ngroups = (p + 3) / 4;
  auto issue = [&](int grp, int buf) {
    double* dst = stg + buf * 4 * SC;
    for (int s = 0; s < 4; ++s) {
      const int iz = grp * 4 + s;
      if (iz >= p) break;
      const double* src = reinterpret_cast<const double*>(Ci + (size_t)iz * ncol);
      for (int e = tid; e < SC; e += blockDim.x) cp_async8(dst + s * SC + e, src + e, true);
    }
    cp_commit();
  };
  issue(0, 0);
  const int nit = PT, nm0 = M18 / 8;
  for (int grp = 0; grp < ngroups; ++grp) {
    const int buf = grp & 1;
    __syncthreads();  // the buffer the next issue overwrites is free
    if (grp + 1 < ngroups) {
      issue(grp + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    // this warp's X-stage outputs: start their HBM reads now
    double o0[XTW], o1[XTW];
#pragma unroll
    for (int i = 0; i < XTW; ++i) {
      o0[i] = o1[i] = 0.0;
      const int tile = warp + kWI * i;
      if (tile < 4 * PT * PT) {
        const int mt = tile / PT, nt = tile % PT;
        const int s = mt / PT, iy = (mt % PT) * 8 + gq, iz = grp * 4 + s, ix = nt * 8 + 2 * t;
        if (iz < p && iy < p) {
          const double* o = out + (size_t)iz * pp + iy * p;
          if (ix < p) o0[i] = o[ix];
          if (ix + 1 < p) o1[i] = o[ix + 1];
        }
      }
    }
    const double* S = stg + buf * 4 * SC;
    // Y stage: d[(s,iy), m0] = sum_{(my,part)} A'[iy][(my,part)] C1[s][col(my, m0)].part
    for (int tile = warp; tile < 4 * nit * nm0; tile += kWI) {
      const int s = tile / (nit * nm0), it = (tile / nm0) % nit, nt = tile % nm0;
      double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
      const int ksteps = NY8 / 2;  // K' = 2*NY8, 4 per step
      const int m0 = nt * 8 + gq;
      for (int ks = 0; ks < ksteps; ++ks) {
        const int kk = ks * 4 + t, my = kk >> 1, part = kk & 1;
        const int cidx = colidx[my * M18 + m0];
        const double bv = cidx >= 0 ? S[s * SC + 2 * cidx + part] : 0.0;
        dmma(cr0, cr1, Ar[(it * 8 + gq) * SA + kk], bv);
        dmma(ci0, ci1, Ai[(it * 8 + gq) * SA + kk], bv);
      }
      const int r = s * P8 + it * 8 + gq;
      const int cbase = 2 * (nt * 8 + 2 * t);
      dd[r * SX + cbase] = cr0;
      dd[r * SX + cbase + 1] = ci0;
      dd[r * SX + cbase + 2] = cr1;
      dd[r * SX + cbase + 3] = ci1;
    }
    __syncthreads();
    // X stage: out[(s,iy), ix] += pf * sum_{(m0,part)} dd[(s,iy)][(m0,part)] EXw[ix][(m0,part)]
#pragma unroll
    for (int i = 0; i < XTW; ++i) {
      const int tile = warp + kWI * i;
      if (tile >= 4 * PT * PT) continue;
      const int mt = tile / PT, nt = tile % PT;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < NX8 / 4; ++ks)
        dmma(c0, c1, dd[(mt * 8 + gq) * SX + ks * 4 + t], EXw[(nt * 8 + gq) * SX + ks * 4 + t]);
      const int s = mt / PT, iy = (mt % PT) * 8 + gq, iz = grp * 4 + s, ix = nt * 8 + 2 * t;
      if (iz < p && iy < p) {
        double* o = out + (size_t)iz * pp + iy * p;
        if (ix < p) o[ix] = o0[i] + pf * c0;
        if (ix + 1 < p) o[ix + 1] = o1[i] + pf * c1;
      }
    }
  }
}

// inv_xy with the Hermitian split of the Y stage.  conj E[+-my] = Er -+ i Ei,
// so with U = C[+my] + C[-my], V = C[+my] - C[-my] (my >= 1)
//   d.re = C[0].re + sum_my Er Ur + Ei Vi,   d.im = C[0].im + sum_my Er Ui - Ei Vr
// -- two real GEMMs with K = 2M (A' = [Er | +-Ei], B' = [U ; V] parts)
// instead of a complex GEMM with K = 2 (2M + 1).  The compressed C1 rows of
// four slabs are scattered by cp.async into dense (my, m0) slabs (zero
// outside the band); a pre-pass forms B'; the m0 = 0 column is a CUDA-core
// dot product.  X stage as before over K = (m0, re|im), m0 = 0..M.
template <int PT, int PC, int NC>
__global__ void __launch_bounds__(kWI * 32, 1) k_inv_xy2(PWGrid g, const int* __restrict__ tboxes, int ntb, int d,
                                                        const double2* __restrict__ C, double pf,
                                                        double* __restrict__ incoming) {
  constexpr int P8 = PT * 8;
  constexpr int XTW = (4 * PT * PT + kWI - 1) / kWI;  // X tiles per warp
  const int p = PC > 0 ? PC : g.p, N = NC > 0 ? NC : g.N, M = (N - 1) / 2, ncol = g.ncol, pp = p * p;
  const int M1 = M + 1, MT = (M + 7) / 8, M8 = MT * 8, K2 = 2 * M8;
  const int SA2 = r4(K2);                    // A' rows iy
  const int SB = (M8 % 16 == 8) ? M8 : M8 + 8;  // B' rows k' (== 8 mod 16)
  const int NXK = (2 * M1 + 3) / 4 * 4;      // X-stage K
  const int SX = r4(NXK);
  const int ND = N * M1;                     // dense slab entries (my + M, m0)
  extern __shared__ double sm[];
  double* Are = sm;                          // [P8][SA2]
  double* Aim = Are + P8 * SA2;              // [P8][SA2]
  double* EXw = Aim + P8 * SA2;              // [P8 (ix)][SX]
  double* dd = EXw + P8 * SX;                // [4*P8][SX]
  double* Bre = dd + 4 * P8 * SX;            // [4][K2][SB]
  double* Bim = Bre + 4 * K2 * SB;           // [4][K2][SB]
  double2* den = reinterpret_cast<double2*>(Bim + 4 * K2 * SB);  // [2][4][ND]
  int* dix = reinterpret_cast<int*>(den + 2 * 4 * ND);            // [ncol]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  for (int e = tid; e < P8 * SA2; e += blockDim.x) {
    const int iy = e / SA2, k = e % SA2;
    double vr = 0.0, vi = 0.0;
    if (iy < p && k < K2) {
      const int myp = k < M8 ? k : k - M8;
      if (myp < M) {
        const double2 ev = g.E[(size_t)(myp + 1 + M) * p + iy];
        vr = k < M8 ? ev.x : ev.y;
        vi = k < M8 ? ev.x : -ev.y;
      }
    }
    Are[e] = vr;
    Aim[e] = vi;
  }
  for (int e = tid; e < P8 * SX; e += blockDim.x) {  // Re(conj(E) d) = Er d.re + Ei d.im, weight 1 | 2
    const int ix = e / SX, k = e % SX, m0 = k >> 1, part = k & 1;
    double v = 0.0;
    if (ix < p && m0 < M1) {
      const double2 ev = g.E[(size_t)(m0 + M) * p + ix];
      v = (m0 ? 2.0 : 1.0) * (part ? ev.y : ev.x);
    }
    EXw[e] = v;
  }
  for (int e = tid; e < 4 * P8 * SX; e += blockDim.x) dd[e] = 0.0;
  for (int e = tid; e < 2 * 4 * ND; e += blockDim.x) den[e] = make_double2(0.0, 0.0);
  for (int e = tid; e < 2 * 4 * K2 * SB; e += blockDim.x) Bre[e] = 0.0;  // Bre and Bim
  for (int c = tid; c < ncol; c += blockDim.x) dix[c] = (g.col_my[c] + M) * M1 + g.col_m0[c];
  __syncthreads();
  // persistent: the CTA walks items (box, component) with stride gridDim.x;
  // the flattened (item, slab group) sequence keeps one group in flight
  const int ngroups = (p + 3) / 4, nitems = ntb * d;
  const int nsteps = ((nitems - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * ngroups;
  auto issue = [&](int step, int buf) {
    const int w = blockIdx.x + (step / ngroups) * gridDim.x, grp = step % ngroups;
    const double2* Ci = C + (size_t)w * g.pz * ncol;
    double2* dst = den + buf * 4 * ND;
    for (int s = 0; s < 4; ++s) {
      const int iz = grp * 4 + s;
      if (iz >= p) break;
      const double2* src = Ci + (size_t)iz * ncol;
      for (int c = tid; c < ncol; c += blockDim.x) dev::cp_async16(dst + s * ND + dix[c], src + c);
    }
    cp_commit();
  };
  if (nsteps > 0) issue(0, 0);
  const int nyu = 4 * PT * MT;  // Y units (s, iy tile, m0 tile)
  for (int step = 0; step < nsteps; ++step) {
    const int buf = step & 1;
    const int w = blockIdx.x + (step / ngroups) * gridDim.x, grp = step % ngroups;
    const int tb = w / d, j = w % d;
    double* out = incoming + ((size_t)tboxes[tb] * d + j) * (size_t)(p * pp);
    __syncthreads();  // the buffer the next issue overwrites is free
    if (step + 1 < nsteps) {
      issue(step + 1, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncthreads();
    // this warp's X-stage outputs: start their HBM reads now
    double o0[XTW], o1[XTW];
#pragma unroll
    for (int i = 0; i < XTW; ++i) {
      o0[i] = o1[i] = 0.0;
      const int tile = warp + kWI * i;
      if (tile < 4 * PT * PT) {
        const int mt = tile / PT, nt = tile % PT;
        const int s = mt / PT, iy = (mt % PT) * 8 + gq, iz = grp * 4 + s, ix = nt * 8 + 2 * t;
        if (iz < p && iy < p) {
          const double* o = out + (size_t)iz * pp + iy * p;
          if (ix < p) o0[i] = o[ix];
          if (ix + 1 < p) o1[i] = o[ix + 1];
        }
      }
    }
    const double2* D = den + buf * 4 * ND;
    // B' = [U ; V] parts for my, m0 = 1..M
    for (int e = tid; e < 4 * M * M; e += blockDim.x) {
      const int s = e / (M * M), r = e % (M * M), myp = r / M, m0p = r % M;
      const double2 cp = D[s * ND + (myp + 1 + M) * M1 + m0p + 1];
      const double2 cm = D[s * ND + (M - myp - 1) * M1 + m0p + 1];
      double* br = Bre + s * K2 * SB;
      double* bi = Bim + s * K2 * SB;
      br[myp * SB + m0p] = cp.x + cm.x;         // Ur
      br[(M8 + myp) * SB + m0p] = cp.y - cm.y;  // Vi
      bi[myp * SB + m0p] = cp.y + cm.y;         // Ui
      bi[(M8 + myp) * SB + m0p] = cp.x - cm.x;  // Vr
    }
    // m0 = 0 column on the CUDA cores (real part only: the X stage weighs the
    // imaginary part by Im E(0, ix) = 0)
    for (int e = tid; e < 4 * p; e += blockDim.x) {
      const int s = e / p, iy = e % p;
      const double2* Ds = D + s * ND;
      double re = Ds[M * M1].x;
      for (int myp = 0; myp < M; ++myp) {
        const double2 cp = Ds[(myp + 1 + M) * M1], cm = Ds[(M - myp - 1) * M1];
        const double er = Are[iy * SA2 + myp], ei = Are[iy * SA2 + M8 + myp];
        re = fma(er, cp.x + cm.x, fma(ei, cp.y - cm.y, re));
      }
      dd[(s * P8 + iy) * SX] = re;
      dd[(s * P8 + iy) * SX + 1] = 0.0;
    }
    __syncthreads();
    // Y stage: d[(s,iy), m0] for m0 = 1..M, plus the my = 0 term
    for (int u = warp; u < nyu; u += kWI) {
      const int s = u / (PT * MT), it = (u / MT) % PT, nt = u % MT;
      double r0 = 0.0, r1 = 0.0, i0 = 0.0, i1 = 0.0;
      const double* br = Bre + s * K2 * SB;
      const double* bi = Bim + s * K2 * SB;
#pragma unroll 4
      for (int ks = 0; ks < K2 / 4; ++ks) {
        const int k = ks * 4 + t;
        dmma(r0, r1, Are[(it * 8 + gq) * SA2 + k], br[k * SB + nt * 8 + gq]);
        dmma(i0, i1, Aim[(it * 8 + gq) * SA2 + k], bi[k * SB + nt * 8 + gq]);
      }
      const int row = s * P8 + it * 8 + gq;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m0 = nt * 8 + 2 * t + e + 1;
        if (m0 <= M) {
          const double2 c0 = D[s * ND + M * M1 + m0];
          dd[row * SX + 2 * m0] = (e ? r1 : r0) + c0.x;
          dd[row * SX + 2 * m0 + 1] = (e ? i1 : i0) + c0.y;
        }
      }
    }
    __syncthreads();
    // X stage: out[(s,iy), ix] += pf * sum_{(m0,part)} dd[(s,iy)][(m0,part)] EXw[ix][(m0,part)]
#pragma unroll
    for (int i = 0; i < XTW; ++i) {
      const int tile = warp + kWI * i;
      if (tile >= 4 * PT * PT) continue;
      const int mt = tile / PT, nt = tile % PT;
      double c0 = 0.0, c1 = 0.0;
      for (int ks = 0; ks < NXK / 4; ++ks)
        dmma(c0, c1, dd[(mt * 8 + gq) * SX + ks * 4 + t], EXw[(nt * 8 + gq) * SX + ks * 4 + t]);
      const int s = mt / PT, iy = (mt % PT) * 8 + gq, iz = grp * 4 + s, ix = nt * 8 + 2 * t;
      if (iz < p && iy < p) {
        double* o = out + (size_t)iz * pp + iy * p;
        if (ix < p) o[ix] = o0[i] + pf * c0;
        if (ix + 1 < p) o[ix + 1] = o1[i] + pf * c1;
      }
    }
  }
}

// fwd_xy, warp-independent form (3D, p <= 24, N <= 33): the unit of work is
// one (box, channel, z-slab); every warp walks units with a global stride,
// its w slab arriving by one 1D TMA bulk copy (per-warp mbarriers, double
// buffered), and needs no CTA barrier.  X stage with all PT x NX tiles register-blocked (a k-step loads
// PT + NX fragments for PT NX DMMAs), then the Hermitian-split Y stage
// (P = Er ar, Q = Ei ai, R = Er ai, S = Ei ar; b[+-my] = (P -+ Q) + i (R +- S))
// with all 2 x 2 tiles of the four products at once, the my = 0 row and the
// m0 = 0 column on the CUDA cores, and the in-band columns stored to B.
// warps per CTA: 8 when the shared memory holds them (~27 KB per warp with
// the staged B row), else 7
constexpr int kWF3 = 8;

template <int PC, int NC, int WF>
__global__ void __launch_bounds__(WF * 32, 1) k_fwd_xy3(PWGrid g, const int* __restrict__ boxes, int nbox, int nch,
                                                         const double* __restrict__ outgoing,
                                                         double2* __restrict__ B) {
  constexpr int PT = 3, MTC = 2, P8 = PT * 8, SE = P8 + 4, SY = P8 + 4, NXT = 5;  // NX8 = 40 columns
  const int p = PC > 0 ? PC : g.p, N = NC > 0 ? NC : g.N, M = (N - 1) / 2, ncol = g.ncol, pp = p * p;
  const int M1 = M + 1, M8 = MTC * 8, NX8 = NXT * 8;
  constexpr int SA = 20;  // X outputs by (m0 - 1 | M for m0 = 0) in separate re / im arrays, == 4 mod 8
  extern __shared__ double sm[];
  double* EXT = sm;                   // [NX8][SE]
  double* EYr = EXT + NX8 * SE;       // [M8][SY]  rows my - 1
  double* EYi = EYr + M8 * SY;        // [M8][SY]
  short* colidx = reinterpret_cast<short*>(EYi + M8 * SY);  // [N][M1]
  double* wbase = EYi + M8 * SY + (N * M1 + 7) / 8 * 2;
  const int per_warp = 2 * P8 * SE + 2 * P8 * SA + 2 * ((ncol + 1) / 2 * 2);  // doubles (the staged row even)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  double* win = wbase + warp * per_warp;  // [2][P8][SE]
  double* ar = win + 2 * P8 * SE;         // [P8][SA]  X output, real parts
  double* ai = ar + P8 * SA;              // [P8][SA]  imaginary parts
  double2* stg = reinterpret_cast<double2*>(ai + P8 * SA);  // [ncol] this unit's B row
  for (int e = tid; e < NX8 * SE; e += blockDim.x) {
    const int n = e / SE, ix = e % SE;
    double v = 0.0;
    if (ix < p) {
      if (n < 2 * M) {
        const double2 ev = g.E[(size_t)(n / 2 + 1 + M) * p + ix];
        v = (n & 1) ? ev.y : ev.x;
      } else if (n == 2 * M) {
        v = 1.0;
      }
    }
    EXT[e] = v;
  }
  for (int e = tid; e < M8 * SY; e += blockDim.x) {
    const int r = e / SY, iy = e % SY;
    double vr = 0.0, vi = 0.0;
    if (r < M && iy < p) {
      const double2 ev = g.E[(size_t)(r + 1 + M) * p + iy];
      vr = ev.x;
      vi = ev.y;
    }
    EYr[e] = vr;
    EYi[e] = vi;
  }
  for (int e = tid; e < N * M1; e += blockDim.x) colidx[e] = -1;
  __shared__ uint64_t wbar[2 * WF];  // per warp: one mbarrier per w buffer
  for (int e = lane; e < per_warp; e += 32) win[e] = 0.0;
  if (lane == 0) {
    dev::mbar_init(&wbar[2 * warp], 1);
    dev::mbar_init(&wbar[2 * warp + 1], 1);
    dev::mbar_fence_init();
  }
  dev::fence_proxy_async_smem();  // the zero fill precedes the bulk copies into the same bytes
  __syncthreads();
  for (int c = tid; c < ncol; c += blockDim.x) colidx[(g.col_my[c] + M) * M1 + g.col_m0[c]] = (short)c;
  __syncthreads();
  const int total = nbox * nch * p;
  const int nw = gridDim.x * WF;
  // a unit's w slab (p x p contiguous doubles) arrives by one 1D TMA bulk copy
  // from the 16-byte boundary at or below its start (sh = 1 leading double)
  // into a flat [iy][ix] copy; fragment reads of the padding are predicated
  auto slab = [&](int u) {
    const int item = u / p, iz = u % p;
    return outgoing + ((size_t)boxes[item / nch] * nch + item % nch) * (size_t)(p * pp) + (size_t)iz * pp;
  };
  auto issue = [&](int u, int buf) {  // lane 0
    const double* src = slab(u);
    const int sh = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
    const uint32_t bytes = (uint32_t)(((pp + sh) * 8 + 15) & ~15);
    dev::mbar_expect_tx(&wbar[2 * warp + buf], bytes);
    dev::bulk_g2s(win + buf * P8 * SE, src - sh, bytes, &wbar[2 * warp + buf]);
  };
  bool va[PT], vk[PT * 2];  // this lane's fragment rows (iy) and columns (ix) inside the slab
#pragma unroll
  for (int i = 0; i < PT; ++i) va[i] = i * 8 + gq < p;
#pragma unroll
  for (int ks = 0; ks < PT * 2; ++ks) vk[ks] = ks * 4 + t < p;
  int u = blockIdx.x * WF + warp;
  if (u < total && lane == 0) issue(u, 0);
  for (int k = 0; u < total; ++k, u += nw) {
    const int buf = k & 1;
    if (u + nw < total && lane == 0) issue(u + nw, buf ^ 1);  // that buffer was released by the previous unit
    dev::mbar_wait(&wbar[2 * warp + buf], (uint32_t)((k >> 1) & 1));
    const int item = u / p, iz = u % p;
    double2* Bo = B + (size_t)item * g.pz * ncol + (size_t)iz * ncol;
    const double* A = win + buf * P8 * SE + ((reinterpret_cast<uintptr_t>(slab(u)) >> 3) & 1);
    // X stage: (ar + i ai)[iy][m0'] = sum_ix w[iy][ix] EXT[2 m0' + part][ix]
    {
      double c[PT][NXT][2];
#pragma unroll
      for (int i = 0; i < PT; ++i)
#pragma unroll
        for (int j = 0; j < NXT; ++j) c[i][j][0] = c[i][j][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks) {
        double av[PT], bv[NXT];
#pragma unroll
        for (int i = 0; i < PT; ++i) {
          av[i] = A[(i * 8 + gq) * p + ks * 4 + t];
          if ((PC == 0 || (i == PT - 1 && PC % 8 != 0) || (ks == PT * 2 - 1 && PC % 4 != 0)) && !(va[i] && vk[ks]))
            av[i] = 0.0;
        }
#pragma unroll
        for (int j = 0; j < NXT; ++j) bv[j] = EXT[(j * 8 + gq) * SE + ks * 4 + t];
#pragma unroll
        for (int i = 0; i < PT; ++i)
#pragma unroll
          for (int j = 0; j < NXT; ++j) dmma(c[i][j][0], c[i][j][1], av[i], bv[j]);
      }
#pragma unroll
      for (int i = 0; i < PT; ++i)
#pragma unroll
        for (int j = 0; j < NXT; ++j) {
          ar[(i * 8 + gq) * SA + j * 4 + t] = c[i][j][0];
          ai[(i * 8 + gq) * SA + j * 4 + t] = c[i][j][1];
        }
    }
    __syncwarp();
    // the row is assembled in shared memory (column order is the z-extent
    // order, scattered relative to the fragments) and leaves by one TMA bulk
    // store, instead of one scattered 16-byte global store per element
    auto put = [&](int my, int m0, double re, double im) {
      const int c = colidx[(my + M) * M1 + m0];
      if (c >= 0) stg[c] = make_double2(re, im);
    };
    if (lane == 0) dev::bulk_wait_read0();  // the previous unit's row has left the staging buffer
    __syncwarp();
    // Y stage (m0 >= 1, my >= 1)
    {
      double P[MTC][MTC][2], Q[MTC][MTC][2], R[MTC][MTC][2], S[MTC][MTC][2];
#pragma unroll
      for (int i = 0; i < MTC; ++i)
#pragma unroll
        for (int j = 0; j < MTC; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) P[i][j][e] = Q[i][j][e] = R[i][j][e] = S[i][j][e] = 0.0;
#pragma unroll
      for (int ks = 0; ks < PT * 2; ++ks) {
        const int kk = ks * 4 + t;
        double er[MTC], ei[MTC], br[MTC], bi[MTC];
#pragma unroll
        for (int i = 0; i < MTC; ++i) {
          er[i] = EYr[(i * 8 + gq) * SY + kk];
          ei[i] = EYi[(i * 8 + gq) * SY + kk];
          br[i] = ar[kk * SA + i * 8 + gq];
          bi[i] = ai[kk * SA + i * 8 + gq];
        }
#pragma unroll
        for (int i = 0; i < MTC; ++i)
#pragma unroll
          for (int j = 0; j < MTC; ++j) {
            dmma(P[i][j][0], P[i][j][1], er[i], br[j]);
            dmma(Q[i][j][0], Q[i][j][1], ei[i], bi[j]);
            dmma(R[i][j][0], R[i][j][1], er[i], bi[j]);
            dmma(S[i][j][0], S[i][j][1], ei[i], br[j]);
          }
      }
#pragma unroll
      for (int i = 0; i < MTC; ++i)
#pragma unroll
        for (int j = 0; j < MTC; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int my = i * 8 + gq + 1, m0 = j * 8 + 2 * t + e + 1;
            if (my <= M && m0 <= M) {
              const double p_ = P[i][j][e], q_ = Q[i][j][e], r_ = R[i][j][e], s_ = S[i][j][e];
              put(my, m0, p_ - q_, r_ + s_);
              put(-my, m0, p_ + q_, r_ - s_);
            }
          }
    }
    // remainders on the CUDA cores: the m0 = 0 column (my >= 1; a real) and the my = 0 row
    if (lane < M) {
      double P0 = 0.0, S0 = 0.0;
      for (int iy = 0; iy < p; ++iy) {
        const double a0 = ar[iy * SA + M];
        P0 = fma(EYr[lane * SY + iy], a0, P0);
        S0 = fma(EYi[lane * SY + iy], a0, S0);
      }
      put(lane + 1, 0, P0, S0);
      put(-(lane + 1), 0, P0, -S0);
    }
    if (lane <= M) {
      const int m0 = lane;
      double re = 0.0, im = 0.0;
      if (m0 == 0) {
        for (int iy = 0; iy < p; ++iy) re += ar[iy * SA + M];
      } else {
        for (int iy = 0; iy < p; ++iy) {
          re += ar[iy * SA + m0 - 1];
          im += ai[iy * SA + m0 - 1];
        }
      }
      put(0, m0, re, im);
    }
    dev::fence_proxy_async_smem();  // the row's generic-proxy writes, visible to the TMA store
    __syncwarp();
    if (lane == 0) {
      dev::bulk_s2g(Bo, stg, (uint32_t)ncol * 16u);
      dev::bulk_commit();
    }
    __syncwarp();  // ar / ai and this w buffer are rewritten by the next units
  }
  if (lane == 0) dev::bulk_wait0();  // (the CTA's shared memory must outlive its stores)
}

// inv_xy, warp-independent form (3D, p <= 24, N <= 33).  The unit of work is
// one (box, component, z-slab); every warp walks units with a global stride
// and needs no CTA barrier: its slab of C1 (the compressed (my, m0) row of
// one iz) arrives by cp.async, double buffered, scattered into a dense
// (my, m0) tile; the Hermitian-split Y stage reads U = C[+my] + C[-my],
// V = C[+my] - C[-my] straight from that tile at fragment-load time
//   d.re = C0.re + [Er | Ei] [Ur ; Vi],  d.im = C0.im + [Er | -Ei] [Ui ; Vr]
// (all PT x MT output tiles at once: the A and B fragments of a k-step are
// loaded once for 2 PT MT DMMAs), the m0 = 0 column on the CUDA cores, and
// the X stage with all PT x PT tiles of the slab register-blocked
//   out[iy, ix] += pf sum_(m0, part) d[iy][(m0, part)] EXw[ix][(m0, part)]
// (the output slab is read at the start of the unit).  Dense-tile rows have a
// stride == 2 mod 8 complex, so the 16-byte B-fragment loads of a quarter
// warp hit distinct bank groups.
constexpr int kWI3 = 7;  // warps per CTA (shared memory: ~29 KB per warp)

__host__ __device__ constexpr int r2c(int x) { return (x + 5) / 8 * 8 + 2; }  // >= x, == 2 mod 8

template <int PC, int NC>
__global__ void __launch_bounds__(kWI3 * 32, 1) k_inv_xy3(PWGrid g, const int* __restrict__ tboxes, int ntb, int d,
                                                         const double2* __restrict__ C, double pf,
                                                         double* __restrict__ incoming) {
  constexpr int PT = 3, MTC = 2, P8 = PT * 8;
  const int p = PC > 0 ? PC : g.p, N = NC > 0 ? NC : g.N, M = (N - 1) / 2, ncol = g.ncol, pp = p * p;
  const int M1 = M + 1, M8 = MTC * 8, K2 = 2 * M8;
  const int SA2 = r4(K2);                // A' rows (iy), == 4 mod 8
  const int NXK = (2 * M1 + 3) / 4 * 4;  // X-stage K
  const int SX = r4(NXK);
  const int SD = r2c(M1);                // dense tile row stride (complex)
  extern __shared__ double sm[];
  double* Are = sm;                      // [P8][SA2]  [Er | Ei]
  double* Aim = Are + P8 * SA2;          // [P8][SA2]  [Er | -Ei]
  double* EXw = Aim + P8 * SA2;          // [P8 (ix)][SX]
  int* dix = reinterpret_cast<int*>(EXw + P8 * SX);  // [ncol], padded to 16 bytes
  double* wbase = EXw + P8 * SX + (ncol + 3) / 4 * 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, t = lane & 3;
  const size_t per_warp = 2 * (size_t)N * SD * 2 + (size_t)P8 * SX;  // doubles
  double2* den = reinterpret_cast<double2*>(wbase + warp * per_warp);  // [2][N][SD]
  double* dd = wbase + warp * per_warp + 2 * (size_t)N * SD * 2;       // [P8][SX]
  for (int e = tid; e < P8 * SA2; e += blockDim.x) {
    const int iy = e / SA2, k = e % SA2;
    double vr = 0.0, vi = 0.0;
    if (iy < p && k < K2) {
      const int myp = k < M8 ? k : k - M8;
      if (myp < M) {
        const double2 ev = g.E[(size_t)(myp + 1 + M) * p + iy];
        vr = k < M8 ? ev.x : ev.y;
        vi = k < M8 ? ev.x : -ev.y;
      }
    }
    Are[e] = vr;
    Aim[e] = vi;
  }
  for (int e = tid; e < P8 * SX; e += blockDim.x) {  // Re(conj(E) d) = Er d.re + Ei d.im, weight 1 | 2
    const int ix = e / SX, k = e % SX, m0 = k >> 1, part = k & 1;
    double v = 0.0;
    if (ix < p && m0 < M1) {
      const double2 ev = g.E[(size_t)(m0 + M) * p + ix];
      v = (m0 ? 2.0 : 1.0) * (part ? ev.y : ev.x);
    }
    EXw[e] = v;
  }
  for (int c = tid; c < ncol; c += blockDim.x) dix[c] = (g.col_my[c] + M) * SD + g.col_m0[c];
  for (size_t e = lane; e < per_warp; e += 32) wbase[warp * per_warp + e] = 0.0;  // out-of-band entries stay 0
  __syncthreads();
  const int total = ntb * d * p;
  const int nw = gridDim.x * kWI3;
  auto issue = [&](int u, int buf) {
    const int item = u / p, iz = u % p;
    const double2* src = C + ((size_t)item * g.pz + iz) * ncol;
    double2* dst = den + buf * N * SD;
    for (int c = lane; c < ncol; c += 32) dev::cp_async16(dst + dix[c], src + c);
    cp_commit();
  };
  int u = blockIdx.x * kWI3 + warp;
  if (u < total) issue(u, 0);
  for (int k = 0; u < total; ++k, u += nw) {
    const int buf = k & 1;
    if (u + nw < total) {
      issue(u + nw, buf ^ 1);
      cp_wait1();
    } else {
      cp_wait0();
    }
    __syncwarp();
    const int item = u / p, iz = u % p, tb = item / d, j = item % d;
    double* out = incoming + ((size_t)tboxes[tb] * d + j) * (size_t)(p * pp) + (size_t)iz * pp;
    // the output slab's current values (read early; added to at the end)
    double o[PT][PT][2];
#pragma unroll
    for (int mt = 0; mt < PT; ++mt)
#pragma unroll
      for (int nt = 0; nt < PT; ++nt) {
        const int iy = mt * 8 + gq, ix = nt * 8 + 2 * t;
        o[mt][nt][0] = (iy < p && ix < p) ? out[iy * p + ix] : 0.0;
        o[mt][nt][1] = (iy < p && ix + 1 < p) ? out[iy * p + ix + 1] : 0.0;
      }
    const double2* D = den + buf * N * SD;
    // m0 = 0 column (CUDA cores): lane = iy.  Only its real part is formed:
    // the X stage weighs the imaginary part by Im E(0, ix) = 0
    if (lane < p) {
      double re = D[M * SD].x;
      for (int r = 0; r < M; ++r) {
        const double2 cp = D[(r + 1 + M) * SD], cm = D[(M - 1 - r) * SD];
        const double er = Are[lane * SA2 + r], ei = Are[lane * SA2 + M8 + r];
        re = fma(er, cp.x + cm.x, fma(ei, cp.y - cm.y, re));
      }
      dd[lane * SX] = re;
      dd[lane * SX + 1] = 0.0;
    }
    // Y stage: all PT x MT tiles, re and im
    double yr[PT][MTC][2], yi[PT][MTC][2];
#pragma unroll
    for (int a = 0; a < PT; ++a)
#pragma unroll
      for (int b = 0; b < MTC; ++b) yr[a][b][0] = yr[a][b][1] = yi[a][b][0] = yi[a][b][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < K2 / 4; ++ks) {
      const int kk = ks * 4 + t;
      const bool vpart = kk >= M8;
      const int r = vpart ? kk - M8 : kk;  // my - 1
      double bre[MTC], bim[MTC];
#pragma unroll
      for (int nt = 0; nt < MTC; ++nt) {
        const int m0 = nt * 8 + gq + 1;
        double2 cp = make_double2(0.0, 0.0), cm = cp;
        if (r < M && m0 <= M) {
          cp = D[(r + 1 + M) * SD + m0];
          cm = D[(M - 1 - r) * SD + m0];
        }
        bre[nt] = vpart ? cp.y - cm.y : cp.x + cm.x;  // Vi | Ur
        bim[nt] = vpart ? cp.x - cm.x : cp.y + cm.y;  // Vr | Ui
      }
#pragma unroll
      for (int it = 0; it < PT; ++it) {
        const double are = Are[(it * 8 + gq) * SA2 + kk], aim = Aim[(it * 8 + gq) * SA2 + kk];
#pragma unroll
        for (int nt = 0; nt < MTC; ++nt) {
          dmma(yr[it][nt][0], yr[it][nt][1], are, bre[nt]);
          dmma(yi[it][nt][0], yi[it][nt][1], aim, bim[nt]);
        }
      }
    }
#pragma unroll
    for (int it = 0; it < PT; ++it)
#pragma unroll
      for (int nt = 0; nt < MTC; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m0 = nt * 8 + 2 * t + e + 1, row = it * 8 + gq;
          if (m0 <= M) {
            const double2 c0 = D[M * SD + m0];
            dd[row * SX + 2 * m0] = yr[it][nt][e] + c0.x;
            dd[row * SX + 2 * m0 + 1] = yi[it][nt][e] + c0.y;
          }
        }
    __syncwarp();
    // X stage: all PT x PT tiles of the slab
    double x[PT][PT][2];
#pragma unroll
    for (int a = 0; a < PT; ++a)
#pragma unroll
      for (int b = 0; b < PT; ++b) x[a][b][0] = x[a][b][1] = 0.0;
    for (int ks = 0; ks < NXK / 4; ++ks) {
      double av[PT], bv[PT];
#pragma unroll
      for (int a = 0; a < PT; ++a) {
        av[a] = dd[(a * 8 + gq) * SX + ks * 4 + t];
        bv[a] = EXw[(a * 8 + gq) * SX + ks * 4 + t];
      }
#pragma unroll
      for (int a = 0; a < PT; ++a)
#pragma unroll
        for (int b = 0; b < PT; ++b) dmma(x[a][b][0], x[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int mt = 0; mt < PT; ++mt)
#pragma unroll
      for (int nt = 0; nt < PT; ++nt) {
        const int iy = mt * 8 + gq, ix = nt * 8 + 2 * t;
        if (iy < p) {
          if (ix < p) out[iy * p + ix] = o[mt][nt][0] + pf * x[mt][nt][0];
          if (ix + 1 < p) out[iy * p + ix + 1] = o[mt][nt][1] + pf * x[mt][nt][1];
        }
      }
    __syncwarp();  // dd and this den buffer are rewritten by the next units
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

void attr(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

bool pw_mma_supported(const PWGrid& g) {
  return g.dim == 3 && g.p <= 32 && g.N <= 48 && g.pz == g.p;
}

void launch_forward_mma(const PWGrid& g, const int* boxes, int nbox, int nch, const double* outgoing, double2* B,
                        double2* G, cudaStream_t st) {
  if (nbox <= 0) return;
  const int PT = (g.p + 7) / 8 <= 3 ? 3 : 4;  // the instantiated template sizes
  const int M = g.M, M1 = M + 1, MT = (M + 7) / 8, P8 = PT * 8;
  {  // x and y stages: B[box][ch][iz][col]
    const int NX8 = (2 * M + 1 + 7) / 8 * 8;
    const size_t sm = sizeof(double) * ((size_t)NX8 * (P8 + 4) + 2 * (size_t)MT * 8 * (P8 + 4) +
                                        2 * 4 * (size_t)P8 * (P8 + 4) + 4 * (size_t)P8 * r8(NX8 > 16 * MT ? NX8 : 16 * MT)) +
                      sizeof(int) * (size_t)g.N * M1;
    auto sm3 = [&](int wf) {
      return sizeof(double) * (40 * 28 + 2 * 16 * 28 + (size_t)(g.N * M1 + 7) / 8 * 2 +
                               (size_t)wf * (2 * 24 * 28 + 2 * 24 * 20 + 2 * ((g.ncol + 1) / 2 * 2)));
    };
    if (PT == 3 && g.N <= 33 && g.dim == 3) {  // warp-independent slabs
      const int wf = sm3(kWF3) <= 227 * 1024 ? kWF3 : kWF3 - 1;
      const int units = nbox * nch * g.p;
      const int ctas = std::max(1, std::min(num_sms(), (units + wf - 1) / wf));
#define FX3(PC_, NC_)                                                                                        \
  do {                                                                                                       \
    if (wf == kWF3) {                                                                                        \
      attr((const void*)k_fwd_xy3<PC_, NC_, kWF3>, sm3(kWF3));                                               \
      k_fwd_xy3<PC_, NC_, kWF3><<<ctas, kWF3 * 32, sm3(kWF3), st>>>(g, boxes, nbox, nch, outgoing, B);      \
    } else {                                                                                                 \
      attr((const void*)k_fwd_xy3<PC_, NC_, kWF3 - 1>, sm3(kWF3 - 1));                                       \
      k_fwd_xy3<PC_, NC_, kWF3 - 1><<<ctas, (kWF3 - 1) * 32, sm3(kWF3 - 1), st>>>(g, boxes, nbox, nch,       \
                                                                               outgoing, B);                 \
    }                                                                                                        \
  } while (0)
      if (g.p == 23 && g.N == 33) FX3(23, 33);
      else if (g.p == 22 && g.N == 33) FX3(22, 33);
      else FX3(0, 0);
#undef FX3
    } else {
#define FX2(PT_, PC_, NC_)                                                                                    \
  do {                                                                                                        \
    attr((const void*)k_fwd_xy2<PT_, PC_, NC_>, sm);                                                          \
    k_fwd_xy2<PT_, PC_, NC_><<<std::min(nbox * nch, 2 * num_sms()), kW * 32, sm, st>>>(g, boxes, nbox, nch,   \
                                                                                     outgoing, B);            \
  } while (0)
    if (g.p == 23 && g.N == 33) FX2(3, 23, 33);
    else if (g.p == 22 && g.N == 33) FX2(3, 22, 33);
    else if (g.p == 30 && g.N == 45) FX2(4, 30, 45);
    else if (PT <= 3) FX2(3, 0, 0);
    else FX2(4, 0, 0);
#undef FX2
    }
  }
  if (PT == 3 && g.Mz <= 16) {  // z stage, warp-independent blocks
    const size_t sz = sizeof(double) * 2 * 16 * 28 + sizeof(double2) * (size_t)kWZF * 2 * 24 * kZR;
    const int units = nbox * nch * ((g.ncol + kZB - 1) / kZB);
    const int ctas = std::max(1, std::min(num_sms(), (units + kWZF - 1) / kWZF));
    attr((const void*)k_zf3, sz);
    k_zf3<<<ctas, kWZF * 32, sz, st>>>(g, nch, nbox, B, G);
  } else {  // z stage: G[box][ch][mode]
    const int SI = (2 * kCB) % 16 == 8 ? 2 * kCB : 2 * kCB + 8;
    const int M8 = (g.Mz + 7) / 8 * 8;
    const size_t sz = sizeof(double) * (2 * (size_t)M8 * (P8 + 4) + 2 * (size_t)P8 * SI);
    const int items = nbox * nch * ((g.ncol + kCB - 1) / kCB);
    const int ctas = std::min(items, 3 * num_sms());
    if (PT <= 3) {
      attr((const void*)k_zf2<3>, sz);
      k_zf2<3><<<ctas, kW * 32, sz, st>>>(g, nch, nbox, B, G);
    } else {
      attr((const void*)k_zf2<4>, sz);
      k_zf2<4><<<ctas, kW * 32, sz, st>>>(g, nch, nbox, B, G);
    }
  }
}

void launch_inverse_mma(const PWGrid& g, const int* tboxes, int ntb, int d, const double2* F, double2* C, double pf,
                        double* incoming, cudaStream_t st) {
  if (ntb <= 0) return;
  const int PT = (g.p + 7) / 8 <= 3 ? 3 : 4;  // the instantiated template sizes
  const int P8 = PT * 8, M = g.M, M1 = M + 1, MT = (M + 7) / 8, M8 = MT * 8;
  if (PT == 3 && g.Mz <= 16) {  // z stage, warp-independent blocks
    const size_t sz = sizeof(double) * 2 * 24 * 36 + sizeof(double2) * (size_t)kWZI * 2 * 33 * kZR;
    const int units = ntb * d * ((g.ncol + kZB - 1) / kZB);
    const int ctas = std::max(1, std::min(num_sms(), (units + kWZI - 1) / kWZI));
    attr((const void*)k_zi3, sz);
    k_zi3<<<ctas, kWZI * 32, sz, st>>>(g, d, ntb, F, C);
  } else {  // z stage: C1[box][j][iz][col]
    const int M8z = (g.Mz + 7) / 8 * 8;
    const size_t sz = sizeof(double) * 2 * (size_t)P8 * r4(2 * M8z) + sizeof(double2) * 2 * (size_t)g.Nz * (kCB + 2);
    const int items = ntb * d * ((g.ncol + kCB - 1) / kCB);
    const int ctas = std::min(items, 2 * num_sms());
    if (PT <= 3) {
      attr((const void*)k_zi2<3>, sz);
      k_zi2<3><<<ctas, kW * 32, sz, st>>>(g, d, ntb, F, C);
    } else {
      attr((const void*)k_zi2<4>, sz);
      k_zi2<4><<<ctas, kW * 32, sz, st>>>(g, d, ntb, F, C);
    }
  }
  {  // y and x stages into the incoming proxies
    const int K2 = 2 * M8, SA2 = r4(K2), SB = (M8 % 16 == 8) ? M8 : M8 + 8, NXK = (2 * M1 + 3) / 4 * 4,
              SX2 = r4(NXK);
    const size_t sm2 = sizeof(double) * (2 * (size_t)P8 * SA2 + (size_t)P8 * SX2 + 4 * (size_t)P8 * SX2 +
                                         2 * 4 * (size_t)K2 * SB) +
                       sizeof(double2) * 2 * 4 * (size_t)g.N * M1 + sizeof(int) * (size_t)g.ncol;
    const int SD3 = r2c(M1), NXK3 = (2 * M1 + 3) / 4 * 4, SX3 = r4(NXK3);
    const size_t sm3 = sizeof(double) * (2 * (size_t)P8 * r4(32) + (size_t)P8 * SX3 + (size_t)(g.ncol + 3) / 4 * 2 +
                                         (size_t)kWI3 * (2 * (size_t)g.N * SD3 * 2 + (size_t)P8 * SX3));
    if (PT == 3 && g.N <= 33 && sm3 <= 227 * 1024) {  // warp-independent slabs
      const int units = ntb * d * g.p;
      const int ctas = std::max(1, std::min(num_sms(), (units + kWI3 - 1) / kWI3));
#define IX3(PC_, NC_)                                                                                        \
  do {                                                                                                       \
    attr((const void*)k_inv_xy3<PC_, NC_>, sm3);                                                             \
    k_inv_xy3<PC_, NC_><<<ctas, kWI3 * 32, sm3, st>>>(g, tboxes, ntb, d, C, pf, incoming);                   \
  } while (0)
      if (g.p == 23 && g.N == 33) IX3(23, 33);
      else if (g.p == 22 && g.N == 33) IX3(22, 33);
      else IX3(0, 0);
#undef IX3
    } else if (sm2 > 227 * 1024) {  // the split kernel stages dense slabs: too big for the largest grids
      const int M18 = (M1 + 7) / 8 * 8, NY8 = (g.N + 7) / 8 * 8, NX8 = (2 * M1 + 7) / 8 * 8;
      const int SA = r4(2 * NY8), SX = r4(NX8 > 2 * M18 ? NX8 : 2 * M18);
      const size_t smem = sizeof(double) * (2 * (size_t)P8 * SA + (size_t)P8 * SX + 4 * (size_t)P8 * SX +
                                            2 * 4 * 2 * (size_t)g.ncol) + sizeof(int) * (size_t)NY8 * M18;
      if (PT <= 3) {
        attr((const void*)k_inv_xy_mma<3, 0, 0>, smem);
        k_inv_xy_mma<3, 0, 0><<<dim3(ntb, d), kWI * 32, smem, st>>>(g, tboxes, d, C, pf, incoming);
      } else {
        attr((const void*)k_inv_xy_mma<4, 0, 0>, smem);
        k_inv_xy_mma<4, 0, 0><<<dim3(ntb, d), kWI * 32, smem, st>>>(g, tboxes, d, C, pf, incoming);
      }
    } else {
#define IX2(PT_, PC_, NC_)                                                                                  \
  do {                                                                                                      \
    attr((const void*)k_inv_xy2<PT_, PC_, NC_>, sm2);                                                       \
    k_inv_xy2<PT_, PC_, NC_><<<std::min(ntb * d, num_sms()), kWI * 32, sm2, st>>>(g, tboxes, ntb, d, C, pf, \
                                                                                    incoming);              \
  } while (0)
      if (g.p == 23 && g.N == 33) IX2(3, 23, 33);
      else if (g.p == 22 && g.N == 33) IX2(3, 22, 33);
      else if (g.p == 30 && g.N == 45) IX2(4, 30, 45);
      else if (PT <= 3) IX2(3, 0, 0);
      else IX2(4, 0, 0);
#undef IX2
    }
  }
}

}  // namespace sdmkb
