// Host setup numerics (see setup.hpp).  Each routine restates the reference
// algorithm it must agree with; the citation is the reference file:line.
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <functional>

namespace sdmkb {

namespace {

constexpr double PI = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- plan ----
// Tuned (q, p, N_per | qg, pg, N_perg) rows at eps = 1e-3, 1e-6, 1e-9, 1e-12
// (params.cpp:21-38) and leaf sizes (params.cpp:40-41).
const double kRowsStokeslet[4][6] = {
    {10, 12, 3, 14, 14, 5}, {17, 23, 5, 25, 28, 9}, {25, 33, 9, 38, 43, 13}, {31, 44, 11, 50, 58, 17}};
const double kRowsStresslet[4][6] = {
    {9, 11, 3, 11, 12, 3}, {17, 22, 5, 26, 28, 9}, {25, 33, 9, 40, 44, 13}, {32, 44, 11, 54, 60, 17}};
const double kRowsRotlet[4][6] = {
    {7, 8, 3, 9, 9, 3}, {14, 18, 5, 21, 23, 7}, {20, 28, 7, 34, 38, 11}, {27, 39, 9, 47, 53, 15}};
const double kLeaf2[4] = {120, 240, 360, 480};
const double kLeaf3[4] = {600, 1200, 2000, 3000};

// piecewise linear in t = -log10 eps over {3,6,9,12}, extrapolated (params.cpp:45-49)
double column_at(const double v[4], double t) {
  int s = (int)std::floor((t - 3.0) / 3.0);
  s = s < 0 ? 0 : (s > 2 ? 2 : s);
  double u = (t - 3.0 - 3.0 * s) / 3.0;
  return v[s] + u * (v[s + 1] - v[s]);
}
int round_up(double v) { return (int)std::ceil(v - 1e-9); }

// ----------------------------------------------------------- Legendre ----
// P_0..P_n at x by the three-term recurrence (detail/legendre.hpp:12-18)
void leg_values(double x, int n, double* P) {
  P[0] = 1.0;
  if (n < 1) return;
  P[1] = x;
  for (int k = 1; k < n; ++k) P[k + 1] = ((2 * k + 1) * x * P[k] - k * P[k - 1]) / (k + 1);
}

// values + first three derivatives (detail/legendre.hpp:22-38)
void leg_values_d3(double x, int n, double* P, double* d1, double* d2, double* d3) {
  leg_values(x, n, P);
  d1[0] = d2[0] = d3[0] = 0.0;
  if (n < 1) return;
  d1[1] = 1.0;
  d2[1] = d3[1] = 0.0;
  for (int k = 1; k < n; ++k) {
    double f = 2 * k + 1;
    d1[k + 1] = d1[k - 1] + f * P[k];
    d2[k + 1] = d2[k - 1] + f * d1[k];
    d3[k + 1] = d3[k - 1] + f * d2[k];
  }
}

// D[m][n] = P_n^(m)(0) (legendre.cpp:7-22)
std::vector<std::vector<double>> leg_derivs_zero(int mmax, int nmax) {
  std::vector<std::vector<double>> D(mmax + 1, std::vector<double>(nmax + 1, 0.0));
  D[0][0] = 1.0;
  for (int k = 1; k + 1 <= nmax; ++k) D[0][k + 1] = -k * D[0][k - 1] / (k + 1);
  for (int m = 1; m <= mmax; ++m) {
    if (nmax >= 1) D[m][1] = (m == 1) ? 1.0 : 0.0;
    for (int k = 1; k + 1 <= nmax; ++k)
      D[m][k + 1] = ((2 * k + 1) * m * D[m - 1][k] - k * D[m][k - 1]) / (k + 1);
  }
  return D;
}

// Gauss-Legendre rule on [-1,1] by Newton on P_n (legendre.cpp:24-62)
void gl_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double t = std::cos(PI * (i + 0.75) / (n + 0.5));
    double pn = 0.0, dpn = 0.0;
    for (int it = 0; it < 64; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 1; k < n; ++k) {
        double p2 = ((2 * k + 1) * t * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      pn = p1;
      dpn = n * (t * p1 - p0) / (t * t - 1.0);
      double step = -pn / dpn;
      t += step;
      if (std::fabs(step) < 1e-15) break;
    }
    x[i] = -t;
    x[n - 1 - i] = t;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dpn * dpn);
  }
  if (n % 2 == 1) {
    double p0 = 1.0, p1 = 0.0;
    for (int k = 1; k < n; ++k) {
      double p2 = (-k * p0) / (k + 1);
      p0 = p1;
      p1 = p2;
    }
    double dp = n * (0.0 - p0) / (0.0 - 1.0);
    x[n / 2] = 0.0;
    w[n / 2] = 2.0 / (dp * dp);
  }
}

const std::vector<double>& gl_nodes(int n, bool weights) {
  static thread_local std::vector<double> x32, w32, x64, w64;
  std::vector<double>& x = n == 32 ? x32 : x64;
  std::vector<double>& w = n == 32 ? w32 : w64;
  if (x.empty()) gl_rule(n, x, w);
  return weights ? w : x;
}

// psi0c and derivatives from the even Legendre series (windows.cpp:20-41)
void psi_at(const WindowFn& w, double x, int order, double* out) {
  int nmax = 2 * ((int)w.leg.size() - 1);
  std::vector<double> P(nmax + 2), d1(nmax + 2), d2(nmax + 2), d3(nmax + 2);
  if (order == 0)
    leg_values(x, nmax, P.data());
  else
    leg_values_d3(x, nmax, P.data(), d1.data(), d2.data(), d3.data());
  for (int i = 0; i <= order; ++i) out[i] = 0.0;
  for (size_t j = 0; j < w.leg.size(); ++j) {
    double a = w.leg[j];
    out[0] += a * P[2 * j];
    if (order >= 1) out[1] += a * d1[2 * j];
    if (order >= 2) out[2] += a * d2[2 * j];
    if (order >= 3) out[3] += a * d3[2 * j];
  }
}

// ---------------------------------------------------------- Chebyshev ----
// Adaptive fit on first-kind nodes, doubling n -> 2n-1 until the top eighth
// of the spectrum is below tol (chebyshev.cpp:21-58).
Cheb cheb_fit(const std::function<double(double)>& f, double lo, double hi, double tol,
              int max_n = 4097) {
  Cheb t;
  t.lo = lo;
  t.hi = hi;
  for (int n = 17; n <= max_n; n = 2 * n - 1) {
    std::vector<double> fv(n), c(n, 0.0);
    for (int i = 0; i < n; ++i)
      fv[i] = f(0.5 * (lo + hi) + 0.5 * (hi - lo) * std::cos(M_PI * (2 * i + 1) / (2.0 * n)));
    double cmax = 0.0;
    for (int k = 0; k < n; ++k) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += fv[i] * std::cos(k * M_PI * (2 * i + 1) / (2.0 * n));
      c[k] = s * (k == 0 ? 1.0 : 2.0) / n;
      cmax = std::max(cmax, std::fabs(c[k]));
    }
    if (cmax == 0.0) {
      t.a.assign(1, 0.0);
      return t;
    }
    double scale = std::max(1.0, cmax), tail = 0.0;
    for (int k = n - std::max(2, n / 8); k < n; ++k) tail = std::max(tail, std::fabs(c[k]));
    if (tail <= tol * scale || 2 * n - 1 > max_n) {
      int keep = n;
      while (keep > 1 && std::fabs(c[keep - 1]) < 0.1 * tol * scale) --keep;
      c.resize(keep);
      t.a = c;
      return t;
    }
  }
  throw RuntimeError("cheb_fit: not converged");
}

// ------------------------------------------------- 2D residual pipeline ----
// Radial Fourier quadrature of the mollified structural functions
// (split2d.cpp:1-326), restated.
double bihar_hat_series(double k, double R, int dim) {  // split2d.cpp:30-49
  double u = k * R;
  if (u >= 1.0) return trunc_bihar_hat(k, R, dim);
  double u2 = u * u, acc = 0.0, pw = 1.0;
  for (int m = 2; m <= 13; ++m) {
    double den = 1.0;
    if (dim == 3) {
      for (int j = 2; j <= 2 * m + 1; ++j) den *= j;
    } else {
      double fm = 1.0;
      for (int j = 2; j <= m; ++j) fm *= j;
      den = std::pow(4.0, m) * fm * fm;
    }
    acc += ((m & 1) ? -1.0 : 1.0) * (m - 1) / den * pw;
    pw *= u2;
  }
  return R * R * R * R * acc;
}

double j0_minus_j1_over_u(double u) {  // split2d.cpp:52-65
  if (u < 0.5) {
    double u2 = u * u, acc = 0.0, pw = 1.0, fm = 1.0;
    for (int m = 0; m <= 8; ++m) {
      if (m > 0) fm *= m;
      double den = 2.0 * std::pow(4.0, m) * fm * (fm * (m + 1));
      acc += ((m & 1) ? -1.0 : 1.0) * (2.0 * m + 1.0) / den * pw;
      pw *= u2;
    }
    return acc;
  }
  return std::cyl_bessel_j(0.0, u) - std::cyl_bessel_j(1.0, u) / u;
}

double j1_combo(double u) {  // split2d.cpp:67-81
  if (u < 0.5) {
    double u2 = u * u, acc = 0.0, pw = u, fj = 1.0;
    for (int j = 0; j <= 8; ++j) {
      if (j > 0) fj *= j;
      double den = std::pow(4.0, j + 1) * fj * (fj * (j + 1)) * (j + 2);
      acc += ((j & 1) ? -1.0 : 1.0) * (2.0 * j + 3.0) / den * pw;
      pw *= u2;
    }
    return acc;
  }
  double j0 = std::cyl_bessel_j(0.0, u), j1 = std::cyl_bessel_j(1.0, u);
  return j1 + (j0 - 2.0 * j1 / u) / u;
}

void sinc_d(double u, double out[4]) {  // split2d.cpp:84-121
  if (u < 0.5) {
    if (u == 0.0) {
      out[0] = 1.0;
      out[1] = 0.0;
      out[2] = -1.0 / 3.0;
      out[3] = 0.0;
      return;
    }
    double u2 = u * u, f0 = 0, f1 = 0, f2 = 0, f3 = 0, fact = 1.0, pw = 1.0;
    for (int m = 0; m <= 10; ++m) {
      if (m > 0) fact *= (2.0 * m) * (2.0 * m + 1.0);
      double c = ((m & 1) ? -1.0 : 1.0) / fact;
      f0 += c * pw;
      if (m >= 1) f1 += c * 2.0 * m * pw / u;
      if (m >= 1) f2 += c * 2.0 * m * (2.0 * m - 1.0) * pw / u2;
      if (m >= 2) f3 += c * 2.0 * m * (2.0 * m - 1.0) * (2.0 * m - 2.0) * pw / (u2 * u);
      pw *= u2;
    }
    out[0] = f0;
    out[1] = f1;
    out[2] = f2;
    out[3] = f3;
    return;
  }
  double s = std::sin(u), c = std::cos(u);
  double f0 = s / u, f1 = (c - f0) / u, f2 = -f0 - 2.0 * f1 / u;
  out[0] = f0;
  out[1] = f1;
  out[2] = f2;
  out[3] = -f1 - 2.0 * f2 / u + 2.0 * f1 / (u * u);
}

struct Quad {
  std::vector<double> k, wb, wp;
};

Quad quad_grid(int dim, const WindowFn& w, double R, double K, int panels) {  // split2d.cpp:129-152
  Quad q;
  const std::vector<double>& gx = gl_nodes(32, false);
  const std::vector<double>& gw = gl_nodes(32, true);
  double hk = K / panels, norm = 1.0 / (2.0 * std::pow(PI, dim - 1));
  for (int pn = 0; pn < panels; ++pn) {
    double mid = (pn + 0.5) * hk, half = 0.5 * hk;
    for (size_t i = 0; i < gx.size(); ++i) {
      double k = mid + half * gx[i], wt = gw[i] * half;
      q.k.push_back(k);
      q.wb.push_back(wt * bihar_hat_series(k, R, dim) * moll_hat(w, k) * std::pow(k, dim - 1) * norm);
      q.wp.push_back(wt * win_hat(w, k));
    }
  }
  return q;
}

std::array<double, 2> moll_struct(const Quad& q, int kernel, int dim, double R, double r) {  // split2d.cpp:155-215
  if (kernel == kRotlet) {
    double mo = 0.0;
    if (dim == 2) {
      for (size_t i = 0; i < q.k.size(); ++i) mo += q.wp[i] * std::cyl_bessel_j(1.0, q.k[i] * r);
      return {0.0, r * mo};
    }
    for (size_t i = 0; i < q.k.size(); ++i) {
      double d[4];
      sinc_d(q.k[i] * r, d);
      mo += q.wp[i] * q.k[i] * d[1];
    }
    return {0.0, -(2.0 * r * r / PI) * mo};
  }
  double sd = 0.0, so = 0.0;
  for (size_t i = 0; i < q.k.size(); ++i) {
    double k = q.k[i], u = k * r, xd, xo;
    if (dim == 2) {
      double j1 = std::cyl_bessel_j(1.0, u), g2 = j0_minus_j1_over_u(u), g3 = j1_combo(u);
      if (kernel == kStokeslet) {
        xd = 8.0 * PI * r * k * k * g2;
        xo = 8.0 * PI * (k * j1 - r * k * k * g2);
      } else {
        double base = k * j1 - r * k * k * g2, cub = r * r * k * k * k * g3;
        xd = 8.0 * PI * (base - cub);
        xo = 8.0 * PI * (base - cub / 3.0);
      }
    } else {
      double d[4];
      sinc_d(u, d);
      double F1 = k * d[1], F2 = k * k * d[2], F3 = k * k * k * d[3];
      if (kernel == kStokeslet) {
        xd = -8.0 * PI * (F1 + r * F2);
        xo = 8.0 * PI * (-F1 + r * F2);
      } else {
        xd = -8.0 * PI * r * r * F3;
        xo = 8.0 * PI * (-F1 + r * F2 - r * r * F3 / 3.0);
      }
    }
    sd += q.wb[i] * xd;
    so += q.wb[i] * xo;
  }
  if (kernel == kStokeslet) sd += dim == 3 ? 2.0 * r / R : 2.0 * r * (1.0 - std::log(R));
  return {sd, so};
}

Quad converged_quad(int kernel, int dim, const WindowFn& w, double R, double tol, double rmax) {  // split2d.cpp:221-247
  double K = w.kind == kProlate ? w.c : 2.0 * std::sqrt(45.0) / w.sigma;
  int panels = std::max(8, (int)std::ceil(K * (R + rmax) / (2.0 * PI)) + 8);
  double qtol = std::max(1e-13, 1e-4 * tol);
  const double probes[] = {0.02, 0.2, 0.45, 0.7, 0.9, 0.999, rmax};
  Quad a = quad_grid(dim, w, R, K, panels);
  for (int it = 0; it < 4; ++it) {
    Quad b = quad_grid(dim, w, R, K, 2 * panels);
    double worst = 0.0;
    for (double r : probes) {
      if (r > rmax) continue;
      auto va = moll_struct(a, kernel, dim, R, r), vb = moll_struct(b, kernel, dim, R, r);
      for (int j = 0; j < 2; ++j)
        worst = std::max(worst, std::fabs(va[j] - vb[j]) / std::max(1.0, std::fabs(vb[j])));
    }
    if (worst < qtol) return b;
    a = std::move(b);
    panels *= 2;
  }
  throw RuntimeError("numeric_residual_pipeline: quadrature failed to converge");
}

// phi_tail_moment: int_r^inf t phi(t) dt (split.cpp:25-42)
double tail_moment(const WindowFn& w, double r) {
  if (w.kind == kGaussian) {
    double s = r / w.sigma;
    return w.sigma * std::exp(-s * s) / (2.0 * std::sqrt(PI));
  }
  if (r >= 1.0) return 0.0;
  const std::vector<double>& gx = gl_nodes(64, false);
  const std::vector<double>& gw = gl_nodes(64, true);
  double a = std::max(r, 0.0), mid = 0.5 * (a + 1.0), half = 0.5 * (1.0 - a), s = 0.0;
  for (size_t i = 0; i < gx.size(); ++i) {
    double t = mid + half * gx[i];
    s += gw[i] * t * win_phi(w, t);
  }
  return half * s;
}

}  // namespace

// ------------------------------------------------------------- public ----
Plan select_plan(int kernel, double eps, int window, int dim) {  // params.cpp:60-115
  if (dim != 2 && dim != 3) throw InvalidArgument("select_parameters: dim must be 2 or 3");
  if (!(eps >= 1e-13 && eps <= 1e-2))
    throw InvalidArgument("select_parameters: accuracy must lie in [1e-13, 1e-2]");
  const double(*rows)[6] = nullptr;
  if (kernel == kStokeslet) rows = kRowsStokeslet;
  else if (kernel == kStresslet) rows = kRowsStresslet;
  else if (kernel == kRotlet) rows = kRowsRotlet;
  else throw InvalidArgument("select_parameters: no tuned parameters for this kernel");
  if (window != kProlate && window != kGaussian) throw InvalidArgument("select_parameters: bad window");
  double t = -std::log10(eps);
  auto col = [&](int f) {
    double v[4] = {rows[0][f], rows[1][f], rows[2][f], rows[3][f]};
    return column_at(v, t);
  };
  Plan P;
  P.kernel = kernel;
  P.dim = dim;
  P.window = window;
  P.tol = eps;
  int off = window == kProlate ? 0 : 3;
  double q = col(off + 0), p = col(off + 1), nper = col(off + 2);
  if (window == kProlate)
    P.c = q * M_PI / 3.0;
  else
    P.sigma = std::sqrt(6.0 / (M_PI * q));
  P.p = round_up(p);
  P.N1 = 2 * round_up(q) - 1;
  int np = round_up(nper);
  P.N_per = (np % 2 == 0) ? np + 1 : np;
  P.n_s = (int)std::lround(column_at(dim == 2 ? kLeaf2 : kLeaf3, t));
  P.table_tol = std::max(0.03 * eps, dim == 2 ? 1e-12 : 1e-14);
  return P;
}

int channels_out(int kernel, int dim) {  // params.cpp:117-125
  switch (kernel) {
    case kStokeslet: return dim;
    case kStresslet: return dim * (dim + 1) / 2;
    case kRotlet: return dim == 3 ? 3 : 1;
  }
  throw InvalidArgument("outgoing_channels: unsupported kernel");
}

int strength_width(int kernel, int dim) {  // split.cpp:46-55
  switch (kernel) {
    case kStokeslet: return dim;
    case kStresslet: return 2 * dim;
    case kRotlet: return dim == 3 ? 3 : 1;
    case kBiharmonic:
    case kHarmonic: return 1;
  }
  return 0;
}

// PSWF psi0c in the normalized even-Legendre basis: smallest eigenpair of the
// symmetric tridiagonal prolate operator by Sturm bisection, then inverse
// iteration with one Rayleigh-quotient shift update (prolate.cpp:69-165).
WindowFn make_prolate(double c) {
  if (!(c > 0.0)) throw InvalidArgument("build_prolate: c must be positive");
  double c2 = c * c;
  int m = ((int)std::ceil(2.0 * c) + 60) / 2 + 1;
  std::vector<double> dg(m), of(m - 1);
  for (int j = 0; j < m; ++j) {
    double n = 2.0 * j;
    dg[j] = n * (n + 1.0) + c2 * (2.0 * n * (n + 1) - 1.0) / ((2.0 * n + 3) * (2.0 * n - 1));
  }
  for (int j = 0; j + 1 < m; ++j) {
    double n = 2.0 * j;
    of[j] = c2 * (n + 1.0) * (n + 2.0) / ((2.0 * n + 3) * std::sqrt((2.0 * n + 1) * (2.0 * n + 5)));
  }
  auto below = [&](double x) {  // Sturm count of eigenvalues < x
    int cnt = 0;
    double q = dg[0] - x;
    if (q < 0) ++cnt;
    for (int i = 1; i < m; ++i) {
      q = dg[i] - x - of[i - 1] * of[i - 1] / (q == 0.0 ? 1e-300 : q);
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  double lo = dg[0], hi = dg[0];
  for (int j = 0; j < m; ++j) {
    double rad = (j > 0 ? std::fabs(of[j - 1]) : 0.0) + (j + 1 < m ? std::fabs(of[j]) : 0.0);
    lo = std::min(lo, dg[j] - rad);
    hi = std::max(hi, dg[j] + rad);
  }
  for (int it = 0; it < 200 && hi - lo > 1e-14 * (std::fabs(lo) + std::fabs(hi) + 1.0); ++it) {
    double mid = 0.5 * (lo + hi);
    (below(mid) >= 1 ? hi : lo) = mid;
  }
  double shift = 0.5 * (lo + hi);
  auto rayleigh = [&](const std::vector<double>& v) {
    double r = 0.0;
    for (int j = 0; j < m; ++j) {
      double tv = dg[j] * v[j];
      if (j > 0) tv += of[j - 1] * v[j - 1];
      if (j + 1 < m) tv += of[j] * v[j + 1];
      r += v[j] * tv;
    }
    return r;
  };
  std::vector<double> v(m, 1.0 / std::sqrt((double)m));
  for (int it = 0; it < 6; ++it) {
    // Thomas solve of (T - shift) y = v, in place
    std::vector<double> dd(m), up(of);
    for (int i = 0; i < m; ++i) dd[i] = dg[i] - shift;
    for (int i = 0; i + 1 < m; ++i) {
      if (dd[i] == 0.0) dd[i] = 1e-300;
      double f = of[i] / dd[i];
      dd[i + 1] -= f * up[i];
      v[i + 1] -= f * v[i];
    }
    if (dd[m - 1] == 0.0) dd[m - 1] = 1e-300;
    v[m - 1] /= dd[m - 1];
    for (int i = m - 1; i-- > 0;) v[i] = (v[i] - up[i] * v[i + 1]) / dd[i];
    double nv = 0.0;
    for (double x : v) nv += x * x;
    nv = std::sqrt(nv);
    if (!(nv > 0.0) || !std::isfinite(nv)) throw RuntimeError("build_prolate: inverse iteration failed");
    for (double& x : v) x /= nv;
    if (it == 2) shift = rayleigh(v);
  }
  double chi = rayleigh(v);
  std::vector<double> a(m);
  double amax = 0.0;
  for (int j = 0; j < m; ++j) {
    a[j] = v[j] * std::sqrt((4.0 * j + 1.0) / 2.0);
    amax = std::max(amax, std::fabs(a[j]));
  }
  int keep = m;
  while (keep > 1 && std::fabs(a[keep - 1]) < 1e-16 * amax) --keep;
  a.resize(keep);
  auto D0 = leg_derivs_zero(0, 2 * keep);
  double psi0 = 0.0, psi1 = 0.0;
  for (int j = 0; j < keep; ++j) {
    psi0 += a[j] * D0[0][2 * j];
    psi1 += a[j];
  }
  if (psi0 < 0) {
    for (double& x : a) x = -x;
    psi0 = -psi0;
    psi1 = -psi1;
  }
  WindowFn w;
  w.kind = kProlate;
  w.c = c;
  w.leg = a;
  w.psi0 = psi0;
  w.chi0 = chi;
  double I0 = 2.0 * a[0];
  w.norm_r = 1.0 / I0;
  w.lambda0 = I0 / psi0;
  w.trunc_error = std::fabs(psi1 / psi0);
  return w;
}

WindowFn make_gaussian(double sigma) {  // windows.cpp:45-53
  if (!(sigma > 0.0)) throw InvalidArgument("build_gaussian: sigma must be positive");
  WindowFn w;
  w.kind = kGaussian;
  w.sigma = sigma;
  w.norm_r = 1.0 / (sigma * std::sqrt(M_PI));
  w.trunc_error = std::exp(-1.0 / (sigma * sigma));
  return w;
}

double win_phi(const WindowFn& w, double r) {  // windows.cpp:55-62
  if (w.kind == kGaussian) return std::exp(-r * r / (w.sigma * w.sigma)) * w.norm_r;
  if (std::fabs(r) > 1.0) return 0.0;
  double v;
  psi_at(w, r, 0, &v);
  return v * w.norm_r;
}

double win_dphi(const WindowFn& w, double r) {  // windows.cpp:64-70
  if (w.kind == kGaussian) return -2.0 * r / (w.sigma * w.sigma) * win_phi(w, r);
  if (std::fabs(r) > 1.0) return 0.0;
  double v[2];
  psi_at(w, r, 1, v);
  return v[1] * w.norm_r;
}

double win_hat(const WindowFn& w, double k) {  // windows.cpp:72-78
  if (w.kind == kGaussian) return std::exp(-k * k * w.sigma * w.sigma / 4.0);
  if (std::fabs(k) > w.c) return 0.0;
  double v;
  psi_at(w, k / w.c, 0, &v);
  return v / w.psi0;
}

double win_hat_d(const WindowFn& w, double k, int order) {  // windows.cpp:80-97
  if (order < 1 || order > 3) throw InvalidArgument("window_fourier_deriv: order must be 1..3");
  if (w.kind == kGaussian) {
    double s2 = w.sigma * w.sigma, g = std::exp(-k * k * s2 / 4.0);
    if (order == 1) return -0.5 * k * s2 * g;
    if (order == 2) return (-0.5 * s2 + 0.25 * k * k * s2 * s2) * g;
    return (0.75 * k * s2 * s2 - 0.125 * k * k * k * s2 * s2 * s2) * g;
  }
  if (std::fabs(k) > w.c) return 0.0;
  double v[4];
  psi_at(w, k / w.c, order, v);
  return v[order] / (std::pow(w.c, order) * w.psi0);
}

double win_tail(const WindowFn& w, double r) {  // windows.cpp:99-110
  if (r < 0) r = -r;
  if (w.kind == kGaussian) return std::erfc(r / w.sigma);
  if (r >= 1.0) return 0.0;
  int nmax = 2 * ((int)w.leg.size() - 1) + 1;
  std::vector<double> P(nmax + 1);
  leg_values(r, nmax, P.data());
  double acc = 0.0;
  for (size_t j = 0; j < w.leg.size(); ++j) {
    int n = 2 * (int)j;
    double integral = n == 0 ? 1.0 - r : (P[n - 1] - P[n + 1]) / (2 * n + 1);
    acc += w.leg[j] * integral;
  }
  return 2.0 * acc * w.norm_r;
}

std::array<double, 5> win_hat_taylor(const WindowFn& w) {  // windows.cpp:112-138
  std::array<double, 5> b{};
  if (w.kind == kGaussian) {
    double q = -w.sigma * w.sigma / 4.0, f = 1.0;
    for (int j = 0; j <= 4; ++j) {
      b[j] = f;
      f *= q / (j + 1);
    }
    return b;
  }
  int nmax = 2 * ((int)w.leg.size() - 1);
  auto D = leg_derivs_zero(8, nmax);
  double fact = 1.0, cp = 1.0;
  for (int j = 0; j <= 4; ++j) {
    if (j > 0) {
      fact *= (2.0 * j - 1.0) * (2.0 * j);
      cp *= w.c * w.c;
    }
    double s = 0.0;
    for (size_t m = 0; m < w.leg.size(); ++m) s += w.leg[m] * D[2 * j][2 * m];
    b[j] = s / (cp * fact * w.psi0);
  }
  return b;
}

double moll_hat(const WindowFn& w, double k) {  // split.cpp:68-72
  k = std::fabs(k);
  if (w.kind == kProlate && k >= w.c) return 0.0;
  return win_hat(w, k) - 0.5 * k * win_hat_d(w, k, 1);
}

std::array<double, 5> moll_hat_taylor(const WindowFn& w) {  // split.cpp:74-78
  auto b = win_hat_taylor(w);
  return {b[0], 0.0, -b[2], -2.0 * b[3], -3.0 * b[4]};
}

double trunc_bihar_hat(double k, double R, int dim) {  // symbols.cpp:22-51
  if (dim != 2 && dim != 3) throw InvalidArgument("truncated_biharmonic_fourier: dim must be 2 or 3");
  if (R <= 0.0) throw InvalidArgument("truncated_biharmonic_fourier: R must be positive");
  k = std::fabs(k);
  double u = k * R;
  if (u < 0.1) {
    double u2 = u * u, acc = 0.0, pw = 1.0;
    for (int m = 2; m <= 9; ++m) {
      double den = 1.0;
      if (dim == 3) {
        for (int j = 2; j <= 2 * m + 1; ++j) den *= j;
      } else {
        double fm = 1.0;
        for (int j = 2; j <= m; ++j) fm *= j;
        den = std::pow(4.0, m) * fm * fm;
      }
      acc += ((m % 2 == 0) ? 1.0 : -1.0) * (m - 1) / den * pw;
      pw *= u2;
    }
    return R * R * R * R * acc;
  }
  double k4 = k * k * k * k;
  if (dim == 3) return (1.0 + 0.5 * std::cos(u) - 1.5 * std::sin(u) / u) / k4;
  return (1.0 - std::cyl_bessel_j(0.0, u) - 0.5 * u * std::cyl_bessel_j(1.0, u)) / k4;
}

double trunc_harm_hat(double k, double R, int dim) {  // symbols.cpp:53-92
  if (dim != 2 && dim != 3) throw InvalidArgument("truncated_harmonic_fourier: dim must be 2 or 3");
  if (R <= 0.0) throw InvalidArgument("truncated_harmonic_fourier: R must be positive");
  k = std::fabs(k);
  double u = k * R, R2 = R * R;
  if (dim == 3) {
    if (u < 0.1) {
      double u2 = u * u, acc = 0.0, pw = 1.0, fact = 1.0;
      for (int m = 1; m <= 8; ++m) {
        fact *= (2.0 * m - 1.0) * (2.0 * m);
        acc += ((m % 2 == 1) ? 1.0 : -1.0) * pw / fact;
        pw *= u2;
      }
      return R2 * acc;
    }
    return (1.0 - std::cos(u)) / (k * k);
  }
  double lr = std::log(R);
  if (u < 0.1) {
    double u2 = u * u, s1 = 0.0, s2 = 0.0, pw = 1.0;
    for (int j = 0; j <= 7; ++j) {
      double fj = 1.0;
      for (int i = 2; i <= j; ++i) fj *= i;
      double f1 = fj * (j + 1), p4 = std::pow(4.0, j), sg = (j % 2 == 0) ? 1.0 : -1.0;
      s1 += sg * pw / (4.0 * p4 * f1 * f1);
      s2 += sg * pw / (2.0 * p4 * fj * f1);
      pw *= u2;
    }
    return R2 * (s1 - lr * s2);
  }
  return (1.0 - std::cyl_bessel_j(0.0, u)) / (k * k) - R * lr * std::cyl_bessel_j(1.0, u) / k;
}

double Cheb::eval(double x) const {  // Clenshaw (chebyshev.cpp:9-19)
  if (a.empty()) return 0.0;
  double t = (2.0 * x - lo - hi) / (hi - lo), b1 = 0.0, b2 = 0.0;
  for (size_t k = a.size(); k-- > 1;) {
    double b0 = 2.0 * t * b1 - b2 + a[k];
    b2 = b1;
    b1 = b0;
  }
  return t * b1 - b2 + a[0];
}

PiecewisePoly piecewise_from_cheb(const Cheb& t, int ni, int min_deg, double rel_tol) {
  PiecewisePoly P;
  P.ni = ni;
  P.lo = t.lo;
  P.hi = t.hi;
  if (t.a.empty()) {
    P.deg = min_deg;
    P.c.assign((size_t)ni * (min_deg + 1), 0.0);
    return P;
  }
  double fmax = 0.0;
  for (int j = 0; j <= 4096; ++j) fmax = std::max(fmax, std::fabs(t.eval(t.lo + (t.hi - t.lo) * j / 4096.0)));
  const double tol = rel_tol * std::max(1.0, fmax);
  for (int deg : {4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24}) {
    if (deg < min_deg) continue;
    const int n = deg + 1;
    std::vector<double> c((size_t)ni * n, 0.0);
    double worst = 0.0;
    for (int i = 0; i < ni; ++i) {
      const double a = t.lo + (t.hi - t.lo) * i / ni, b = t.lo + (t.hi - t.lo) * (i + 1) / ni;
      // Chebyshev interpolation coefficients on [a, b]
      std::vector<double> fv(n), ch(n, 0.0);
      for (int j = 0; j < n; ++j) fv[j] = t.eval(0.5 * (a + b) + 0.5 * (b - a) * std::cos(M_PI * (2 * j + 1) / (2.0 * n)));
      for (int k = 0; k < n; ++k) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += fv[j] * std::cos(k * M_PI * (2 * j + 1) / (2.0 * n));
        ch[k] = s * (k == 0 ? 1.0 : 2.0) / n;
      }
      // Chebyshev -> monomials in w = (x - a) / (b - a) in [0, 1] (the kernel's
      // local coordinate, y - floor(y)): shifted Chebyshev polynomials
      // T*_0 = 1, T*_1 = 2w - 1, T*_{k+1} = (4w - 2) T*_k - T*_{k-1}
      std::vector<double> Tk0(n, 0.0), Tk1(n, 0.0), Tk2(n, 0.0);
      double* mono = c.data() + (size_t)i * n;
      Tk0[0] = 1.0;
      for (int j = 0; j < n; ++j) mono[j] += ch[0] * Tk0[j];
      if (n > 1) {
        Tk1[0] = -1.0;
        Tk1[1] = 2.0;
        for (int j = 0; j < n; ++j) mono[j] += ch[1] * Tk1[j];
      }
      for (int k = 2; k < n; ++k) {
        for (int j = 0; j < n; ++j) Tk2[j] = (j ? 4.0 * Tk1[j - 1] : 0.0) - 2.0 * Tk1[j] - Tk0[j];
        for (int j = 0; j < n; ++j) mono[j] += ch[k] * Tk2[j];
        Tk0 = Tk1;
        Tk1 = Tk2;
      }
      for (int j = 0; j <= 64; ++j) {  // check with the same Horner the kernel uses
        const double w = j / 64.0, x = a + (b - a) * w;
        double v = mono[deg];
        for (int k = deg - 1; k >= 0; --k) v = std::fma(v, w, mono[k]);
        worst = std::max(worst, std::fabs(v - t.eval(x)));
      }
    }
    if (worst <= tol || deg == 24) {
      P.deg = deg;
      P.c = c;
      P.max_err = worst;
      return P;
    }
  }
  return P;
}

// Residual tables: closed forms in phi / Phi in 3D (split.cpp:319-381), the
// Fourier quadrature pipeline in 2D (split.cpp:383-395, split2d.cpp:263-326).
Tables build_tables(int kernel, int dim, const WindowFn& win, double tol) {
  if (dim != 2 && dim != 3) throw InvalidArgument("build_split_kernel: dim must be 2 or 3");
  if (!(tol >= 1e-14 && tol <= 1e-3)) throw InvalidArgument("build_split_kernel: tol must lie in [1e-14, 1e-3]");
  if (dim == 2 && (kernel == kBiharmonic || kernel == kHarmonic))
    throw InvalidArgument("build_split_kernel: scalar kernels are built in 3D only");
  Tables T;
  T.kernel = kernel;
  T.dim = dim;
  T.win = win;
  T.R = 1.0 + std::sqrt((double)dim);
  T.support = win.kind == kProlate ? 1.0 : 1.05;
  T.table_tol = tol;
  const WindowFn& w = win;
  double sup = T.support;
  if (dim == 3) {
    const double ft = 1e-14;
    T.phi = cheb_fit([&](double r) { return win_tail(w, r); }, 0.0, sup, ft);
    switch (kernel) {
      case kStokeslet:
        T.s_diag = cheb_fit([&](double r) { return win_tail(w, r) - 2.0 * r * win_phi(w, r); }, 0.0, sup, ft);
        T.s_offd = cheb_fit([&](double r) { return win_tail(w, r) + 2.0 * r * win_phi(w, r); }, 0.0, sup, ft);
        T.self_const = -win_phi(w, 0.0) / (2.0 * PI);
        T.corr_const = 1.0 / (4.0 * PI * T.R);
        break;
      case kStresslet:
        T.t_diag = cheb_fit([&](double r) { return -2.0 * r * r * win_dphi(w, r); }, 0.0, sup, ft);
        T.t_offd = cheb_fit(
            [&](double r) {
              return win_tail(w, r) + 2.0 * r * win_phi(w, r) - (2.0 / 3.0) * r * r * win_dphi(w, r);
            },
            0.0, sup, ft);
        break;
      case kRotlet:
        T.w_offd = cheb_fit([&](double r) { return win_tail(w, r) + 2.0 * r * win_phi(w, r); }, 0.0, sup, ft);
        break;
      case kBiharmonic:
        T.b_res = cheb_fit(
            [&](double r) { return -(r * win_tail(w, r) - 2.0 * tail_moment(w, r)) / (8.0 * PI); }, 0.0,
            sup, ft);
        T.self_const = tail_moment(w, 0.0) / (4.0 * PI);
        break;
      case kHarmonic:
        T.self_const = -win_phi(w, 0.0) / (2.0 * PI);
        break;
    }
    return T;
  }
  // 2D numeric pipeline
  double R = T.R;
  Quad q = converged_quad(kernel, dim, w, R, tol, sup);
  double ft = std::max(1e-13, 0.05 * tol);
  if (kernel == kStokeslet) {
    T.s_diag = cheb_fit([&](double r) { return moll_struct(q, kernel, dim, R, r)[0]; }, 0.0, sup, ft);
    T.s_offd = cheb_fit([&](double r) { return 2.0 * r - moll_struct(q, kernel, dim, R, r)[1]; }, 0.0, sup, ft);
    double lam = 0.0;
    for (size_t i = 0; i < q.k.size(); ++i) lam += q.wb[i] * q.k[i] * q.k[i];
    lam *= 4.0 * PI;
    lam += 2.0 * (1.0 - std::log(R));
    T.self_const = -lam / (8.0 * PI);
    T.corr_const = (1.0 - std::log(R)) / (4.0 * PI);
  } else if (kernel == kStresslet) {
    T.t_diag = cheb_fit([&](double r) { return -moll_struct(q, kernel, dim, R, r)[0]; }, 0.0, sup, ft);
    T.t_offd = cheb_fit([&](double r) { return 4.0 * r / 3.0 - moll_struct(q, kernel, dim, R, r)[1]; }, 0.0,
                        sup, ft);
  } else if (kernel == kRotlet) {
    T.w_offd = cheb_fit([&](double r) { return 1.0 - moll_struct(q, kernel, dim, R, r)[1]; }, 0.0, sup, ft);
  }
  return T;
}

Tables tables_for_plan(const Plan& P) {  // dmk.cpp:1059-1068
  WindowFn w = P.window == kProlate ? make_prolate(P.c) : make_gaussian(P.sigma);
  double tt = P.table_tol > 0.0 ? P.table_tol : std::max(0.03 * P.tol, P.dim == 2 ? 1e-12 : 1e-14);
  return build_tables(P.kernel, P.dim, w, tt);
}

double self_scaled(const Tables& t, double nu) {  // split.cpp:116-127
  switch (t.kernel) {
    case kStresslet:
    case kRotlet: return 0.0;
    case kStokeslet: return t.dim == 2 ? t.self_const + std::log(nu) / (4.0 * PI) : t.self_const / nu;
    case kHarmonic: return t.self_const / nu;
    case kBiharmonic: return t.self_const * nu;
  }
  return 0.0;
}

// -------------------------------------------------- SDMKSPLT v1 files ----
// Little-endian binary table cache, byte-compatible with the reference's
// export/import (split.cpp:402-506).
namespace {
template <class T>
void wr(std::string& o, T v) { o.append(reinterpret_cast<const char*>(&v), sizeof(T)); }
struct Reader {
  const char* p;
  size_t n, at = 0;
  bool ok = true;
  template <class T>
  T rd() {
    T v{};
    if (at + sizeof(T) > n) {
      ok = false;
      return v;
    }
    std::memcpy(&v, p + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
};
}  // namespace

std::string serialize_tables(const Tables& t) {
  std::string o("SDMKSPLT", 8);
  wr<uint32_t>(o, 1);
  wr<int32_t>(o, t.kernel);
  wr<int32_t>(o, t.dim);
  wr<int32_t>(o, t.win.kind);
  wr<double>(o, t.win.c);
  wr<double>(o, t.win.sigma);
  wr<uint32_t>(o, (uint32_t)t.win.leg.size());
  for (double v : t.win.leg) wr<double>(o, v);
  for (double v : {t.win.lambda0, t.win.norm_r, t.win.trunc_error, t.win.psi0, t.win.chi0, t.R, t.support,
                   t.table_tol, t.self_const, t.corr_const})
    wr<double>(o, v);
  for (const Cheb* c : {&t.s_diag, &t.s_offd, &t.t_diag, &t.t_offd, &t.w_offd, &t.b_res, &t.phi}) {
    wr<double>(o, c->lo);
    wr<double>(o, c->hi);
    wr<uint32_t>(o, (uint32_t)c->a.size());
    for (double v : c->a) wr<double>(o, v);
  }
  return o;
}

Tables parse_tables(const void* bytes, size_t n, const std::string& what) {
  Reader r{static_cast<const char*>(bytes), n};
  if (n < 8 || std::memcmp(bytes, "SDMKSPLT", 8) != 0) throw RuntimeError("import_split_kernel: bad magic in " + what);
  r.at = 8;
  if (r.rd<uint32_t>() != 1) throw RuntimeError("import_split_kernel: unsupported version");
  Tables t;
  t.kernel = r.rd<int32_t>();
  t.dim = r.rd<int32_t>();
  t.win.kind = r.rd<int32_t>();
  t.win.c = r.rd<double>();
  t.win.sigma = r.rd<double>();
  const uint32_t nl = r.rd<uint32_t>();
  if (!r.ok || nl > n / 8) throw RuntimeError("import_split_kernel: truncated file " + what);
  t.win.leg.resize(nl);
  for (double& v : t.win.leg) v = r.rd<double>();
  double* scal[] = {&t.win.lambda0, &t.win.norm_r, &t.win.trunc_error, &t.win.psi0, &t.win.chi0, &t.R,
                    &t.support, &t.table_tol, &t.self_const, &t.corr_const};
  for (double* s : scal) *s = r.rd<double>();
  for (Cheb* c : {&t.s_diag, &t.s_offd, &t.t_diag, &t.t_offd, &t.w_offd, &t.b_res, &t.phi}) {
    c->lo = r.rd<double>();
    c->hi = r.rd<double>();
    const uint32_t m = r.rd<uint32_t>();
    if (!r.ok || m > n / 8) throw RuntimeError("import_split_kernel: truncated file " + what);
    c->a.resize(m);
    for (double& v : c->a) v = r.rd<double>();
  }
  if (!r.ok) throw RuntimeError("import_split_kernel: truncated file " + what);
  return t;
}

void save_tables(const Tables& t, const std::string& path) {
  std::ofstream o(path, std::ios::binary);
  if (!o) throw RuntimeError("export_split_kernel: cannot open " + path);
  const std::string b = serialize_tables(t);
  o.write(b.data(), (std::streamsize)b.size());
  if (!o) throw RuntimeError("export_split_kernel: write failed for " + path);
}

Tables load_tables(const std::string& path) {
  std::ifstream i(path, std::ios::binary);
  if (!i) throw RuntimeError("import_split_kernel: cannot open " + path);
  std::string b((std::istreambuf_iterator<char>(i)), std::istreambuf_iterator<char>());
  return parse_tables(b.data(), b.size(), path);
}

// ------------------------------------------------------ symbol tables ----
// Radial symbol factor by integer |m|^2 on one grid (dmk.cpp:259-318).
std::vector<double> symbol_table(const Tables& t, double h, int s2max, int kind, double rc, double rf) {
  const bool harm = t.kernel == kRotlet;
  const WindowFn& w = t.win;
  auto a = moll_hat_taylor(w);
  double b4 = -a[2], b6 = -a[3] / 2.0, h0 = 0.02, h02 = h0 * h0;
  double b2 = (win_hat(w, h0) - 1.0) / h02 - b4 * h02 - b6 * h02 * h02;
  double rc2 = rc * rc, rf2 = rf * rf;
  std::vector<double> A(s2max + 1, 0.0);
  for (int s2 = 0; s2 <= s2max; ++s2) {
    double k = h * std::sqrt((double)s2), k2 = k * k, v = 0.0;
    if (kind == kRootFree) {
      v = harm ? win_hat(w, k) * trunc_harm_hat(k, t.R, t.dim) : moll_hat(w, k) * trunc_bihar_hat(k, t.R, t.dim);
    } else if (kind == kRootPeriodic) {
      if (s2 != 0) v = harm ? win_hat(w, k) / k2 : moll_hat(w, k) / (k2 * k2);
    } else if (k * rc < 0.05) {
      if (harm)
        v = b2 * (rf2 - rc2) + b4 * (rf2 * rf2 - rc2 * rc2) * k2 + b6 * (rf2 * rf2 * rf2 - rc2 * rc2 * rc2) * k2 * k2;
      else
        v = a[2] * (rf2 * rf2 - rc2 * rc2) + a[3] * (rf2 * rf2 * rf2 - rc2 * rc2 * rc2) * k2 +
            a[4] * (rf2 * rf2 * rf2 * rf2 - rc2 * rc2 * rc2 * rc2) * k2 * k2;
    } else if (harm) {
      v = (win_hat(w, k * rf) - win_hat(w, k * rc)) / k2;
    } else {
      v = (moll_hat(w, k * rf) - moll_hat(w, k * rc)) / (k2 * k2);
    }
    A[s2] = v;
  }
  return A;
}

}  // namespace sdmkb
