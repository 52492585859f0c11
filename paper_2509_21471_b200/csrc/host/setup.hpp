// Host-side setup for the B200 DMK path: tuned plan, PSWF / Gaussian window,
// unit-scale residual Chebyshev tables and per-level Fourier symbol tables.
// This is one-time, per-plan work; the hot path consumes
// its outputs as uploaded device tables.  Everything here restates the
// reference's published algorithm in our own code (citations per function in
// setup.cpp); nothing is linked from the reference.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace sdmkb {

enum Kernel : int { kStokeslet = 0, kStresslet = 1, kRotlet = 2, kBiharmonic = 3, kHarmonic = 4 };
enum WindowKind : int { kProlate = 0, kGaussian = 1 };

// Same field order/meaning as stokesdmk::DmkPlan (dmk.hpp:27-40).
struct Plan {
  int kernel = kStokeslet;
  int dim = 3;
  int window = kProlate;
  double tol = 1e-6;
  double c = 0.0;
  double sigma = 0.0;
  int p = 0;
  int N1 = 0;
  int N_per = 0;
  int n_s = 0;
  double table_tol = 0.0;
};

// Thrown for bad arguments; mapped to SDMK_EINVAL at the C-ABI.
struct InvalidArgument : std::exception {
  std::string msg;
  explicit InvalidArgument(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
struct DomainError : std::exception {
  std::string msg;
  explicit DomainError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
struct RuntimeError : std::exception {
  std::string msg;
  explicit RuntimeError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

Plan select_plan(int kernel, double eps, int window, int dim);
int channels_out(int kernel, int dim);     // outgoing proxy channels
int strength_width(int kernel, int dim);   // doubles per source strength

struct WindowFn {
  int kind = kProlate;
  double c = 0.0, sigma = 0.0;
  std::vector<double> leg;  // coefficients of P_{2j} in psi0c
  double lambda0 = 0.0, norm_r = 0.0, trunc_error = 0.0, psi0 = 0.0, chi0 = 0.0;
};

WindowFn make_prolate(double c);
WindowFn make_gaussian(double sigma);
double win_phi(const WindowFn& w, double r);            // phi(r)
double win_dphi(const WindowFn& w, double r);           // phi'(r)
double win_hat(const WindowFn& w, double k);            // phi_hat(k)
double win_hat_d(const WindowFn& w, double k, int order);
double win_tail(const WindowFn& w, double r);           // Phi(r) = 2 int_r^inf phi
std::array<double, 5> win_hat_taylor(const WindowFn& w);
double moll_hat(const WindowFn& w, double k);           // gamma_hat(k)
std::array<double, 5> moll_hat_taylor(const WindowFn& w);
double trunc_bihar_hat(double k, double R, int dim);
double trunc_harm_hat(double k, double R, int dim);

struct Cheb {
  double lo = 0.0, hi = 1.0;
  std::vector<double> a;
  double eval(double x) const;
};

struct Tables {
  int kernel = kStokeslet;
  int dim = 3;
  WindowFn win;
  double R = 0.0, support = 1.0, table_tol = 0.0, self_const = 0.0, corr_const = 0.0;
  Cheb s_diag, s_offd, t_diag, t_offd, w_offd, b_res, phi;
};

// Piecewise monomial re-expansion of a Chebyshev table for the GPU residual
// kernel: ni equal sub-intervals of [lo, hi], degree deg in the local
// variable u in [-1, 1]; c[i * (deg + 1) + k] multiplies u^k.  Built by
// interpolating the table at Chebyshev points of each sub-interval and
// accepted only if it reproduces the table's Clenshaw value to
// 4e-15 * max(1, |f|) on a dense check grid (else the degree grows).
struct PiecewisePoly {
  int ni = 0, deg = 0;
  double lo = 0.0, hi = 1.0, max_err = 0.0;
  std::vector<double> c;
};
// Piecewise monomial re-expansion of a Chebyshev table: ni equal intervals,
// coefficients in the local coordinate w in [0, 1] of each interval; the
// lowest degree >= min_deg whose Horner values stay within rel_tol * max(1, max|t|)
// of the Chebyshev table on every interval (checked at 65 points per interval)
PiecewisePoly piecewise_from_cheb(const Cheb& t, int ni = 32, int min_deg = 8, double rel_tol = 4e-15);

Tables build_tables(int kernel, int dim, const WindowFn& win, double tol);
// tables exactly as evaluate_with_plan builds them when none are supplied
Tables tables_for_plan(const Plan& plan);
void save_tables(const Tables& t, const std::string& path);  // SDMKSPLT v1
Tables load_tables(const std::string& path);
// the same format in memory (the C++ drop-in's SplitKernel travels as it)
std::string serialize_tables(const Tables& t);
Tables parse_tables(const void* bytes, size_t n, const std::string& what = "memory image");
double self_scaled(const Tables& t, double nu);

enum SymbolKind { kLevelDiff = 0, kRootFree = 1, kRootPeriodic = 2 };
std::vector<double> symbol_table(const Tables& t, double h, int s2max, int kind,
                                 double r_coarse, double r_fine);

}  // namespace sdmkb
