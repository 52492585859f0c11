// Drop-in C++ front end for the B200 DMK path (header-only).
//
// Mirrors the reference's public API (proj/core/include/stokesdmk/dmk.hpp,
// tree.hpp, oracle.hpp, split.hpp, windows.hpp, chebyshev.hpp) so that the
// reference's call sites -- the CLI's make_tables()/timed_evaluate()
// (cli_main.cpp:104-204), the pass-level tests, the acceptance gate and the
// benchmarks (bench_main.cpp:98-132) -- compile unchanged against it:
//
//   #include <stokesdmk_b200/dmk.hpp>      // instead of <stokesdmk/dmk.hpp>
//   using namespace stokesdmk;
//   DmkPlan plan = select_parameters(KernelType::stokeslet, 1e-6, WindowKind::prolate, 3);
//   SplitKernel sk = build_split_kernel(plan.kernel, plan.dim, build_prolate(plan.c), plan.table_tol);
//   std::vector<double> u = evaluate_with_plan(plan, sys, EwaldMode::free_space, &rep, &sk);
//
//   Tree t = build_tree(sys.sources, sys.targets, plan.n_s, 3, false, plan.p);
//   ProxyData og = upward_pass(t, plan, sys.strengths);
//   ProxyData in = make_incoming(t, plan);
//   root_far_field(t, plan, sk, og, false, in);
//   downward_pass(t, plan, sk, og, false, in);
//   std::vector<double> far = target_far_fields(t, plan, in);
//   std::vector<double> res = residual_pass(t, plan, sk, sys.strengths, false);
//
// Everything computes through the extern "C" ABI in <sdmk.h> on the GPU; the
// status codes are rethrown as the reference's exception types
// (std::invalid_argument, std::domain_error, std::runtime_error).
//  * SplitKernel carries the real tables (the same fields as split.hpp:62-80);
//    it crosses the ABI as its SDMKSPLT v1 image (split.cpp:402-506), so a
//    table set built, imported or edited by the caller is the one evaluated.
//  * A Tree holds the reference's fields (boxes, level lists, neighbour
//    lists, permuted points, permutations, quantized coordinates) plus a
//    handle to its device-resident copy, on which the passes run; ProxyData
//    are host arrays in the reference's layout, moved in and out per pass.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sdmk.h"

namespace stokesdmk {

enum class KernelType { stokeslet, stresslet, rotlet, biharmonic, harmonic };
enum class WindowKind { prolate, gaussian };
enum class EwaldMode { free_space, periodic };

// ---- oracle.hpp:29-46 ----
struct ParticleSystem {
  int dim = 3;
  std::vector<double> sources;
  std::vector<double> targets;
  std::vector<double> strengths;
  int num_sources() const { return static_cast<int>(sources.size()) / dim; }
  bool targets_alias_sources() const { return targets.empty(); }
  int num_targets() const {
    return targets_alias_sources() ? num_sources() : static_cast<int>(targets.size()) / dim;
  }
  const double* source(int a) const { return sources.data() + a * dim; }
  const double* target(int b) const { return (targets_alias_sources() ? sources.data() : targets.data()) + b * dim; }
};

// ---- dmk.hpp:27-40, 134-145 ----
struct DmkPlan {
  KernelType kernel = KernelType::stokeslet;
  int dim = 3;
  WindowKind window = WindowKind::prolate;
  double tol = 1e-6;
  double c = 0.0;
  double sigma = 0.0;
  int p = 0;
  int N1 = 0;
  int N_per = 0;
  int n_s = 0;
  double table_tol = 0.0;
};

struct DmkReport {
  DmkPlan plan;
  int num_boxes = 0;
  int max_level = 0;
  int num_sources = 0;
  int num_targets = 0;
  double t_tree = 0.0;
  double t_upward = 0.0;
  double t_root = 0.0;
  double t_downward = 0.0;
  double t_residual = 0.0;
};

// ---- windows.hpp:23-38 ----
struct WindowFunction {
  WindowKind kind = WindowKind::prolate;
  double c = 0.0;
  double sigma = 0.0;
  std::vector<double> legendre_coeffs;
  double lambda0 = 0.0;
  double norm_r = 0.0;
  double trunc_error = 0.0;
  double psi0 = 0.0;
  double chi0 = 0.0;
};

// ---- chebyshev.hpp:13-19 ----
struct ChebTable {
  double lo = 0.0, hi = 1.0;
  std::vector<double> coef;
  double eval(double x) const {  // Clenshaw (chebyshev.cpp:9-19)
    if (coef.empty()) return 0.0;
    double t = (2.0 * x - lo - hi) / (hi - lo);
    double b1 = 0.0, b2 = 0.0;
    for (size_t k = coef.size(); k-- > 1;) {
      double b0 = 2.0 * t * b1 - b2 + coef[k];
      b2 = b1;
      b1 = b0;
    }
    return t * b1 - b2 + coef[0];
  }
  bool empty() const { return coef.empty(); }
};

// ---- split.hpp:37-80 ----
struct Mollifier {
  WindowFunction window;
};

struct SplitKernel {
  KernelType kernel = KernelType::stokeslet;
  int dim = 3;
  Mollifier mollifier;
  double window_radius_R = 0.0;
  double support = 1.0;
  double table_tol = 0.0;
  double self_const = 0.0;
  double corr_const = 0.0;
  ChebTable s_diag, s_offd;
  ChebTable t_diag, t_offd;
  ChebTable w_offd;
  ChebTable b_res;
  ChebTable phi;
};

// ---- tree.hpp:21-81 ----
inline constexpr int kTreeMaxLevel = 30;

struct TreeBox {
  int level = 0;
  int parent = -1;
  int first_child = -1;
  bool leaf = true;
  std::array<std::int32_t, 3> anchor = {0, 0, 0};
  int src_begin = 0, src_end = 0;
  int tgt_begin = 0, tgt_end = 0;
};

struct NeighborEntry {
  int box = -1;
  std::array<std::int8_t, 3> shift = {0, 0, 0};
};

struct TreeNeighbors {
  std::vector<NeighborEntry> colleagues;
  std::vector<NeighborEntry> coarse;
  std::vector<NeighborEntry> fine;
};

namespace detail {
struct TreeState;
}

struct Tree {
  int dim = 3;
  bool periodic = false;
  int n_s = 0;
  int proxy_order = 0;
  int max_level = 0;
  bool depth_capped = false;
  bool targets_alias_sources = false;

  std::vector<TreeBox> boxes;
  std::vector<std::vector<int>> level_boxes;
  std::vector<TreeNeighbors> neighbors;

  std::vector<double> src_points, tgt_points;
  std::vector<int> src_perm, tgt_perm;
  std::vector<std::array<std::int32_t, 3>> src_q, tgt_q;

  int num_boxes() const { return static_cast<int>(boxes.size()); }
  double box_side(int b) const { return std::ldexp(1.0, -boxes[b].level); }
  std::array<double, 3> box_center(int b) const {  // tree.cpp:221-228
    std::array<double, 3> c = {0.0, 0.0, 0.0};
    const double side = box_side(b);
    for (int i = 0; i < dim; ++i) c[i] = std::ldexp(double(boxes[b].anchor[i]), -kTreeMaxLevel) - 0.5 + 0.5 * side;
    return c;
  }
  int box_src_count(int b) const { return boxes[b].src_end - boxes[b].src_begin; }
  int box_tgt_count(int b) const { return boxes[b].tgt_end - boxes[b].tgt_begin; }

  // B200: the device-resident copy the passes run on (shared by copies)
  std::shared_ptr<detail::TreeState> device;
};

// ---- dmk.hpp:64-79 ----
struct ProxyData {
  int p = 0;
  int dim = 3;
  int channels = 0;
  std::vector<double> values;

  int nodes_per_box() const {
    int n = p * p;
    return dim == 3 ? n * p : n;
  }
  int box_stride() const { return channels * nodes_per_box(); }
  double* box(int id) { return values.data() + size_t(id) * box_stride(); }
  const double* box(int id) const { return values.data() + size_t(id) * box_stride(); }
};

namespace detail {

inline void check(int code) {
  if (code == SDMK_OK) return;
  std::string msg = sdmk_last_error();
  if (code == SDMK_EINVAL) throw std::invalid_argument(msg);
  if (code == SDMK_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

inline int& device_slot() {
  static thread_local int dev = 0;
  return dev;
}

struct ContextHolder {
  sdmk_context* c = nullptr;
  ~ContextHolder() {
    if (c) sdmk_destroy(c);
  }
};

inline ContextHolder& holder() {
  static thread_local ContextHolder h;
  return h;
}

inline sdmk_context* context() {
  ContextHolder& h = holder();
  if (!h.c) check(sdmk_create(device_slot(), &h.c));
  return h.c;
}

// Trees keep their own context (device-resident tree + arenas); released
// contexts are pooled per thread so repeated build_tree calls reuse buffers.
struct ContextPool {
  std::vector<sdmk_context*> free;
  ~ContextPool() {
    for (sdmk_context* c : free) sdmk_destroy(c);
  }
};
inline ContextPool& pool() {
  static thread_local ContextPool p;
  return p;
}

struct TreeState {
  sdmk_context* ctx = nullptr;
  int device = 0;
  explicit TreeState(int dev) : device(dev) {
    ContextPool& p = pool();
    if (!p.free.empty() && device_slot() == dev) {
      ctx = p.free.back();
      p.free.pop_back();
    } else {
      check(sdmk_create(dev, &ctx));
    }
  }
  ~TreeState() {
    if (!ctx) return;
    ContextPool& p = pool();
    if (p.free.size() < 4 && device_slot() == device)
      p.free.push_back(ctx);
    else
      sdmk_destroy(ctx);
  }
  TreeState(const TreeState&) = delete;
  TreeState& operator=(const TreeState&) = delete;
};

inline sdmk_context* tree_context(const Tree& t, const char* who) {
  if (!t.device || !t.device->ctx)
    throw std::invalid_argument(std::string(who) + ": tree was not built by build_tree (no device copy)");
  return t.device->ctx;
}

inline sdmk_plan to_c(const DmkPlan& p) {
  sdmk_plan c;
  c.kernel = static_cast<int32_t>(p.kernel);
  c.dim = p.dim;
  c.window = static_cast<int32_t>(p.window);
  c.tol = p.tol;
  c.c = p.c;
  c.sigma = p.sigma;
  c.p = p.p;
  c.N1 = p.N1;
  c.N_per = p.N_per;
  c.n_s = p.n_s;
  c.table_tol = p.table_tol;
  return c;
}

inline DmkPlan from_c(const sdmk_plan& c) {
  DmkPlan p;
  p.kernel = static_cast<KernelType>(c.kernel);
  p.dim = c.dim;
  p.window = static_cast<WindowKind>(c.window);
  p.tol = c.tol;
  p.c = c.c;
  p.sigma = c.sigma;
  p.p = c.p;
  p.N1 = c.N1;
  p.N_per = c.N_per;
  p.n_s = c.n_s;
  p.table_tol = c.table_tol;
  return p;
}

// ---- SDMKSPLT v1 (split.cpp:402-506): little-endian, fixed field order ----
template <class T>
inline void put(std::string& o, T v) {
  o.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

inline std::string table_image(const SplitKernel& sk) {
  const WindowFunction& w = sk.mollifier.window;
  std::string o("SDMKSPLT", 8);
  put<uint32_t>(o, 1);
  put<int32_t>(o, static_cast<int32_t>(sk.kernel));
  put<int32_t>(o, sk.dim);
  put<int32_t>(o, static_cast<int32_t>(w.kind));
  put<double>(o, w.c);
  put<double>(o, w.sigma);
  put<uint32_t>(o, static_cast<uint32_t>(w.legendre_coeffs.size()));
  for (double v : w.legendre_coeffs) put<double>(o, v);
  for (double v : {w.lambda0, w.norm_r, w.trunc_error, w.psi0, w.chi0, sk.window_radius_R, sk.support, sk.table_tol,
                   sk.self_const, sk.corr_const})
    put<double>(o, v);
  for (const ChebTable* t : {&sk.s_diag, &sk.s_offd, &sk.t_diag, &sk.t_offd, &sk.w_offd, &sk.b_res, &sk.phi}) {
    put<double>(o, t->lo);
    put<double>(o, t->hi);
    put<uint32_t>(o, static_cast<uint32_t>(t->coef.size()));
    for (double v : t->coef) put<double>(o, v);
  }
  return o;
}

struct ImageReader {
  const std::string& s;
  size_t at = 0;
  std::string what;
  template <class T>
  T get() {
    if (at + sizeof(T) > s.size()) throw std::runtime_error("import_split_kernel: truncated file " + what);
    T v;
    std::memcpy(&v, s.data() + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
};

inline SplitKernel parse_image(const std::string& img, const std::string& what) {
  if (img.size() < 8 || std::memcmp(img.data(), "SDMKSPLT", 8) != 0)
    throw std::runtime_error("import_split_kernel: bad magic in " + what);
  ImageReader r{img, 8, what};
  if (r.get<uint32_t>() != 1) throw std::runtime_error("import_split_kernel: unsupported version");
  SplitKernel sk;
  WindowFunction& w = sk.mollifier.window;
  sk.kernel = static_cast<KernelType>(r.get<int32_t>());
  sk.dim = r.get<int32_t>();
  w.kind = static_cast<WindowKind>(r.get<int32_t>());
  w.c = r.get<double>();
  w.sigma = r.get<double>();
  w.legendre_coeffs.resize(r.get<uint32_t>());
  for (double& v : w.legendre_coeffs) v = r.get<double>();
  for (double* v : {&w.lambda0, &w.norm_r, &w.trunc_error, &w.psi0, &w.chi0, &sk.window_radius_R, &sk.support,
                    &sk.table_tol, &sk.self_const, &sk.corr_const})
    *v = r.get<double>();
  for (ChebTable* t : {&sk.s_diag, &sk.s_offd, &sk.t_diag, &sk.t_offd, &sk.w_offd, &sk.b_res, &sk.phi}) {
    t->lo = r.get<double>();
    t->hi = r.get<double>();
    t->coef.resize(r.get<uint32_t>());
    for (double& v : t->coef) v = r.get<double>();
  }
  return sk;
}

inline const unsigned char* bytes(const std::string& s) { return reinterpret_cast<const unsigned char*>(s.data()); }

// validate_system's length checks (oracle.cpp:103-118), before any array is read
inline void check_lengths(KernelType kernel, const ParticleSystem& sys) {
  if (kernel != KernelType::stokeslet && kernel != KernelType::stresslet && kernel != KernelType::rotlet)
    throw std::invalid_argument("particle sums support the Stokeslet, stresslet, and rotlet kernels");
  const int d = sys.dim;
  if (d != 2 && d != 3) throw std::invalid_argument("ParticleSystem: dim must be 2 or 3");
  if (sys.sources.empty() || sys.sources.size() % d != 0)
    throw std::invalid_argument("ParticleSystem: bad source array length");
  if (!sys.targets.empty() && sys.targets.size() % d != 0)
    throw std::invalid_argument("ParticleSystem: bad target array length");
  const size_t n = sys.sources.size() / d;
  const size_t nc = static_cast<size_t>(sdmk_strength_components(static_cast<int>(kernel), d));
  if (sys.strengths.size() != n * nc) throw std::invalid_argument("ParticleSystem: bad strength array length");
}

inline void check_tree_plan(const Tree& tree, const DmkPlan& plan) {  // dmk.cpp:534-539
  if (tree.dim != plan.dim) throw std::invalid_argument("dmk: tree and plan dimensions differ");
  if (tree.proxy_order != plan.p) throw std::invalid_argument("dmk: tree proxy order does not match plan");
}

inline std::vector<double> window_eval_n(const WindowFunction& w, int what, const double* x, int64_t n) {
  double sc[5] = {w.lambda0, w.norm_r, w.trunc_error, w.psi0, w.chi0};
  std::vector<double> out(static_cast<size_t>(n));
  check(sdmk_host_window_eval(static_cast<int>(w.kind), w.c, w.sigma, w.legendre_coeffs.data(),
                              static_cast<int>(w.legendre_coeffs.size()), sc, what, n, x, out.data()));
  return out;
}

}  // namespace detail

// ---- split.cpp:46-66 / params.cpp:117-125 ----
inline int strength_components(KernelType kernel, int dim) {
  return sdmk_strength_components(static_cast<int>(kernel), dim);
}
inline int field_components(KernelType kernel, int dim) {
  return (kernel == KernelType::biharmonic || kernel == KernelType::harmonic) ? 1 : dim;
}

inline DmkPlan select_parameters(KernelType kernel, double eps, WindowKind window, int dim) {
  sdmk_plan c;
  detail::check(sdmk_select_parameters(static_cast<int>(kernel), eps, static_cast<int>(window), dim, &c));
  return detail::from_c(c);
}

inline int outgoing_channels(KernelType kernel, int dim) {
  int r = sdmk_outgoing_channels(static_cast<int>(kernel), dim);
  if (r < 0) throw std::invalid_argument("outgoing_channels: unsupported kernel");
  return r;
}

// ---- windows.hpp:40-56 ----
inline WindowFunction build_window_(WindowKind kind, double c, double sigma) {
  WindowFunction w;
  w.kind = kind;
  w.c = c;
  w.sigma = sigma;
  double sc[5];
  int n = sdmk_host_build_window(static_cast<int>(kind), c, sigma, sc, nullptr, 0);
  if (n < 0) detail::check(SDMK_EINVAL);
  w.legendre_coeffs.resize(static_cast<size_t>(n));
  detail::check(sdmk_host_build_window(static_cast<int>(kind), c, sigma, sc, w.legendre_coeffs.data(), n) < 0
                    ? SDMK_EINVAL
                    : SDMK_OK);
  w.lambda0 = sc[0];
  w.norm_r = sc[1];
  w.trunc_error = sc[2];
  w.psi0 = sc[3];
  w.chi0 = sc[4];
  return w;
}
inline WindowFunction build_prolate(double c) {
  if (!(c > 0.0)) throw std::invalid_argument("build_prolate: c must be positive");
  return build_window_(WindowKind::prolate, c, 0.0);
}
inline WindowFunction build_gaussian(double sigma) {
  if (!(sigma > 0.0)) throw std::invalid_argument("build_gaussian: sigma must be positive");
  return build_window_(WindowKind::gaussian, 0.0, sigma);
}
inline double window_eval(const WindowFunction& w, double r) { return detail::window_eval_n(w, 0, &r, 1)[0]; }
inline double window_deriv(const WindowFunction& w, double r) { return detail::window_eval_n(w, 1, &r, 1)[0]; }
inline double window_fourier(const WindowFunction& w, double k) { return detail::window_eval_n(w, 2, &k, 1)[0]; }
inline double phi_tail(const WindowFunction& w, double r) { return detail::window_eval_n(w, 3, &r, 1)[0]; }
inline double mollifier_fourier(const Mollifier& m, double k) {
  return detail::window_eval_n(m.window, 4, &k, 1)[0];
}

// ---- split.hpp:82-154 ----
inline SplitKernel build_split_kernel(KernelType kernel, int dim, const WindowFunction& window, double tol) {
  const int k = static_cast<int>(kernel), wk = static_cast<int>(window.kind);
  int64_t n = sdmk_host_build_tables(k, dim, wk, window.c, window.sigma, tol, nullptr, 0);
  if (n < 0) detail::check(sdmk_last_error()[0] ? SDMK_EINVAL : SDMK_ERUNTIME);
  std::string img(static_cast<size_t>(n), '\0');
  if (sdmk_host_build_tables(k, dim, wk, window.c, window.sigma, tol, reinterpret_cast<unsigned char*>(&img[0]), n) != n)
    detail::check(SDMK_ERUNTIME);
  return detail::parse_image(img, "build_split_kernel");
}

inline void export_split_kernel(const SplitKernel& sk, const std::string& path) {
  std::ofstream o(path, std::ios::binary);
  if (!o) throw std::runtime_error("export_split_kernel: cannot open " + path);
  const std::string img = detail::table_image(sk);
  o.write(img.data(), static_cast<std::streamsize>(img.size()));
  if (!o) throw std::runtime_error("export_split_kernel: write failed for " + path);
}

inline SplitKernel import_split_kernel(const std::string& path) {
  std::ifstream i(path, std::ios::binary);
  if (!i) throw std::runtime_error("import_split_kernel: cannot open " + path);
  std::string img((std::istreambuf_iterator<char>(i)), std::istreambuf_iterator<char>());
  return detail::parse_image(img, path);
}

inline double self_interaction(const SplitKernel& sk) { return sk.self_const; }

inline double self_interaction_scaled(const SplitKernel& sk, double nu) {  // split.cpp:116-127
  switch (sk.kernel) {
    case KernelType::stresslet:
    case KernelType::rotlet: return 0.0;
    case KernelType::stokeslet:
      if (sk.dim == 2) return sk.self_const + std::log(nu) / (4.0 * 3.141592653589793238462643383279502884);
      return sk.self_const / nu;
    case KernelType::harmonic: return sk.self_const / nu;
    case KernelType::biharmonic: return sk.self_const * nu;
  }
  return 0.0;
}

// ---- oracle.hpp:48-58 ----
inline void validate_system(KernelType kernel, const ParticleSystem& sys, bool periodic) {  // oracle.cpp:103-131
  detail::check_lengths(kernel, sys);
  for (double v : sys.strengths)
    if (!std::isfinite(v)) throw std::invalid_argument("ParticleSystem: non-finite strength");
  for (const std::vector<double>* pts : {&sys.sources, &sys.targets})
    for (double v : *pts) {
      if (!std::isfinite(v)) throw std::invalid_argument("ParticleSystem: non-finite coordinate");
      if (!periodic && (v < -0.5 || v > 0.5)) throw std::invalid_argument("ParticleSystem: coordinate outside the unit box");
    }
}

inline ParticleSystem wrap_into_box(const ParticleSystem& sys) {  // oracle.cpp:133-141
  ParticleSystem w = sys;
  for (std::vector<double>* pts : {&w.sources, &w.targets})
    for (double& v : *pts) v -= std::floor(v + 0.5);
  return w;
}

// ---- tree.hpp:83-104 ----
inline Tree build_tree(const std::vector<double>& sources, const std::vector<double>& targets, int n_s, int dim,
                       bool periodic, int proxy_order) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("build_tree: dim must be 2 or 3");
  if (n_s < 1) throw std::invalid_argument("build_tree: n_s must be >= 1");
  if (proxy_order < 1) throw std::invalid_argument("build_tree: proxy order must be >= 1");
  if (sources.empty() || sources.size() % dim != 0 || targets.size() % dim != 0)
    throw std::invalid_argument("build_tree: bad point array length");
  Tree t;
  t.device = std::make_shared<detail::TreeState>(detail::device_slot());
  sdmk_context* c = t.device->ctx;
  const int64_t ns = static_cast<int64_t>(sources.size()) / dim, nt = static_cast<int64_t>(targets.size()) / dim;
  detail::check(sdmk_tree_build(c, dim, periodic ? 1 : 0, n_s, proxy_order, ns, sources.data(), nt,
                                nt > 0 ? targets.data() : nullptr));
  int32_t info[7];
  detail::check(sdmk_tree_info(c, info));
  const int nb = info[0];
  t.dim = dim;
  t.periodic = periodic;
  t.n_s = n_s;
  t.proxy_order = proxy_order;
  t.max_level = info[1];
  t.depth_capped = info[5] != 0;
  t.targets_alias_sources = info[4] != 0;
  std::vector<int32_t> bx(static_cast<size_t>(nb) * 11);
  detail::check(sdmk_tree_boxes(c, bx.data()));
  t.boxes.resize(nb);
  t.level_boxes.assign(t.max_level + 1, {});
  for (int b = 0; b < nb; ++b) {  // tree.cpp:170-171: level lists in id order
    const int32_t* o = bx.data() + 11 * size_t(b);
    TreeBox& x = t.boxes[b];
    x.level = o[0];
    x.parent = o[1];
    x.first_child = o[2];
    x.leaf = o[3] != 0;
    x.anchor = {o[4], o[5], o[6]};
    x.src_begin = o[7];
    x.src_end = o[8];
    x.tgt_begin = o[9];
    x.tgt_end = o[10];
    t.level_boxes[x.level].push_back(b);
  }
  std::vector<int64_t> counts(static_cast<size_t>(nb) * 3);
  detail::check(sdmk_tree_neighbors(c, counts.data(), nullptr));
  int64_t total = 0;
  for (int64_t v : counts) total += v;
  std::vector<int32_t> ent(static_cast<size_t>(total) * 4);
  detail::check(sdmk_tree_neighbors(c, counts.data(), ent.data()));
  t.neighbors.resize(nb);
  size_t at = 0;
  for (int b = 0; b < nb; ++b) {
    std::vector<NeighborEntry>* lists[3] = {&t.neighbors[b].colleagues, &t.neighbors[b].coarse,
                                            &t.neighbors[b].fine};
    for (int k = 0; k < 3; ++k) {
      lists[k]->resize(static_cast<size_t>(counts[3 * size_t(b) + k]));
      for (NeighborEntry& e : *lists[k]) {
        const int32_t* o = ent.data() + 4 * at++;
        e.box = o[0];
        e.shift = {static_cast<std::int8_t>(o[1]), static_cast<std::int8_t>(o[2]), static_cast<std::int8_t>(o[3])};
      }
    }
  }
  t.src_perm.resize(static_cast<size_t>(ns));
  if (!t.targets_alias_sources) t.tgt_perm.resize(static_cast<size_t>(nt));
  detail::check(sdmk_tree_perm(c, t.src_perm.data(), t.targets_alias_sources ? nullptr : t.tgt_perm.data()));
  t.src_points.resize(sources.size());
  t.src_q.resize(static_cast<size_t>(ns));
  if (!t.targets_alias_sources) {
    t.tgt_points.resize(targets.size());
    t.tgt_q.resize(static_cast<size_t>(nt));
  }
  detail::check(sdmk_tree_sorted(c, t.src_points.data(), t.targets_alias_sources ? nullptr : t.tgt_points.data(),
                                 reinterpret_cast<int32_t*>(t.src_q.data()),
                                 t.targets_alias_sources ? nullptr : reinterpret_cast<int32_t*>(t.tgt_q.data())));
  return t;
}

inline const TreeNeighbors& neighbor_query(const Tree& tree, int box) { return tree.neighbors.at(box); }

inline std::vector<double> proxy_nodes(const Tree& tree, int box) {  // tree.cpp:305-323
  const int p = tree.proxy_order, d = tree.dim;
  const auto ctr = tree.box_center(box);
  const double half = 0.5 * tree.box_side(box);
  std::vector<double> nodes1(p);
  for (int i = 0; i < p; ++i) nodes1[i] = std::cos((2 * i + 1) * 3.141592653589793238462643383279502884 / (2.0 * p));
  int total = 1;
  for (int i = 0; i < d; ++i) total *= p;
  std::vector<double> out(static_cast<size_t>(total) * d);
  for (int flat = 0; flat < total; ++flat) {
    int rem = flat;
    for (int i = 0; i < d; ++i) {
      out[static_cast<size_t>(flat) * d + i] = ctr[i] + half * nodes1[rem % p];
      rem /= p;
    }
  }
  return out;
}

inline void dump_tree(const Tree& tree, std::ostream& os) {  // the canonical text of tree.cpp:325-354
  const auto put_list = [&](const char* tag, const std::vector<NeighborEntry>& lst) {
    os << ' ' << tag << "={";
    for (size_t i = 0; i < lst.size(); ++i) {
      if (i) os << ' ';
      os << lst[i].box;
      const auto& s = lst[i].shift;
      if (s[0] || s[1] || s[2]) os << '@' << int(s[0]) << ',' << int(s[1]) << ',' << int(s[2]);
    }
    os << '}';
  };
  os << "tree dim=" << tree.dim << " periodic=" << int(tree.periodic) << " n_s=" << tree.n_s
     << " p=" << tree.proxy_order << " boxes=" << tree.num_boxes() << " max_level=" << tree.max_level << '\n';
  for (int b = 0; b < tree.num_boxes(); ++b) {
    const TreeBox& bx = tree.boxes[b];
    os << b << " L" << bx.level << " a=" << bx.anchor[0] << ',' << bx.anchor[1];
    if (tree.dim == 3) os << ',' << bx.anchor[2];
    os << (bx.leaf ? " leaf" : " node") << " src=[" << bx.src_begin << ',' << bx.src_end << ") tgt=["
       << bx.tgt_begin << ',' << bx.tgt_end << ")";
    put_list("col", tree.neighbors[b].colleagues);
    put_list("crs", tree.neighbors[b].coarse);
    put_list("fin", tree.neighbors[b].fine);
    os << '\n';
  }
}

// ---- dmk.hpp:81-131: the passes, on the tree's device copy ----
inline ProxyData upward_pass(const Tree& tree, const DmkPlan& plan, const std::vector<double>& strengths) {
  detail::check_tree_plan(tree, plan);
  ProxyData og;
  og.p = plan.p;
  og.dim = plan.dim;
  og.channels = outgoing_channels(plan.kernel, plan.dim);
  og.values.resize(static_cast<size_t>(tree.num_boxes()) * og.box_stride());
  sdmk_plan c = detail::to_c(plan);
  detail::check(sdmk_pass_upward(detail::tree_context(tree, "upward_pass"), &c,
                                 static_cast<int64_t>(strengths.size()), strengths.data(), og.values.data()));
  return og;
}

inline ProxyData make_incoming(const Tree& tree, const DmkPlan& plan) {  // dmk.cpp:657-667
  detail::check_tree_plan(tree, plan);
  ProxyData in;
  in.p = plan.p;
  in.dim = plan.dim;
  in.channels = plan.dim;
  in.values.assign(static_cast<size_t>(tree.num_boxes()) * in.box_stride(), 0.0);
  return in;
}

inline void root_far_field(const Tree& tree, const DmkPlan& plan, const SplitKernel& sk, const ProxyData& outgoing,
                           bool periodic, ProxyData& incoming) {
  detail::check_tree_plan(tree, plan);
  const std::string img = detail::table_image(sk);
  sdmk_plan c = detail::to_c(plan);
  detail::check(sdmk_pass_root_far_field(detail::tree_context(tree, "root_far_field"), &c, detail::bytes(img),
                                         static_cast<int64_t>(img.size()),
                                         static_cast<int64_t>(outgoing.values.size()), outgoing.values.data(),
                                         periodic ? 1 : 0, static_cast<int64_t>(incoming.values.size()),
                                         incoming.values.data()));
}

inline void downward_pass(const Tree& tree, const DmkPlan& plan, const SplitKernel& sk, const ProxyData& outgoing,
                          bool periodic, ProxyData& incoming) {
  detail::check_tree_plan(tree, plan);
  const std::string img = detail::table_image(sk);
  sdmk_plan c = detail::to_c(plan);
  detail::check(sdmk_pass_downward(detail::tree_context(tree, "downward_pass"), &c, detail::bytes(img),
                                   static_cast<int64_t>(img.size()), static_cast<int64_t>(outgoing.values.size()),
                                   outgoing.values.data(), periodic ? 1 : 0,
                                   static_cast<int64_t>(incoming.values.size()), incoming.values.data()));
}

inline std::vector<double> target_far_fields(const Tree& tree, const DmkPlan& plan, const ProxyData& incoming) {
  detail::check_tree_plan(tree, plan);
  const size_t nt = tree.targets_alias_sources ? tree.src_perm.size() : tree.tgt_perm.size();
  std::vector<double> u(nt * static_cast<size_t>(plan.dim));
  sdmk_plan c = detail::to_c(plan);
  detail::check(sdmk_pass_target_far_fields(detail::tree_context(tree, "target_far_fields"), &c,
                                            static_cast<int64_t>(incoming.values.size()), incoming.values.data(),
                                            u.data()));
  return u;
}

inline std::vector<double> residual_pass(const Tree& tree, const DmkPlan& plan, const SplitKernel& sk,
                                         const std::vector<double>& strengths, bool periodic) {
  detail::check_tree_plan(tree, plan);
  const size_t nt = tree.targets_alias_sources ? tree.src_perm.size() : tree.tgt_perm.size();
  std::vector<double> u(nt * static_cast<size_t>(plan.dim));
  const std::string img = detail::table_image(sk);
  sdmk_plan c = detail::to_c(plan);
  detail::check(sdmk_pass_residual(detail::tree_context(tree, "residual_pass"), &c, detail::bytes(img),
                                   static_cast<int64_t>(img.size()), static_cast<int64_t>(strengths.size()),
                                   strengths.data(), periodic ? 1 : 0, u.data()));
  return u;
}

// ---- dmk.hpp:147-161 ----
inline std::vector<double> evaluate_with_plan(const DmkPlan& plan, const ParticleSystem& sys, EwaldMode mode,
                                              DmkReport* report = nullptr, const SplitKernel* tables = nullptr) {
  // dmk.cpp:1046-1055, in the reference's order; lengths are checked before any array is read
  if (plan.dim != sys.dim) throw std::invalid_argument("evaluate: plan and system dimensions differ");
  detail::check_lengths(plan.kernel, sys);
  sdmk_plan c = detail::to_c(plan);
  const int d = sys.dim;
  const int64_t ns = static_cast<int64_t>(sys.sources.size()) / d;
  const int64_t nt = static_cast<int64_t>(sys.targets.size()) / d;
  std::vector<double> u(static_cast<size_t>(nt > 0 ? nt : ns) * d);
  sdmk_report r{};
  std::string img;
  if (tables) img = detail::table_image(*tables);  // the caller's tables, window included
  detail::check(sdmk_evaluate_with_tables(detail::context(), &c, tables ? detail::bytes(img) : nullptr,
                                          static_cast<int64_t>(img.size()), d, ns, sys.sources.data(), nt,
                                          nt > 0 ? sys.targets.data() : nullptr, sys.strengths.data(),
                                          static_cast<int>(mode), u.data(), &r));
  if (report) {
    report->plan = plan;
    report->num_boxes = r.num_boxes;
    report->max_level = r.max_level;
    report->num_sources = r.num_sources;
    report->num_targets = r.num_targets;
    report->t_tree = r.t_tree;
    report->t_upward = r.t_upward;
    report->t_root = r.t_root;
    report->t_downward = r.t_downward;
    report->t_residual = r.t_residual;
  }
  return u;
}

inline std::vector<double> evaluate(KernelType kernel, const ParticleSystem& sys, double eps, WindowKind window,
                                    EwaldMode mode, DmkReport* report = nullptr) {
  return evaluate_with_plan(select_parameters(kernel, eps, window, sys.dim), sys, mode, report);
}

// ---- oracle.hpp:60-75: reference sums on the GPU; see sdmk_direct_sum ----
inline std::vector<double> direct_sum(KernelType kernel, const ParticleSystem& sys) {
  detail::check_lengths(kernel, sys);
  const int d = sys.dim;
  const int64_t ns = static_cast<int64_t>(sys.sources.size()) / d;
  const int64_t nt = static_cast<int64_t>(sys.targets.size()) / d;
  std::vector<double> u(static_cast<size_t>(nt > 0 ? nt : ns) * d);
  detail::check(sdmk_direct_sum(detail::context(), static_cast<int>(kernel), d, ns, sys.sources.data(), nt,
                                nt > 0 ? sys.targets.data() : nullptr, sys.strengths.data(), u.data()));
  return u;
}

inline std::vector<double> direct_residual_sum(const SplitKernel& sk, const ParticleSystem& sys, double cutoff,
                                               bool periodic) {
  if (sys.dim != sk.dim) throw std::invalid_argument("direct_residual_sum: dimension mismatch");
  detail::check_lengths(sk.kernel, sys);
  const int d = sys.dim;
  const int64_t ns = static_cast<int64_t>(sys.sources.size()) / d;
  const int64_t nt = static_cast<int64_t>(sys.targets.size()) / d;
  std::vector<double> u(static_cast<size_t>(nt > 0 ? nt : ns) * d);
  const std::string img = detail::table_image(sk);
  detail::check(sdmk_direct_residual_sum_tables(detail::context(), detail::bytes(img),
                                                static_cast<int64_t>(img.size()), d, ns, sys.sources.data(), nt,
                                                nt > 0 ? sys.targets.data() : nullptr, sys.strengths.data(), cutoff,
                                                periodic ? 1 : 0, u.data()));
  return u;
}

// ---- additions beyond the reference API: several GPUs, one process each ----
// (include/sdmk.h sdmk_comm_init).  Call use_device before the first
// evaluation on a thread; rank 0 makes the id, every rank passes the same
// bytes to init_comm; later evaluations on this thread return the full u on
// every rank.
namespace b200 {
inline void use_device(int device) {
  if (detail::holder().c && detail::device_slot() != device)
    throw std::invalid_argument("use_device: this thread already evaluates on another GPU");
  detail::device_slot() = device;
}

inline std::array<unsigned char, 128> nccl_unique_id() {
  std::array<unsigned char, 128> id{};
  detail::check(sdmk_comm_unique_id(id.data()));
  return id;
}

inline void init_comm(int rank, int nranks, const std::array<unsigned char, 128>& id) {
  detail::check(sdmk_comm_init(detail::context(), rank, nranks, id.data()));
}
}  // namespace b200

}  // namespace stokesdmk
