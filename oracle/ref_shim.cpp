/*
 * oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the
 * product).  A thin extern "C" shim over the UNMODIFIED reference library
 * (stokesdmk, compiled from /root/reference/proj/core/src by oracle/Makefile
 * into oracle/_ref/libsdmk_ref.so).  Only tests/, __graft_entry__.smoke() and
 * bench.py's reference / cpu_baseline leg load it.
 *
 * Every entry point forwards to the reference's own public API:
 *   select_parameters      params.cpp:60-115
 *   build_prolate          prolate.cpp:69-165
 *   build_split_kernel     split.cpp:319-396
 *   build_tree / dump_tree tree.cpp:230-298, 325-354
 *   upward_pass            dmk.cpp:555-655
 *   make_incoming/root_far_field/downward_pass  dmk.cpp:657-857
 *   target_far_fields      dmk.cpp:861-915
 *   residual_pass          dmk.cpp:919-1032
 *   evaluate_with_plan     dmk.cpp:1036-1117
 *   direct_sum             oracle.cpp:143-179
 *   export_split_kernel    split.cpp:444-471
 * The shim keeps one "current problem" (plan, wrapped system, tables, tree)
 * so a test can fetch every pass of the same tree.  Not thread safe.
 */
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "stokesdmk/dmk.hpp"
#include "stokesdmk/oracle.hpp"
#include "stokesdmk/split.hpp"
#include "stokesdmk/tree.hpp"
#include "stokesdmk/windows.hpp"

using namespace stokesdmk;

extern "C" {

struct ref_plan {
  int kernel, dim, window;
  double tol, c, sigma;
  int p, N1, N_per, n_s;
  double table_tol;
};

struct ref_report {
  int num_boxes, max_level, num_sources, num_targets;
  double t_tree, t_upward, t_root, t_downward, t_residual;
};
}

namespace {

std::string g_err;
DmkPlan g_plan;
ParticleSystem g_sys;  /* wrapped when periodic */
bool g_periodic = false;
SplitKernel g_sk;
Tree g_tree;
bool g_have = false;

DmkPlan to_plan(const ref_plan* p) {
  DmkPlan d;
  d.kernel = KernelType(p->kernel);
  d.dim = p->dim;
  d.window = WindowKind(p->window);
  d.tol = p->tol;
  d.c = p->c;
  d.sigma = p->sigma;
  d.p = p->p;
  d.N1 = p->N1;
  d.N_per = p->N_per;
  d.n_s = p->n_s;
  d.table_tol = p->table_tol;
  return d;
}

void from_plan(const DmkPlan& d, ref_plan* p) {
  p->kernel = int(d.kernel);
  p->dim = d.dim;
  p->window = int(d.window);
  p->tol = d.tol;
  p->c = d.c;
  p->sigma = d.sigma;
  p->p = d.p;
  p->N1 = d.N1;
  p->N_per = d.N_per;
  p->n_s = d.n_s;
  p->table_tol = d.table_tol;
}

/* same table construction as evaluate_with_plan (dmk.cpp:1059-1068) */
SplitKernel tables_for(const DmkPlan& plan) {
  WindowFunction win = (plan.window == WindowKind::prolate)
                           ? build_prolate(plan.c)
                           : build_gaussian(plan.sigma);
  double tt = plan.table_tol > 0.0
                  ? plan.table_tol
                  : std::max(0.03 * plan.tol, plan.dim == 2 ? 1e-12 : 1e-14);
  return build_split_kernel(plan.kernel, plan.dim, win, tt);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = std::string("domain_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 3;
  }
}

void copy_out(const std::vector<double>& v, double* out) {
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

int ref_select_parameters(int kernel, double eps, int window, int dim,
                          ref_plan* out) {
  return guard([&] {
    from_plan(select_parameters(KernelType(kernel), eps, WindowKind(window), dim),
              out);
  });
}

/* Validates, wraps (periodic), builds tables and the tree of one problem. */
int ref_setup(const ref_plan* plan, int dim, int64_t n_src, const double* src,
              int64_t n_tgt, const double* tgt, const double* str,
              int periodic) {
  return guard([&] {
    g_have = false;
    g_plan = to_plan(plan);
    ParticleSystem s;
    s.dim = dim;
    s.sources.assign(src, src + n_src * dim);
    if (n_tgt > 0) s.targets.assign(tgt, tgt + n_tgt * dim);
    int sc = strength_components(g_plan.kernel, dim);
    s.strengths.assign(str, str + n_src * sc);
    g_periodic = periodic != 0;
    validate_system(g_plan.kernel, s, g_periodic);
    g_sys = g_periodic ? wrap_into_box(s) : s;
    g_sk = tables_for(g_plan);
    g_tree = build_tree(g_sys.sources, g_sys.targets, g_plan.n_s, dim,
                        g_periodic, g_plan.p);
    g_have = true;
  });
}

/* num_boxes, max_level, n_src, n_tgt, alias, depth_capped, nch */
int ref_tree_info(int* out) {
  if (!g_have) return 1;
  out[0] = g_tree.num_boxes();
  out[1] = g_tree.max_level;
  out[2] = int(g_tree.src_perm.size());
  out[3] = g_tree.targets_alias_sources ? int(g_tree.src_perm.size())
                                        : int(g_tree.tgt_perm.size());
  out[4] = g_tree.targets_alias_sources;
  out[5] = g_tree.depth_capped;
  out[6] = outgoing_channels(g_plan.kernel, g_plan.dim);
  return 0;
}

/* 11 ints per box: level parent first_child leaf a0 a1 a2 sb se tb te */
int ref_tree_boxes(int* out) {
  if (!g_have) return 1;
  for (int b = 0; b < g_tree.num_boxes(); ++b) {
    const TreeBox& x = g_tree.boxes[b];
    int* o = out + 11 * size_t(b);
    o[0] = x.level;
    o[1] = x.parent;
    o[2] = x.first_child;
    o[3] = x.leaf;
    o[4] = x.anchor[0];
    o[5] = x.anchor[1];
    o[6] = x.anchor[2];
    o[7] = x.src_begin;
    o[8] = x.src_end;
    o[9] = x.tgt_begin;
    o[10] = x.tgt_end;
  }
  return 0;
}

int ref_tree_perm(int* src_perm, int* tgt_perm) {
  if (!g_have) return 1;
  std::memcpy(src_perm, g_tree.src_perm.data(), g_tree.src_perm.size() * 4);
  if (tgt_perm && !g_tree.targets_alias_sources)
    std::memcpy(tgt_perm, g_tree.tgt_perm.data(), g_tree.tgt_perm.size() * 4);
  return 0;
}

/* Canonical text dump; returns the length (copies at most cap bytes). */
int64_t ref_tree_dump(char* buf, int64_t cap) {
  if (!g_have) return -1;
  std::ostringstream os;
  dump_tree(g_tree, os);
  std::string s = os.str();
  if (buf && cap > 0) std::memcpy(buf, s.data(), std::min<int64_t>(cap, s.size()));
  return int64_t(s.size());
}

int ref_upward(double* out) {
  return guard([&] { copy_out(upward_pass(g_tree, g_plan, g_sys.strengths).values, out); });
}

/* stage 0: incoming after root_far_field; 1: after downward_pass too */
int ref_incoming(int stage, double* out) {
  return guard([&] {
    ProxyData og = upward_pass(g_tree, g_plan, g_sys.strengths);
    ProxyData in = make_incoming(g_tree, g_plan);
    root_far_field(g_tree, g_plan, g_sk, og, g_periodic, in);
    if (stage >= 1) downward_pass(g_tree, g_plan, g_sk, og, g_periodic, in);
    copy_out(in.values, out);
  });
}

int ref_target_far(double* out) {
  return guard([&] {
    ProxyData og = upward_pass(g_tree, g_plan, g_sys.strengths);
    ProxyData in = make_incoming(g_tree, g_plan);
    root_far_field(g_tree, g_plan, g_sk, og, g_periodic, in);
    downward_pass(g_tree, g_plan, g_sk, og, g_periodic, in);
    copy_out(target_far_fields(g_tree, g_plan, in), out);
  });
}

int ref_residual(double* out) {
  return guard([&] {
    copy_out(residual_pass(g_tree, g_plan, g_sk, g_sys.strengths, g_periodic), out);
  });
}

/* evaluate_with_plan with prebuilt tables (the CLI's timed region,
   cli_main.cpp:186-204); report holds DmkReport's pass times. */
int ref_evaluate(double* out, ref_report* rep) {
  return guard([&] {
    DmkReport r;
    EwaldMode mode = g_periodic ? EwaldMode::periodic : EwaldMode::free_space;
    std::vector<double> u = evaluate_with_plan(g_plan, g_sys, mode, &r, &g_sk);
    copy_out(u, out);
    if (rep) {
      rep->num_boxes = r.num_boxes;
      rep->max_level = r.max_level;
      rep->num_sources = r.num_sources;
      rep->num_targets = r.num_targets;
      rep->t_tree = r.t_tree;
      rep->t_upward = r.t_upward;
      rep->t_root = r.t_root;
      rep->t_downward = r.t_downward;
      rep->t_residual = r.t_residual;
    }
  });
}

int ref_direct_sum(double* out) {
  return guard([&] { copy_out(direct_sum(g_plan.kernel, g_sys), out); });
}

int ref_direct_residual_sum(double cutoff, double* out) {
  return guard([&] {
    copy_out(direct_residual_sum(g_sk, g_sys, cutoff, g_periodic), out);
  });
}

/* the slow single-level split reference (oracle.cpp ewald_reference):
   periodic = 1 for the Fourier series over 2 pi kappa, 0 for free space */
int ref_ewald_reference(int periodic, double* out) {
  return guard([&] {
    copy_out(ewald_reference(g_sk, g_sys, periodic ? EwaldMode::periodic : EwaldMode::free_space), out);
  });
}

/* split.cpp self_interaction_scaled: the self coefficient at scale nu */
int ref_self_scaled(double nu, double* out) {
  return guard([&] { *out = self_interaction_scaled(g_sk, nu); });
}

int ref_periodic_zero_mode(double* out) {
  return guard([&] { copy_out(periodic_zero_mode(g_plan.kernel, g_sys), out); });
}

/* SDMKSPLT v1 binary table file of the current problem's tables */
int ref_export_tables(const char* path) {
  return guard([&] { export_split_kernel(g_sk, path); });
}

/* window: legendre coeffs + scalars (kind c sigma lambda0 norm_r trunc psi0 chi0) */
int ref_window(double* scalars, double* coeffs, int cap) {
  const WindowFunction& w = g_sk.mollifier.window;
  scalars[0] = double(w.kind);
  scalars[1] = w.c;
  scalars[2] = w.sigma;
  scalars[3] = w.lambda0;
  scalars[4] = w.norm_r;
  scalars[5] = w.trunc_error;
  scalars[6] = w.psi0;
  scalars[7] = w.chi0;
  int n = int(w.legendre_coeffs.size());
  for (int i = 0; i < n && i < cap; ++i) coeffs[i] = w.legendre_coeffs[i];
  return n;
}

/* unit-scale public window / mollifier functions, for table pinning */
double ref_window_fourier(double k) { return window_fourier(g_sk.mollifier.window, k); }
double ref_mollifier_fourier(double k) { return mollifier_fourier(g_sk.mollifier, k); }
double ref_window_eval(double r) { return window_eval(g_sk.mollifier.window, r); }
double ref_phi_tail(double r) { return phi_tail(g_sk.mollifier.window, r); }
double ref_truncated_biharmonic_fourier(double k, double R, int dim) {
  return truncated_biharmonic_fourier(k, R, dim);
}
double ref_truncated_harmonic_fourier(double k, double R, int dim) {
  return truncated_harmonic_fourier(k, R, dim);
}
int ref_mollifier_taylor(double* a5) {
  auto a = mollifier_fourier_taylor(g_sk.mollifier);
  for (int i = 0; i < 5; ++i) a5[i] = a[i];
  return 0;
}
int ref_residual_apply(const double* x, double nu, const double* s, double* u) {
  return guard([&] { residual_apply(g_sk, x, nu, s, u); });
}


/* ---- full-size parity support (tools/parity_configs.py) ----
   ref_run_full runs the passes of evaluate_with_plan (dmk.cpp:1070-1084) once
   on the current problem, in the same order and with the same calls, keeps
   the outgoing / incoming proxies alive for ref_proxy, and returns the
   target far field, the residual and u assembled exactly as
   dmk.cpp:1086-1102 does (u = far + residual; corr_const * Kahan sum of f
   for the free-space Stokeslet; periodic_zero_mode for the periodic
   stresslet).  rep receives the pass times (steady clock, as DmkReport). */
ProxyData g_og, g_in;

int ref_run_full(double* far, double* res, double* u, ref_report* rep) {
  return guard([&] {
    using clock = std::chrono::steady_clock;
    auto secs = [](clock::time_point a, clock::time_point b) {
      return std::chrono::duration<double>(b - a).count();
    };
    const DmkPlan& plan = g_plan;
    auto t1 = clock::now();
    g_og = upward_pass(g_tree, plan, g_sys.strengths);
    auto t2 = clock::now();
    g_in = make_incoming(g_tree, plan);
    root_far_field(g_tree, plan, g_sk, g_og, g_periodic, g_in);
    auto t3 = clock::now();
    downward_pass(g_tree, plan, g_sk, g_og, g_periodic, g_in);
    std::vector<double> uf = target_far_fields(g_tree, plan, g_in);
    auto t4 = clock::now();
    std::vector<double> ur = residual_pass(g_tree, plan, g_sk, g_sys.strengths, g_periodic);
    auto t5 = clock::now();
    copy_out(uf, far);
    copy_out(ur, res);
    const int d = plan.dim;
    const int nt = g_sys.num_targets();
    for (size_t i = 0; i < uf.size(); ++i) uf[i] += ur[i];
    if (plan.kernel == KernelType::stokeslet && !g_periodic && g_sk.corr_const != 0.0) {
      double sum[3] = {0, 0, 0}, comp[3] = {0, 0, 0};
      const int ns = g_sys.num_sources();
      for (int a = 0; a < ns; ++a)
        for (int j = 0; j < d; ++j) {  /* Kahan, dmk.cpp:540-548 */
          double y = g_sys.strengths[size_t(a) * d + j] - comp[j];
          double t = sum[j] + y;
          comp[j] = (t - sum[j]) - y;
          sum[j] = t;
        }
      for (int t = 0; t < nt; ++t)
        for (int j = 0; j < d; ++j) uf[size_t(t) * d + j] += g_sk.corr_const * sum[j];
    }
    if (plan.kernel == KernelType::stresslet && g_periodic) {
      std::vector<double> u0 = periodic_zero_mode(plan.kernel, g_sys);
      for (size_t i = 0; i < uf.size(); ++i) uf[i] += u0[i];
    }
    copy_out(uf, u);
    if (rep) {
      rep->num_boxes = g_tree.num_boxes();
      rep->max_level = g_tree.max_level;
      rep->num_sources = g_sys.num_sources();
      rep->num_targets = nt;
      rep->t_tree = 0.0;
      rep->t_upward = secs(t1, t2);
      rep->t_root = secs(t2, t3);
      rep->t_downward = secs(t3, t4);
      rep->t_residual = secs(t4, t5);
    }
  });
}

/* replaces the current problem's split tables by build_split_kernel with
   another window (prolate c, or gaussian sigma when c <= 0), same kernel,
   dim and table_tol: the evaluate_with_plan(..., &tables) case where the
   tables' window differs from the plan's (dmk.cpp:1059-1069) */
int ref_set_window(double c, double sigma) {
  return guard([&] {
    WindowFunction w = c > 0.0 ? build_prolate(c) : build_gaussian(sigma);
    g_sk = build_split_kernel(g_plan.kernel, g_plan.dim, w, g_sk.table_tol);
  });
}

/* pointer to the kept proxies of ref_run_full (0 outgoing, 1 incoming) */
const double* ref_proxy(int which, int64_t* n) {
  const ProxyData& P = which == 0 ? g_og : g_in;
  *n = int64_t(P.values.size());
  return P.values.data();
}

void ref_release() {
  g_og = ProxyData();
  g_in = ProxyData();
}

/* build_tree alone on the current problem's wrapped points (seconds) */
double ref_time_tree() {
  auto a = std::chrono::steady_clock::now();
  Tree t = build_tree(g_sys.sources, g_sys.targets, g_plan.n_s, g_plan.dim, g_periodic, g_plan.p);
  auto b = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(b - a).count();
}

/* The residual pass's pair loop (dmk.cpp:941-1013) over the reference's own
   tree with residual_apply left out: out[0] = pairs tested (every source of
   every near range except the alias diagonal), out[1] = pairs in support
   (r2 < sup2 and r2 != 0), out[2] = coincident pairs.  Same ranges, same
   shift arithmetic and the same unfused r2 as the reference. */
int ref_count_pairs(int64_t* out) {
  return guard([&] {
    const Tree& tree = g_tree;
    const int d = g_plan.dim;
    const bool alias = tree.targets_alias_sources;
    const std::vector<double>& tp = alias ? tree.src_points : tree.tgt_points;
    std::vector<int> leaves;
    for (int b = 0; b < tree.num_boxes(); ++b)
      if (tree.boxes[b].leaf && tree.box_tgt_count(b) > 0) leaves.push_back(b);
    int64_t tested = 0, in = 0, zero = 0;
    struct R { int begin, end; double shift[3]; double nu; bool selfr; };
#pragma omp parallel reduction(+ : tested, in, zero)
    {
      std::vector<R> ranges;
#pragma omp for schedule(dynamic, 4)
      for (int li = 0; li < int(leaves.size()); ++li) {
        const int b = leaves[li];
        const TreeBox& box = tree.boxes[b];
        const double r_l = tree.box_side(b), r_f = 0.5 * r_l;
        ranges.clear();
        auto add = [&](int sbx, const std::array<std::int8_t, 3>& sh, double nu, bool selfr) {
          const TreeBox& sb = tree.boxes[sbx];
          if (sb.src_end == sb.src_begin) return;
          R r{sb.src_begin, sb.src_end, {double(sh[0]), double(sh[1]), double(sh[2])}, nu, selfr};
          ranges.push_back(r);
        };
        add(b, {0, 0, 0}, r_l, true);
        const TreeNeighbors& nb = neighbor_query(tree, b);
        for (const NeighborEntry& e : nb.colleagues) {
          if (e.box == b && e.shift[0] == 0 && e.shift[1] == 0 && e.shift[2] == 0) continue;
          if (!tree.boxes[e.box].leaf) continue;
          add(e.box, e.shift, r_f, false);
        }
        for (const NeighborEntry& e : nb.coarse) add(e.box, e.shift, r_l, false);
        for (const NeighborEntry& e : nb.fine) add(e.box, e.shift, r_f, false);
        for (int t = box.tgt_begin; t < box.tgt_end; ++t) {
          const double* xt = tp.data() + size_t(t) * d;
          for (const R& r : ranges) {
            const double sup = r.nu * g_sk.support, sup2 = sup * sup;
            for (int a = r.begin; a < r.end; ++a) {
              if (alias && r.selfr && a == t) continue;
              const double* xs = tree.src_points.data() + size_t(a) * d;
              double r2 = 0.0;
              for (int ax = 0; ax < d; ++ax) {
                double x = xt[ax] - (xs[ax] + r.shift[ax]);
                r2 += x * x;
              }
              ++tested;
              if (r2 >= sup2) continue;
              if (r2 == 0.0) { ++zero; continue; }
              ++in;
            }
          }
        }
      }
    }
    out[0] = tested;
    out[1] = in;
    out[2] = zero;
  });
}

}  // extern "C"
