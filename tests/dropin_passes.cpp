// C++ drop-in exercised end to end: the reference's pass-level call sites
// (dmk.hpp:64-131, tree.hpp:25-104, split.hpp:62-154) and the benchmark call
// sites (bench_main.cpp:98-132), compiled against <stokesdmk_b200/dmk.hpp>,
// linked with libsdmk_b200.so and run on the GPU.  tests/test_gpu_dropin.py
// writes the inputs, runs this program and compares every output with the
// compiled reference (oracle/_ref).
//
// usage: dropin_passes <case dir>
//   in:  <dir>/case.txt   "kernel dim eps periodic n_src n_tgt window"
//        <dir>/src.bin, [tgt.bin], str.bin      point-major doubles
//        [<dir>/ref_tables.bin]                  SDMKSPLT file exported by the reference
//        [<dir>/window_c.txt]                    a prolate c different from the plan's
//   out: tree.txt, perm.bin, upward.bin, incoming0.bin, incoming1.bin, far.bin,
//        residual.bin, u.bin, [u_reftables.bin], [u_window.bin, window_tables.bin],
//        bench.txt, api.txt
#include <stokesdmk_b200/dmk.hpp>

#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

using namespace stokesdmk;

static std::vector<double> read_bin(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return {};
  std::string b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<double> v(b.size() / sizeof(double));
  std::memcpy(v.data(), b.data(), v.size() * sizeof(double));
  return v;
}

template <class T>
static void write_bin(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static bool exists(const std::string& path) { return std::ifstream(path).good(); }

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: dropin_passes <case dir>\n";
    return 2;
  }
  const std::string dir = argv[1];
  int kernel = 0, dim = 3, periodic = 0, window = 0;
  long n_src = 0, n_tgt = 0;
  double eps = 1e-6;
  {
    std::ifstream c(dir + "/case.txt");
    c >> kernel >> dim >> eps >> periodic >> n_src >> n_tgt >> window;
  }
  ParticleSystem sys;
  sys.dim = dim;
  sys.sources = read_bin(dir + "/src.bin");
  if (n_tgt > 0) sys.targets = read_bin(dir + "/tgt.bin");
  sys.strengths = read_bin(dir + "/str.bin");
  const EwaldMode mode = periodic ? EwaldMode::periodic : EwaldMode::free_space;

  // ---- the CLI's make_tables (cli_main.cpp:104-134) ----
  DmkPlan plan = select_parameters(static_cast<KernelType>(kernel), eps, static_cast<WindowKind>(window), dim);
  WindowFunction win = plan.window == WindowKind::prolate ? build_prolate(plan.c) : build_gaussian(plan.sigma);
  SplitKernel sk = build_split_kernel(plan.kernel, plan.dim, win, plan.table_tol);

  // ---- the pass sequence of evaluate_with_plan (dmk.cpp:1070-1084) ----
  ParticleSystem w = periodic ? wrap_into_box(sys) : sys;
  validate_system(plan.kernel, sys, periodic != 0);
  Tree tree = build_tree(w.sources, w.targets, plan.n_s, dim, periodic != 0, plan.p);
  {
    std::ofstream t(dir + "/tree.txt");
    dump_tree(tree, t);
  }
  std::vector<int> perm = tree.src_perm;
  perm.insert(perm.end(), tree.tgt_perm.begin(), tree.tgt_perm.end());
  write_bin(dir + "/perm.bin", perm);
  ProxyData og = upward_pass(tree, plan, w.strengths);
  write_bin(dir + "/upward.bin", og.values);
  ProxyData in = make_incoming(tree, plan);
  root_far_field(tree, plan, sk, og, periodic != 0, in);
  write_bin(dir + "/incoming0.bin", in.values);
  downward_pass(tree, plan, sk, og, periodic != 0, in);
  write_bin(dir + "/incoming1.bin", in.values);
  write_bin(dir + "/far.bin", target_far_fields(tree, plan, in));
  write_bin(dir + "/residual.bin", residual_pass(tree, plan, sk, w.strengths, periodic != 0));

  DmkReport rep;
  std::vector<double> u = evaluate_with_plan(plan, sys, mode, &rep, &sk);
  write_bin(dir + "/u.bin", u);

  // ---- tables written by the reference's export_split_kernel ----
  if (exists(dir + "/ref_tables.bin")) {
    SplitKernel imp = import_split_kernel(dir + "/ref_tables.bin");
    write_bin(dir + "/u_reftables.bin", evaluate_with_plan(plan, sys, mode, nullptr, &imp));
    export_split_kernel(imp, dir + "/reexported.bin");  // byte-identical round trip
  }
  // ---- tables built with another window than the plan's: honoured ----
  if (exists(dir + "/window_c.txt")) {
    double c2 = 0.0;
    std::ifstream(dir + "/window_c.txt") >> c2;
    SplitKernel sk2 = build_split_kernel(plan.kernel, plan.dim, build_prolate(c2), plan.table_tol);
    export_split_kernel(sk2, dir + "/window_tables.bin");
    write_bin(dir + "/u_window.bin", evaluate_with_plan(plan, sys, mode, nullptr, &sk2));
  }

  // ---- the benchmark call sites, bench_main.cpp:100-132 (generate_points
  //      is out of scope: the points above stand in for it) ----
  {
    std::vector<double> none;
    Tree t = build_tree(w.sources, none, 600, dim, false, 23);  // BM_TreeBuild
    DmkPlan bp = select_parameters(KernelType::stokeslet, 1e-6, WindowKind::prolate, dim);  // BM_Evaluate
    SplitKernel bsk = build_split_kernel(KernelType::stokeslet, dim, build_prolate(bp.c), bp.table_tol);
    ParticleSystem bs;
    bs.dim = dim;
    bs.sources = w.sources;
    bs.strengths.assign(w.sources.size(), 0.25);
    std::vector<double> bu = evaluate_with_plan(bp, bs, EwaldMode::free_space, nullptr, &bsk);
    std::ofstream b(dir + "/bench.txt");
    b << t.num_boxes() << ' ' << bu.size() << '\n';
  }

  // ---- assorted API surface with the reference's values ----
  {
    std::ofstream a(dir + "/api.txt");
    a.precision(17);
    a << tree.num_boxes() << ' ' << tree.max_level << ' ' << tree.level_boxes.size() << ' '
      << tree.src_points.size() << ' ' << tree.src_q.size() << '\n';
    a << sk.self_const << ' ' << sk.corr_const << ' ' << sk.support << ' ' << self_interaction_scaled(sk, 0.25) << '\n';
    a << outgoing_channels(plan.kernel, dim) << ' ' << strength_components(plan.kernel, dim) << ' '
      << og.channels << ' ' << og.box_stride() << '\n';
    a << window_eval(win, 0.3) << ' ' << window_fourier(win, 2.0) << ' ' << phi_tail(win, 0.5) << '\n';
    std::vector<double> pn = proxy_nodes(tree, tree.num_boxes() - 1);
    a << pn.size() << ' ' << pn[0] << '\n';
    a << neighbor_query(tree, 0).colleagues.size() << ' ' << sys.source(1)[0] << ' ' << sys.target(0)[0] << '\n';
    // error paths with the reference's exception types
    int caught = 0;
    try {
      ParticleSystem bad = sys;
      bad.strengths.pop_back();
      evaluate_with_plan(plan, bad, mode);
    } catch (const std::invalid_argument& e) {
      caught += std::string(e.what()) == "ParticleSystem: bad strength array length";
    }
    try {
      DmkPlan p2 = plan;
      p2.p += 1;
      upward_pass(tree, p2, w.strengths);
    } catch (const std::invalid_argument& e) {
      caught += std::string(e.what()) == "dmk: tree proxy order does not match plan";
    }
    try {
      std::vector<double> outside = {0.7, 0.0, 0.0};
      build_tree(outside, {}, 10, 3, false, 4);
    } catch (const std::invalid_argument& e) {
      caught += std::string(e.what()) == "build_tree: point outside the unit box";
    }
    try {
      upward_pass(tree, plan, std::vector<double>(3));
    } catch (const std::invalid_argument& e) {
      caught += std::string(e.what()) == "upward_pass: strength array size mismatch";
    }
    try {
      Tree empty;
      empty.dim = plan.dim;
      empty.proxy_order = plan.p;
      upward_pass(empty, plan, w.strengths);
    } catch (const std::invalid_argument&) {
      ++caught;
    }
    a << caught << '\n';
  }
  std::printf("ok %d boxes\n", tree.num_boxes());
  return 0;
}
