// Compile-only check: reference-style call sites (cli_main.cpp:104-204,
// bench_main.cpp:114-132) build unchanged against the drop-in header.
#include <stokesdmk_b200/dmk.hpp>

#include <algorithm>

using namespace stokesdmk;

SplitKernel make_tables(const DmkPlan& plan) {
  WindowFunction win = plan.window == WindowKind::prolate ? build_prolate(plan.c) : build_gaussian(plan.sigma);
  double tt = plan.table_tol > 0.0 ? plan.table_tol : std::max(0.03 * plan.tol, plan.dim == 2 ? 1e-12 : 1e-14);
  return build_split_kernel(plan.kernel, plan.dim, win, tt);
}

std::vector<double> timed_evaluate(const DmkPlan& plan, const ParticleSystem& sys, EwaldMode mode,
                                   const SplitKernel& sk, int reps, DmkReport& best) {
  std::vector<double> u;
  for (int r = 0; r < std::max(1, reps); ++r) {
    DmkReport rep;
    u = evaluate_with_plan(plan, sys, mode, &rep, &sk);
    if (r == 0) best = rep;
    else best.t_tree = std::min(best.t_tree, rep.t_tree);
  }
  return u;
}

// the multi-GPU additions (one process per GPU; include/sdmk.h sdmk_comm_init)
[[maybe_unused]] static std::vector<double> sharded_evaluate(int rank, int nranks, const DmkPlan& plan,
                                                             const ParticleSystem& sys,
                                                             const std::array<unsigned char, 128>& id) {
  stokesdmk::b200::use_device(rank);
  stokesdmk::b200::init_comm(rank, nranks, id);
  return evaluate_with_plan(plan, sys, EwaldMode::free_space);
}

int main() {
  ParticleSystem sys;
  sys.dim = 3;
  sys.sources = {0.1, 0.2, 0.3, -0.1, -0.2, -0.3};
  sys.strengths = {1.0, 0.0, 0.0, 0.0, 1.0, 0.0};
  DmkPlan plan = select_parameters(KernelType::stokeslet, 1e-6, WindowKind::prolate, 3);
  SplitKernel sk = make_tables(plan);
  DmkReport rep;
  std::vector<double> u = timed_evaluate(plan, sys, EwaldMode::free_space, sk, 2, rep);
  std::vector<double> v = evaluate(KernelType::stokeslet, sys, 1e-6, WindowKind::prolate, EwaldMode::free_space);
  // acceptance.cpp-style accuracy check against the exact sum (acceptance.cpp:451-474)
  std::vector<double> ex = direct_sum(KernelType::stokeslet, sys);
  std::vector<double> res = direct_residual_sum(sk, sys, 1.0, false);
  return int(u.size() + v.size() + ex.size() + res.size()) == 24 ? 0 : 1;
}
