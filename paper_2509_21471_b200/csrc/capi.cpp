// extern "C" boundary of libsdmk_b200.so (declared in include/sdmk.h).
// Never throws: exceptions become sdmk_status codes plus sdmk_last_error().
#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "../../include/sdmk.h"
#include "engine.hpp"

using namespace sdmkb;

struct sdmk_context {
  Context* ctx;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return SDMK_OK;
  } catch (const InvalidArgument& e) {
    g_err = e.what();
    return SDMK_EINVAL;
  } catch (const DomainError& e) {
    g_err = e.what();
    return SDMK_EDOMAIN;
  } catch (const RuntimeError& e) {
    g_err = e.what();
    return SDMK_ERUNTIME;
  } catch (const OomError& e) {
    g_err = e.what();
    return SDMK_EOOM;
  } catch (const CudaError& e) {
    g_err = e.what();
    return SDMK_ECUDA;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SDMK_EOOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SDMK_ERUNTIME;
  }
}

Plan to_plan(const sdmk_plan* p) {
  Plan P;
  P.kernel = p->kernel;
  P.dim = p->dim;
  P.window = p->window;
  P.tol = p->tol;
  P.c = p->c;
  P.sigma = p->sigma;
  P.p = p->p;
  P.N1 = p->N1;
  P.N_per = p->N_per;
  P.n_s = p->n_s;
  P.table_tol = p->table_tol;
  return P;
}

void from_plan(const Plan& P, sdmk_plan* p) {
  p->kernel = P.kernel;
  p->dim = P.dim;
  p->window = P.window;
  p->tol = P.tol;
  p->c = P.c;
  p->sigma = P.sigma;
  p->p = P.p;
  p->N1 = P.N1;
  p->N_per = P.N_per;
  p->n_s = P.n_s;
  p->table_tol = P.table_tol;
}

Context* need_ctx(sdmk_context* c) {
  if (!c || !c->ctx) throw InvalidArgument("null sdmk_context");
  return c->ctx;
}

}  // namespace

extern "C" {

const char* sdmk_last_error(void) { return g_err.c_str(); }

int sdmk_device_ok(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return prop.major == 10 && prop.minor == 0;
}

int sdmk_create(int device, sdmk_context** out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("sdmk_create: null output pointer");
    *out = nullptr;
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) throw InvalidArgument("sdmk_create: no such CUDA device");
    if (!sdmk_device_ok(device)) throw CudaError("sdmk_create: device is not an sm_100 (B200) GPU");
    auto* c = new sdmk_context;
    c->ctx = new Context(device);
    *out = c;
  });
}

int sdmk_destroy(sdmk_context* c) {
  return guarded([&] {
    if (!c) return;
    delete c->ctx;
    delete c;
  });
}

int sdmk_select_parameters(int kernel, double eps, int window, int dim, sdmk_plan* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("sdmk_select_parameters: null output");
    from_plan(select_plan(kernel, eps, window, dim), out);
  });
}

int sdmk_outgoing_channels(int kernel, int dim) {
  int r = -1;
  if (guarded([&] { r = channels_out(kernel, dim); }) != SDMK_OK) return -1;
  return r;
}

int sdmk_strength_components(int kernel, int dim) { return strength_width(kernel, dim); }

int sdmk_load_tables(sdmk_context* c, const char* path) {
  return guarded([&] { need_ctx(c)->load_tables(path ? path : ""); });
}

int sdmk_save_tables(sdmk_context* c, const sdmk_plan* plan, const char* path) {
  return guarded([&] { save_tables(need_ctx(c)->tables_for(to_plan(plan)), path ? path : ""); });
}

int sdmk_evaluate_with_plan(sdmk_context* c, const sdmk_plan* plan, int dim, int64_t n_src, const double* src,
                            int64_t n_tgt, const double* tgt, const double* str, int mode, double* u,
                            sdmk_report* report) {
  return guarded([&] {
    if (!plan || !src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("evaluate: null array");
    need_ctx(c)->evaluate(to_plan(plan), dim, n_src, src, n_tgt, tgt, str, mode, u, report, false);
  });
}

int sdmk_evaluate(sdmk_context* c, int kernel, int dim, int64_t n_src, const double* src, int64_t n_tgt,
                  const double* tgt, const double* str, double eps, int window, int mode, double* u,
                  sdmk_report* report) {
  return guarded([&] {
    if (!src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("evaluate: null array");
    Plan P = select_plan(kernel, eps, window, dim);
    need_ctx(c)->evaluate(P, dim, n_src, src, n_tgt, tgt, str, mode, u, report, false);
  });
}

int sdmk_evaluate_device(sdmk_context* c, const sdmk_plan* plan, int dim, int64_t n_src, const double* d_src,
                         int64_t n_tgt, const double* d_tgt, const double* d_str, int mode, double* d_u,
                         sdmk_report* report) {
  return guarded([&] {
    if (!plan || !d_src || !d_str || !d_u || (n_tgt > 0 && !d_tgt)) throw InvalidArgument("evaluate: null array");
    need_ctx(c)->evaluate(to_plan(plan), dim, n_src, d_src, n_tgt, d_tgt, d_str, mode, d_u, report, true);
  });
}

int sdmk_setup(sdmk_context* c, const sdmk_plan* plan, int dim, int64_t n_src, const double* src, int64_t n_tgt,
               const double* tgt, const double* str, int mode) {
  return guarded([&] {
    if (!plan || !src || !str || (n_tgt > 0 && !tgt)) throw InvalidArgument("setup: null array");
    need_ctx(c)->setup(to_plan(plan), dim, n_src, src, n_tgt, tgt, str, mode);
  });
}

int sdmk_tree_info(sdmk_context* c, int32_t* info) {
  return guarded([&] {
    const Problem& p = need_ctx(c)->problem();
    if (!p.ready) throw InvalidArgument("no problem set up");
    info[0] = p.tree.num_boxes();
    info[1] = p.tree.max_level;
    info[2] = p.ns;
    info[3] = p.nt;
    info[4] = p.alias;
    info[5] = p.tree.depth_capped;
    info[6] = p.nch;
  });
}

int sdmk_tree_boxes(sdmk_context* c, int32_t* out) {
  return guarded([&] {
    const Problem& p = need_ctx(c)->problem();
    if (!p.ready) throw InvalidArgument("no problem set up");
    for (int b = 0; b < p.tree.num_boxes(); ++b) {
      const Box& x = p.tree.boxes[b];
      int32_t* o = out + 11 * (size_t)b;
      o[0] = x.level;
      o[1] = x.parent;
      o[2] = x.first_child;
      o[3] = x.leaf;
      o[4] = x.anchor[0];
      o[5] = x.anchor[1];
      o[6] = x.anchor[2];
      o[7] = x.sb;
      o[8] = x.se;
      o[9] = x.tb;
      o[10] = x.te;
    }
  });
}

int sdmk_tree_perm(sdmk_context* c, int32_t* src_perm, int32_t* tgt_perm) {
  return guarded([&] {
    if (!src_perm) throw InvalidArgument("sdmk_tree_perm: null output");
    need_ctx(c)->tree_perm(src_perm, tgt_perm);
  });
}

int64_t sdmk_tree_dump(sdmk_context* c, char* buf, int64_t cap) {
  int64_t len = -1;
  guarded([&] {
    Context* x = need_ctx(c);
    if (!x->problem().ready) throw InvalidArgument("no problem set up");
    std::string s = x->tree_dump();
    len = (int64_t)s.size();
    if (buf && cap > 0) std::memcpy(buf, s.data(), (size_t)std::min<int64_t>(cap, len));
  });
  return len;
}

int sdmk_upward_pass(sdmk_context* c, double* out) {
  return guarded([&] { need_ctx(c)->upward(out); });
}

int sdmk_incoming(sdmk_context* c, int stage, double* out) {
  return guarded([&] { need_ctx(c)->incoming(stage, out); });
}

int sdmk_target_far_fields(sdmk_context* c, double* out) {
  return guarded([&] { need_ctx(c)->target_far(out); });
}

int sdmk_residual_pass(sdmk_context* c, double* out) {
  return guarded([&] { need_ctx(c)->residual(out); });
}

// ---- tree-first pass-level API ----
namespace {
const Tables* image_or_null(Context* x, const unsigned char* tables, int64_t nbytes) {
  if (!tables) return nullptr;
  if (nbytes <= 0) throw InvalidArgument("split tables: empty image");
  return &x->tables_image(tables, (size_t)nbytes);
}
}  // namespace

int sdmk_tree_build(sdmk_context* c, int dim, int periodic, int n_s, int proxy_order, int64_t n_src,
                    const double* src, int64_t n_tgt, const double* tgt) {
  return guarded([&] {
    if ((n_src > 0 && !src) || (n_tgt > 0 && !tgt)) throw InvalidArgument("build_tree: null array");
    need_ctx(c)->tree_build(dim, periodic != 0, n_s, proxy_order, n_src, src, n_tgt, tgt);
  });
}

int sdmk_tree_neighbors(sdmk_context* c, int64_t* counts, int32_t* entries) {
  return guarded([&] {
    if (!counts) throw InvalidArgument("sdmk_tree_neighbors: null counts");
    need_ctx(c)->tree_neighbors(counts, entries);
  });
}

int sdmk_tree_sorted(sdmk_context* c, double* src_points, double* tgt_points, int32_t* src_q, int32_t* tgt_q) {
  return guarded([&] { need_ctx(c)->tree_sorted(src_points, tgt_points, src_q, tgt_q); });
}

int sdmk_pass_upward(sdmk_context* c, const sdmk_plan* plan, int64_t n_str, const double* str, double* outgoing) {
  return guarded([&] {
    if (!plan || !str || !outgoing) throw InvalidArgument("upward_pass: null array");
    need_ctx(c)->pass_upward(to_plan(plan), n_str, str, outgoing);
  });
}

int sdmk_pass_root_far_field(sdmk_context* c, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                             int64_t n_out, const double* outgoing, int periodic, int64_t n_in, double* incoming) {
  return guarded([&] {
    if (!plan || !outgoing || !incoming) throw InvalidArgument("root_far_field: null array");
    Context* x = need_ctx(c);
    x->pass_root(to_plan(plan), image_or_null(x, tables, nbytes), n_out, outgoing, periodic != 0, n_in, incoming);
  });
}

int sdmk_pass_downward(sdmk_context* c, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                       int64_t n_out, const double* outgoing, int periodic, int64_t n_in, double* incoming) {
  return guarded([&] {
    if (!plan || !outgoing || !incoming) throw InvalidArgument("downward_pass: null array");
    Context* x = need_ctx(c);
    x->pass_downward(to_plan(plan), image_or_null(x, tables, nbytes), n_out, outgoing, periodic != 0, n_in, incoming);
  });
}

int sdmk_pass_target_far_fields(sdmk_context* c, const sdmk_plan* plan, int64_t n_in, const double* incoming,
                                double* u) {
  return guarded([&] {
    if (!plan || !incoming || !u) throw InvalidArgument("target_far_fields: null array");
    need_ctx(c)->pass_target_far(to_plan(plan), n_in, incoming, u);
  });
}

int sdmk_pass_residual(sdmk_context* c, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                       int64_t n_str, const double* str, int periodic, double* u) {
  return guarded([&] {
    if (!plan || !str || !u) throw InvalidArgument("residual_pass: null array");
    Context* x = need_ctx(c);
    x->pass_residual(to_plan(plan), image_or_null(x, tables, nbytes), n_str, str, periodic != 0, u);
  });
}

int sdmk_evaluate_with_tables(sdmk_context* c, const sdmk_plan* plan, const unsigned char* tables, int64_t nbytes,
                              int dim, int64_t n_src, const double* src, int64_t n_tgt, const double* tgt,
                              const double* str, int mode, double* u, sdmk_report* report) {
  return guarded([&] {
    if (!plan || !src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("evaluate: null array");
    Context* x = need_ctx(c);
    const Tables* t = image_or_null(x, tables, nbytes);
    struct Clear {
      Context* x;
      ~Clear() { x->set_tables_override(nullptr); }
    } clear{x};
    x->set_tables_override(t);
    x->evaluate(to_plan(plan), dim, n_src, src, n_tgt, tgt, str, mode, u, report, false);
  });
}

int64_t sdmk_host_build_tables(int kernel, int dim, int window, double c, double sigma, double tol,
                               unsigned char* buf, int64_t cap) {
  int64_t len = -1;
  guarded([&] {
    // build_split_kernel (split.cpp:319-396) with build_prolate / build_gaussian (windows.cpp)
    if (dim != 2 && dim != 3) throw InvalidArgument("build_split_kernel: dim must be 2 or 3");
    if (window == kProlate && !(c > 0.0)) throw InvalidArgument("build_prolate: c must be positive");
    if (window == kGaussian && !(sigma > 0.0)) throw InvalidArgument("build_gaussian: sigma must be positive");
    if (window != kProlate && window != kGaussian) throw InvalidArgument("build_split_kernel: unknown window");
    WindowFn w = window == kProlate ? make_prolate(c) : make_gaussian(sigma);
    std::string img = serialize_tables(build_tables(kernel, dim, w, tol));
    len = (int64_t)img.size();
    if (buf && cap > 0) std::memcpy(buf, img.data(), (size_t)std::min<int64_t>(cap, len));
  });
  return len;
}

int sdmk_host_build_window(int window, double c, double sigma, double* scalars, double* coeffs, int cap) {
  int n = -1;
  guarded([&] {
    if (window != kProlate && window != kGaussian) throw InvalidArgument("window: unknown kind");
    WindowFn w = window == kProlate ? make_prolate(c) : make_gaussian(sigma);
    if (scalars) {
      scalars[0] = w.lambda0;
      scalars[1] = w.norm_r;
      scalars[2] = w.trunc_error;
      scalars[3] = w.psi0;
      scalars[4] = w.chi0;
    }
    n = (int)w.leg.size();
    if (coeffs)
      for (int i = 0; i < n && i < cap; ++i) coeffs[i] = w.leg[i];
  });
  return n;
}

int sdmk_host_window_eval(int window, double c, double sigma, const double* coeffs, int ncoef,
                          const double* scalars, int what, int64_t n, const double* x, double* out) {
  return guarded([&] {
    WindowFn w;
    w.kind = window;
    w.c = c;
    w.sigma = sigma;
    if (coeffs) w.leg.assign(coeffs, coeffs + ncoef);
    if (scalars) {
      w.lambda0 = scalars[0];
      w.norm_r = scalars[1];
      w.trunc_error = scalars[2];
      w.psi0 = scalars[3];
      w.chi0 = scalars[4];
    }
    for (int64_t i = 0; i < n; ++i) {
      switch (what) {
        case 0: out[i] = win_phi(w, x[i]); break;
        case 1: out[i] = win_dphi(w, x[i]); break;
        case 2: out[i] = win_hat(w, x[i]); break;
        case 3: out[i] = win_tail(w, x[i]); break;
        case 4: out[i] = moll_hat(w, x[i]); break;
        default: throw InvalidArgument("window: unknown function");
      }
    }
  });
}

int sdmk_direct_residual_sum_tables(sdmk_context* c, const unsigned char* tables, int64_t nbytes, int dim,
                                    int64_t n_src, const double* src, int64_t n_tgt, const double* tgt,
                                    const double* str, double cutoff, int periodic, double* u) {
  return guarded([&] {
    if (!tables || !src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("direct_residual_sum: null array");
    Context* x = need_ctx(c);
    const Tables& t = x->tables_image(tables, (size_t)nbytes);
    x->direct(t.kernel, dim, n_src, src, n_tgt, tgt, str, &t, cutoff, periodic != 0, u, false);
  });
}

int sdmk_ewald(sdmk_context* c, const sdmk_plan* plan, int64_t n_src, const double* src, int64_t n_tgt,
               const double* tgt, const double* str, double* u, int level, double* info) {
  return guarded([&] {
    if (!plan || !src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("ewald: null array");
    need_ctx(c)->ewald(to_plan(plan), n_src, src, n_tgt, tgt, str, u, level, false, info);
  });
}

int sdmk_ewald_device(sdmk_context* c, const sdmk_plan* plan, int64_t n_src, const double* d_src, int64_t n_tgt,
                      const double* d_tgt, const double* d_str, double* d_u, int level, double* info) {
  return guarded([&] {
    if (!plan || !d_src || !d_str || !d_u || (n_tgt > 0 && !d_tgt)) throw InvalidArgument("ewald: null array");
    need_ctx(c)->ewald(to_plan(plan), n_src, d_src, n_tgt, d_tgt, d_str, d_u, level, true, info);
  });
}

int sdmk_direct_sum(sdmk_context* c, int kernel, int dim, int64_t n_src, const double* src, int64_t n_tgt,
                    const double* tgt, const double* str, double* u) {
  return guarded([&] {
    if (!src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("direct_sum: null array");
    need_ctx(c)->direct(kernel, dim, n_src, src, n_tgt, tgt, str, nullptr, 1.0, false, u, false);
  });
}

int sdmk_direct_residual_sum(sdmk_context* c, const sdmk_plan* plan, int dim, int64_t n_src, const double* src,
                             int64_t n_tgt, const double* tgt, const double* str, double cutoff, int periodic,
                             double* u) {
  return guarded([&] {
    if (!plan || !src || !str || !u || (n_tgt > 0 && !tgt)) throw InvalidArgument("direct_residual_sum: null array");
    Context* x = need_ctx(c);
    const Tables& t = x->tables_for(to_plan(plan));
    x->direct(t.kernel, dim, n_src, src, n_tgt, tgt, str, &t, cutoff, periodic != 0, u, false);
  });
}

int sdmk_set_shard(sdmk_context* c, int rank, int nranks) {
  return guarded([&] { need_ctx(c)->set_shard(rank, nranks); });
}

int sdmk_comm_unique_id(unsigned char id[128]) {
  return guarded([&] {
    if (!id) throw InvalidArgument("sdmk_comm_unique_id: null output");
    Comm::unique_id(id);
  });
}

int sdmk_comm_init(sdmk_context* c, int rank, int nranks, const unsigned char id[128]) {
  return guarded([&] {
    if (!id) throw InvalidArgument("sdmk_comm_init: null id");
    need_ctx(c)->comm_init(rank, nranks, id);
  });
}

int sdmk_set_manual_exchange(sdmk_context* c, int on) {
  return guarded([&] { need_ctx(c)->set_manual_exchange(on != 0); });
}

int sdmk_evaluate_begin(sdmk_context* c, const sdmk_plan* plan, int dim, int64_t ns, const double* src, int64_t nt,
                        const double* tgt, const double* str, int mode, int device_ptrs) {
  return guarded([&] {
    if (!plan || !src || !str || (nt > 0 && !tgt)) throw InvalidArgument("sdmk_evaluate_begin: null pointer");
    need_ctx(c)->evaluate_begin(to_plan(plan), dim, ns, src, nt, tgt, str, mode, device_ptrs != 0);
  });
}

int sdmk_halo_transfer(sdmk_context* from, sdmk_context* to) {
  return guarded([&] {
    Context* a = need_ctx(from);
    Context* b = need_ctx(to);
    const int ra = a->shard_rank(), rb = b->shard_rank();
    double *src = nullptr, *dst = nullptr;
    int64_t ns = 0, nr = 0;
    a->halo_slab(rb, false, &src, &ns);
    b->halo_slab(ra, true, &dst, &nr);
    if (ns != nr) throw InvalidArgument("sdmk_halo_transfer: slab sizes differ (different problems or shards?)");
    if (ns > 0) {
      cuda_check(cudaStreamSynchronize(a->stream()), "stream synchronize");
      cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * ns, cudaMemcpyDefault, b->stream()), "halo copy");
      cuda_check(cudaStreamSynchronize(b->stream()), "stream synchronize");
    }
  });
}

int sdmk_evaluate_end(sdmk_context* c, double* u, sdmk_report* rep) {
  return guarded([&] {
    if (!u) throw InvalidArgument("sdmk_evaluate_end: null output");
    need_ctx(c)->evaluate_end(u, rep);
  });
}

int sdmk_get_stream(sdmk_context* c, void** stream) {
  return guarded([&] { *stream = (void*)need_ctx(c)->stream(); });
}

int sdmk_fp64_peak(sdmk_context* c, double* tflops) {
  return guarded([&] {
    Context* x = need_ctx(c);
    *tflops = measure_fp64_peak_tflops(x->stream());
    cuda_check(cudaGetLastError(), "fp64 peak kernel");
  });
}

int sdmk_set_guard(sdmk_context* c, int on) {
  return guarded([&] { need_ctx(c)->set_guard(on != 0); });
}

int64_t sdmk_guard_check(sdmk_context* c, char* names, int64_t cap) {
  int64_t n = -1;
  const int rc = guarded([&] {
    const std::vector<std::string> bad = need_ctx(c)->guard_check();
    std::string s;
    for (auto& b : bad) s += b + "\n";
    if (names && cap > 0) {
      const size_t k = std::min<size_t>(s.size(), (size_t)cap - 1);
      std::memcpy(names, s.data(), k);
      names[k] = 0;
    }
    n = (int64_t)bad.size();
  });
  return rc == 0 ? n : -1;
}

int sdmk_guard_selftest(sdmk_context* c) {
  int caught = 0;
  const int rc = guarded([&] { caught = need_ctx(c)->guard_selftest() ? 1 : 0; });
  return rc == 0 ? caught : -1;
}

int sdmk_fp64_mma_peak(sdmk_context* c, double* tflops) {
  return guarded([&] {
    Context* x = need_ctx(c);
    *tflops = measure_dmma_peak_tflops(x->stream());
    cuda_check(cudaGetLastError(), "fp64 mma peak kernel");
  });
}

int sdmk_host_save_tables(const sdmk_plan* plan, const char* path) {
  return guarded([&] { save_tables(tables_for_plan(to_plan(plan)), path ? path : ""); });
}

int sdmk_host_symbol_table(const sdmk_plan* plan, double h, int s2max, int kind, double rc, double rf, double* out) {
  return guarded([&] {
    Tables t = tables_for_plan(to_plan(plan));
    std::vector<double> A = symbol_table(t, h, s2max, kind, rc, rf);
    std::memcpy(out, A.data(), A.size() * sizeof(double));
  });
}

int64_t sdmk_host_topology_dump(int dim, int periodic, int n_s, int p, int64_t ns, const int32_t* qs, int64_t nt,
                                const int32_t* qt, char* buf, int64_t cap) {
  int64_t len = -1;
  guarded([&] {
    HostTree t = build_topology(dim, periodic != 0, n_s, p, (int)ns, qs, (int)nt, qt);
    std::string s = dump_topology(t);
    len = (int64_t)s.size();
    if (buf && cap > 0) std::memcpy(buf, s.data(), (size_t)std::min<int64_t>(cap, len));
  });
  return len;
}

int sdmk_host_shard_plan(int dim, int periodic, int n_s, int p, int64_t ns, const int32_t* qs, int64_t nt,
                         const int32_t* qt, int rank, int nranks, int64_t* out) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("shard plan: need 0 <= rank < nranks");
    HostTree t = build_topology(dim, periodic != 0, n_s, p, (int)ns, qs, (int)nt, qt);
    ShardPlan sp = shard_plan(t, rank, nranks);
    int64_t need = 0, tl = 0;
    for (char x : sp.need) need += x;
    for (int b = 0; b < t.num_boxes(); ++b) tl += t.boxes[b].leaf && t.ntgt(b) > 0;
    out[0] = sp.t0;
    out[1] = sp.t1;
    out[2] = (int64_t)sp.leaves.size();
    out[3] = need;
    out[4] = tl;
  });
}

int sdmk_host_shard_bounds(int dim, int periodic, int n_s, int p, int64_t ns, const int32_t* qs, int64_t nt,
                           const int32_t* qt, int nranks, int64_t* out) {
  return guarded([&] {
    if (nranks < 1) throw InvalidArgument("shard bounds: need nranks >= 1");
    HostTree t = build_topology(dim, periodic != 0, n_s, p, (int)ns, qs, (int)nt, qt);
    ShardCosts costs = shard_costs(t);
    std::vector<int64_t> b = shard_bounds(t, nranks, costs);
    std::copy(b.begin(), b.end(), out);
  });
}

int sdmk_host_halo_plan(int dim, int periodic, int n_s, int p, int64_t ns, const int32_t* qs, int64_t nt,
                        const int32_t* qt, int nranks, int64_t* out) {
  return guarded([&] {
    if (nranks < 1) throw InvalidArgument("halo plan: need nranks >= 1");
    HostTree t = build_topology(dim, periodic != 0, n_s, p, (int)ns, qs, (int)nt, qt);
    HaloPlan h = halo_owners(t, nranks);
    halo_reads(t, h);
    for (int f = 0; f < nranks; ++f)
      for (int r = 0; r < nranks; ++r) out[f * nranks + r] = (int64_t)halo_boxes(h, f, r).size();
    int64_t* o = out + nranks * nranks;
    for (int r = 0; r < nranks; ++r) o[r] = 0;
    int64_t above = 0, ncut = 0;
    for (int b = 0; b < t.num_boxes(); ++b) {
      if (h.owner[b] >= 0 && t.boxes[b].leaf) ++o[h.owner[b]];
      above += h.owner[b] == -1;
      ncut += h.cut[b];
    }
    o[nranks] = above;
    o[nranks + 1] = ncut;
  });
}

}  // extern "C"
