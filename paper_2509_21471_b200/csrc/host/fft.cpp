// cuFFT through dlopen (types from cufft.h, symbols resolved at first use).
#include "fft.hpp"

#include <cufft.h>
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "setup.hpp"

namespace sdmkb {

namespace {

struct Cufft {
  decltype(&cufftPlanMany) PlanMany = nullptr;
  decltype(&cufftSetStream) SetStream = nullptr;
  decltype(&cufftExecD2Z) ExecD2Z = nullptr;
  decltype(&cufftExecZ2D) ExecZ2D = nullptr;
  decltype(&cufftDestroy) Destroy = nullptr;
};

const Cufft& cufft() {
  static Cufft f;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libcufft.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libcufft.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcufft.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cuFFT: cannot open libcufft.so.11: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) err = std::string("cuFFT: missing symbol ") + name;
      return p;
    };
    f.PlanMany = (decltype(f.PlanMany))sym("cufftPlanMany");
    f.SetStream = (decltype(f.SetStream))sym("cufftSetStream");
    f.ExecD2Z = (decltype(f.ExecD2Z))sym("cufftExecD2Z");
    f.ExecZ2D = (decltype(f.ExecZ2D))sym("cufftExecZ2D");
    f.Destroy = (decltype(f.Destroy))sym("cufftDestroy");
  });
  if (!err.empty()) throw RuntimeError(err);
  return f;
}

void check(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) throw RuntimeError(std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

}  // namespace

Fft3::~Fft3() {
  if (have_) {
    cufft().Destroy((cufftHandle)fwd_);
    cufft().Destroy((cufftHandle)inv_);
  }
}

void Fft3::plan(int n, int batch, cudaStream_t st) {
  const Cufft& f = cufft();
  if (have_ && n == n_ && batch == batch_) {
    check(f.SetStream((cufftHandle)fwd_, st), "cufftSetStream");
    check(f.SetStream((cufftHandle)inv_, st), "cufftSetStream");
    return;
  }
  if (have_) {
    f.Destroy((cufftHandle)fwd_);
    f.Destroy((cufftHandle)inv_);
    have_ = false;
  }
  int dims[3] = {n, n, n};  // row-major: the last (x) index fastest
  const int rdist = n * n * n, cdist = n * n * (n / 2 + 1);
  cufftHandle a = 0, b = 0;
  check(f.PlanMany(&a, 3, dims, nullptr, 1, rdist, nullptr, 1, cdist, CUFFT_D2Z, batch), "cufftPlanMany D2Z");
  check(f.PlanMany(&b, 3, dims, nullptr, 1, cdist, nullptr, 1, rdist, CUFFT_Z2D, batch), "cufftPlanMany Z2D");
  fwd_ = (int)a;
  inv_ = (int)b;
  n_ = n;
  batch_ = batch;
  have_ = true;
  check(f.SetStream(a, st), "cufftSetStream");
  check(f.SetStream(b, st), "cufftSetStream");
}

void Fft3::forward(double* real, double2* half) {
  check(cufft().ExecD2Z((cufftHandle)fwd_, real, reinterpret_cast<cufftDoubleComplex*>(half)), "cufftExecD2Z");
}

void Fft3::inverse(double2* half, double* real) {
  check(cufft().ExecZ2D((cufftHandle)inv_, reinterpret_cast<cufftDoubleComplex*>(half), real), "cufftExecZ2D");
}

}  // namespace sdmkb
