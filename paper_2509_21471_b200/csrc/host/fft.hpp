// cuFFT through dlopen (libcufft.so.11 is opened on first use, so users of
// the DMK path never need it): batched 3D real <-> half-complex transforms
// for the FFT Ewald far field.
#pragma once

#include <cuda_runtime.h>

namespace sdmkb {

class Fft3 {
 public:
  ~Fft3();
  // (re)plan for an n^3 grid, `batch` transforms, on stream st
  void plan(int n, int batch, cudaStream_t st);
  // forward: real [batch][n^3] (x fastest) -> half spectrum [batch][n][n][n/2+1]
  void forward(double* real, double2* half);
  // inverse (unnormalized): half spectrum -> real
  void inverse(double2* half, double* real);
  int n() const { return n_; }

 private:
  int fwd_ = 0, inv_ = 0;
  int n_ = 0, batch_ = 0;
  bool have_ = false;
};

}  // namespace sdmkb
