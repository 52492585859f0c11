// FP64 throughput microbenchmarks: the roofline denominators for the
// FP64-bound kernels (MEASURED_PEAKS.json carries only HBM and bf16 peaks).
// DFMA: each thread runs 8 independent chains; every SM gets 4 x 256 threads.
// DMMA (mma.sync.m8n8k4.f64, the FP64 tensor-core instruction): each warp runs
// 8 independent accumulator chains; every SM gets 2 x 256 threads.
#include "common.cuh"
#include "launch.hpp"

namespace sdmkb {

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b);
      x1 = fma(x1, a, b);
      x2 = fma(x2, a, b);
      x3 = fma(x3, a, b);
      x4 = fma(x4, a, b);
      x5 = fma(x5, a, b);
      x6 = fma(x6, a, b);
      x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) dev::dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
double best_ms(K launch, cudaStream_t st) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

}  // namespace

double measure_dmma_peak_tflops(cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int iters = 2048, blocks = sms * 2;
  k_dmma<<<blocks, 256, 0, st>>>(out, 32, 1e-3, 1e-3);  // warm-up / clock ramp
  const double ms = best_ms([&] { k_dmma<<<blocks, 256, 0, st>>>(out, iters, 1e-3, 1e-3); }, st);
  cudaFree(out);
  // one m8n8k4 DMMA = 8 x 8 x 4 FMAs per warp
  const double flops = 2.0 * 256 * 4 * 8 * (double)iters * blocks * 8;
  return flops / (ms * 1e-3) / 1e12;
}

double measure_fp64_peak_tflops(cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int iters = 4096, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, 256, 0, st>>>(out, 64, 0.999999, 1e-7);  // warm-up / clock ramp
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    k_dfma<<<blocks, 256, 0, st>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace sdmkb
