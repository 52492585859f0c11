// DMMA throughput vs. independent chains per warp and warps per SM (B200).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, int iters, double a, double b) {
  double c[2 * C];
  for (int i = 0; i < 2 * C; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < C; ++j) mma(c[2 * j], c[2 * j + 1], a, b);
  }
  double s = 0; for (int i = 0; i < 2 * C; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}
template <int C>
void run(double* o, int warps_per_sm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int bs = 32 * warps_per_sm, blocks = 148, iters = 40000 / C;
  k<C><<<blocks, bs>>>(o, 100, 0.999, 1e-7);
  cudaEventRecord(e0); k<C><<<blocks, bs>>>(o, iters, 0.999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * C * (double)iters * blocks * warps_per_sm;
  double cyc = ms * 1e-3 * 1.965e9;
  printf("chains/warp=%2d warps/SM=%2d  %6.2f TFLOP/s  cycles per DMMA per warp-chain %.1f\n", C, warps_per_sm,
         fl / ms / 1e9, cyc / iters);
}
int main() {
  double* o; cudaMalloc(&o, 8);
  for (int w : {1, 2, 4, 8, 16}) { run<1>(o, w); run<2>(o, w); run<4>(o, w); run<8>(o, w); }
  return 0;
}
