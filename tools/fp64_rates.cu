// Issue-rate microbenchmark for the FP64-pipe instructions on k_residual's
// per-pair path (DFMA, DADD, DSETP, F2F f64<->f32, F2I/I2F f64, MUFU rsqrt
// f32 and the f64 high-word approximation).  Each thread runs 8 independent
// chains so latency is hidden; the kernel reports warp-instructions per
// clock per SM.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/fp64_rates.cu -o /tmp/fp64_rates
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

template <int OP>
__global__ void k_rate(double* out, double seed, long long* clk) {
  double a[kChains];
  float f[kChains];
  int n[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    a[c] = seed + threadIdx.x * 1e-3 + c;
    f[c] = (float)a[c];
    n[c] = threadIdx.x + c;
  }
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) a[c] = fma(a[c], 0.999999, 1e-7);                                   // DFMA
      if (OP == 1) a[c] = a[c] + 1e-7;                                                // DADD
      if (OP == 2) a[c] = (a[c] < 3.0) ? a[c] + 1e-9 : a[c];                          // DSETP (+DADD)
      if (OP == 3) f[c] = (float)((double)f[c] * 1.0000001);                          // F2F x2 (+DMUL)
      if (OP == 4) n[c] = (int)((double)n[c] + 0.5);                                  // I2F + F2I (+DADD)
      if (OP == 5) f[c] = rsqrtf(f[c] + 1.0f);                                        // MUFU.RSQ f32
      if (OP == 6) {                                                                  // MUFU.RSQ64H
        double r;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[c] + 1.0));
        a[c] = r;
      }
      if (OP == 7) a[c] = __dadd_rd(a[c], 0x1p52) - 0x1p52 + 0.25;                     // floor via DADD.RD
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c] + f[c] + n[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int ops_per_step, double* out, long long* clk) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 4;
  k_rate<OP><<<blocks, threads>>>(out, 1.0, clk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<OP><<<blocks, threads>>>(out, 1.0, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int mhz = 0;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  const double warp_instr = (double)blocks * threads / 32 * kIters * kChains * ops_per_step;
  const double cycles = ms * 1e-3 * (mhz * 1e3);
  printf("%-28s %8.2f ms  %6.2f warp-instr/clk/SM (at %d MHz nominal)\n", name, ms, warp_instr / cycles / sms, mhz / 1000);
}

int main() {
  double* out;
  long long* clk;
  cudaMalloc(&out, 148 * 4 * 512 * sizeof(double));
  cudaMalloc(&clk, sizeof(long long));
  run<0>("DFMA", 1, out, clk);
  run<1>("DADD", 1, out, clk);
  run<2>("DSETP+DADD(sel)", 2, out, clk);
  run<3>("F2F.F64.F32+DMUL+F2F.F32.F64", 3, out, clk);
  run<4>("I2F.F64+DADD+F2I.F64", 3, out, clk);
  run<5>("FADD+MUFU.RSQ", 2, out, clk);
  run<6>("DADD+MUFU.RSQ64H", 2, out, clk);
  run<7>("DADD.RD+DADD+DADD", 3, out, clk);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
