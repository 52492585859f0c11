// FP64 tensor-core throughput by mma.sync shape on sm_100a: m8n8k4 (sm_80)
// vs m16n8k4 / m16n8k8 / m16n8k16 (sm_90+ shapes).  Independent chains per
// warp, registers only.  usage: ./fp64_mma_shapes
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void m884(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
}
__device__ __forceinline__ void m1684(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
__device__ __forceinline__ void m1688(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]),
                 "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void m16816(double* c, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE>
__global__ void k(double* out, int iters) {
  constexpr int NC = 4;  // independent accumulator chains
  double c[NC][4], a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int j = 0; j < NC; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (SHAPE == 0) m884(c[j], a, b);
      if (SHAPE == 1) m1684(c[j], a, b);
      if (SHAPE == 2) m1688(c[j], a, b);
      if (SHAPE == 3) m16816(c[j], a, b);
    }
  }
  double s = 0;
  for (int j = 0; j < NC; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double macs[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int shape = 0; shape < 4; ++shape)
    for (int bs : {128, 256, 512}) {
      const int blocks = 148 * 4, iters = 4000;
      auto launch = [&](int it) {
        if (shape == 0) k<0><<<blocks, bs>>>(o, it);
        if (shape == 1) k<1><<<blocks, bs>>>(o, it);
        if (shape == 2) k<2><<<blocks, bs>>>(o, it);
        if (shape == 3) k<3><<<blocks, bs>>>(o, it);
      };
      launch(10);
      cudaEventRecord(e0);
      launch(iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * macs[shape] * 4 * (double)iters * blocks * (bs / 32);
      printf("%-9s bs=%3d: %.2f TFLOP/s\n", names[shape], bs, fl / ms / 1e9);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
