#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(double* out, int iters, double a, double b) {
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mma(c[2*j], c[2*j+1], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void kf(double* out, int iters, double a, double b) {
  double x[8]; for (int i=0;i<8;++i) x[i]=threadIdx.x*1e-9+i;
  for (int it=0; it<iters; ++it) {
#pragma unroll
    for (int k=0;k<16;++k)
#pragma unroll
      for (int j=0;j<8;++j) x[j]=fma(x[j],a,b);
  }
  double s=0; for(int i=0;i<8;++i) s+=x[i]; if(s==1.2345) out[0]=s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bs : {128, 256, 512}) for (int per : {2,4,8}) {
    int blocks = 148 * per; int iters = 20000;
    k<<<blocks, bs>>>(o, 100, 0.999, 1e-7);
    cudaEventRecord(e0); k<<<blocks, bs>>>(o, iters, 0.999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * blocks * (bs / 32);
    printf("DMMA bs=%d blocks=%d: %.2f TFLOP/s\n", bs, blocks, fl / ms / 1e9);
  }
  for (int bs : {256, 512}) for (int per : {2,4,8}) {
    int blocks=148*per, iters=4096;
    kf<<<blocks,bs>>>(o,64,0.999,1e-7);
    cudaEventRecord(e0); kf<<<blocks,bs>>>(o,iters,0.999,1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*8*16*(double)iters*blocks*bs;
    printf("DFMA bs=%d blocks=%d: %.2f TFLOP/s\n", bs, blocks, fl/ms/1e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock kHz %d\n", clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
