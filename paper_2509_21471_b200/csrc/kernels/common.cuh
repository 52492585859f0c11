// Shared device-side definitions for the sm_100a DMK kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "launch.hpp"

namespace sdmkb {
namespace dev {

constexpr double kPI = 3.141592653589793238462643383279502884;

// Barycentric Lagrange basis on first-kind Chebyshev nodes with the exact-hit
// rule (dmk.cpp:39-53); nodes/weights come from the host (dmk.cpp:30-36).
__device__ __forceinline__ void cheb_basis(int p, const double* __restrict__ nodes,
                                           const double* __restrict__ wts, double x,
                                           double* __restrict__ out, int stride) {
  int hit = -1;
  for (int i = 0; i < p; ++i)
    if (x == nodes[i]) { hit = i; break; }
  if (hit >= 0) {
    for (int j = 0; j < p; ++j) out[j * stride] = (j == hit) ? 1.0 : 0.0;
    return;
  }
  double s = 0.0;
  for (int i = 0; i < p; ++i) {
    double v = __ddiv_rn(wts[i], __dsub_rn(x, nodes[i]));
    out[i * stride] = v;
    s = __dadd_rn(s, v);
  }
  double inv = __ddiv_rn(1.0, s);
  for (int i = 0; i < p; ++i) out[i * stride] = __dmul_rn(out[i * stride], inv);
}

// FP64 tensor-core MMA, D = A(8x4, row) * B(4x8, col) + C(8x8).  Fragments
// (g = lane >> 2, t = lane & 3): a = A[g][t], b = B[t][g],
// {c0, c1} = C[g][2t], C[g][2t+1].  On B200 this sustains ~37 TFLOP/s
// (vs ~34 for DFMA) with 1/8 of the issue slots (tools/microbench).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 8-byte cp.async global -> shared; !valid zero-fills the destination.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(sz));
}
// 16-byte cp.async (both addresses 16-byte aligned), L2 only
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
// 16-byte cp.async with zero fill when !valid
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// mbarrier + 1D bulk copy (TMA engine, no tensor map): global -> shared,
// completion counted in bytes on the barrier.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// expect bytes without arriving (several threads add their own copies' bytes
// to the phase, one of them arrives)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// shared -> global bulk store (bulk-group completion); the writer threads
// fence their generic-proxy shared writes first
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a += b * c
__device__ __forceinline__ void cfma(double2& a, double2 b, double2 c) {
  a.x = fma(b.x, c.x, a.x);
  a.x = fma(-b.y, c.y, a.x);
  a.y = fma(b.x, c.y, a.y);
  a.y = fma(b.y, c.x, a.y);
}
// a += conj(b) * c
__device__ __forceinline__ void cfma_conj(double2& a, double2 b, double2 c) {
  a.x = fma(b.x, c.x, a.x);
  a.x = fma(b.y, c.y, a.x);
  a.y = fma(b.x, c.y, a.y);
  a.y = fma(-b.y, c.x, a.y);
}

}  // namespace dev
}  // namespace sdmkb
