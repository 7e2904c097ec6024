// Device helpers shared by the simulation, SVD and overlap kernels:
// complex128 arithmetic on double2, CTA/warp-group reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mpskq {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
// a * b
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a * b  (4 DFMA)
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a) * b  (4 DFMA)
__device__ __forceinline__ double2 cfmac(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double cnorm2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// A "thread group" of NT threads works on one state.  NT < 32: several
// groups share a warp (aligned lane slices); NT == 32: one warp; NT > 32: a CTA.
template <int NT>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (NT >= 32)
    return kFull;
  else
    return ((1u << NT) - 1u) << ((threadIdx.x & 31) & ~(NT - 1));
}

template <int NT>
__device__ __forceinline__ void bsync() {
  if constexpr (NT < 32)
    __syncwarp(group_mask<NT>());
  else if constexpr (NT == 32)
    __syncwarp();
  else
    __syncthreads();
}

template <int NT>
__device__ __forceinline__ int block_any(int v) {
  if constexpr (NT <= 32) {
    const unsigned m = group_mask<NT>();
    __syncwarp(m);
    return __any_sync(m, v);
  } else
    return __syncthreads_or(v);
}

// sum over aligned groups of G lanes (G a power of two <= 32); every lane in
// `mask` must call it.  The xor butterfly gives all lanes of a group the
// bitwise-identical result.
__device__ __forceinline__ double group_sum(double v, int G, unsigned mask = kFull) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}
__device__ __forceinline__ double2 group_sum(double2 v, int G, unsigned mask = kFull) {
  for (int o = G >> 1; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(mask, v.x, o);
    v.y += __shfl_xor_sync(mask, v.y, o);
  }
  return v;
}

// sum over the thread group, identical on every thread.  `red` needs NT/32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  if constexpr (NT < 32) {
    return group_sum(v, NT, group_mask<NT>());
  } else if constexpr (NT == 32) {
    return group_sum(v, 32);
  } else {
    v = group_sum(v, 32);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += red[i];
    return s;
  }
}

// lanes per work item so that G * items <= NT, G in [1, 32]
template <int NT>
__device__ __forceinline__ int group_width(int items) {
  int G = 32;
  while (G > 1 && G * items > NT) G >>= 1;
  return G;
}

}  // namespace mpskq

// ---------------------------------------------------------------- TMA bulk copies + mbarriers
namespace mpskq {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
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

}  // namespace mpskq
