// Shared device building blocks for the BB-DG sm_100a kernels.
//
// Index arithmetic for the canonical barycentric order of the reference
// (/root/reference/pkg/src/bbdg/multiindex.py:1-12,48-61), TMA bulk-copy /
// mbarrier helpers, and per-degree compile-time dimensions.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bbdg {

template <int N> struct Dims {
  static constexpr int Np = (N + 1) * (N + 2) * (N + 3) / 6;   // tet space
  static constexpr int Nfp = (N + 1) * (N + 2) / 2;            // face space
  static constexpr int Npm = N * (N + 1) * (N + 2) / 6;        // degree N-1 tet space
};

__host__ __device__ constexpr int tri_dim(int m) { return (m + 1) * (m + 2) / 2; }
__host__ __device__ constexpr int tet_dim(int m) { return (m + 1) * (m + 2) * (m + 3) / 6; }

// pos2: canonical position of (b0, b1, m-b0-b1) in the degree-m triangle space.
__host__ __device__ __forceinline__ int pos2(int m, int b0, int b1) {
  return b0 * (m + 1) - (b0 * (b0 - 1)) / 2 + b1;
}
// pos3: canonical position of (a0, a1, a2, m-a0-a1-a2) in the degree-m tet space.
__host__ __device__ __forceinline__ int pos3(int m, int a0, int a1, int a2) {
  const int r = m - a0;  // remaining degree after a0
  return tet_dim(m) - tet_dim(r) + pos2(r, a1, a2);
}

// ---------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk) + mbarrier, sm_90+/sm_100a PTX.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// expect tx bytes on the current phase without arriving (several producer lanes)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk copy with an L2 eviction-priority policy (createpolicy: evict_last keeps a line for a re-read,
// evict_first lets a last read go first)
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                  uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <typename T> __device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// streaming stores: results are not re-read by this kernel
template <typename T> __device__ __forceinline__ void st_stream(T* p, T v) { __stcs(p, v); }

}  // namespace bbdg
