// Instantiation unit: compiled once per (BBDG_T, BBDG_N) so the 2 x 9 degree /
// dtype combinations build in parallel.  Exposes a launcher table entry
// through a C++ symbol named after the pair.
#include <atomic>

#include "bbdg_internal.h"
#include "bbdg_ept.cuh"
#include "bbdg_nodal.cuh"
#include "bbdg_opt.cuh"
#include "bbdg_tc.cuh"

#ifndef BBDG_T
#error "BBDG_T (float|double) must be defined"
#endif
#ifndef BBDG_N
#error "BBDG_N must be defined"
#endif

namespace bbdg {
namespace {

// persistent launch: grid = min(#groups needed, SMs x resident CTAs), one CTA
// holds NG independent element groups
// Launch attributes are per device: each kernel keeps a per-device cache of its resident CTAs per
// SM (0 = not yet configured).  Concurrent first launches from several host threads may both set
// the (idempotent) attribute; the cache itself is atomic.
constexpr int kMaxDevices = 64;
using DevCache = std::atomic<int>[kMaxDevices];

inline int current_device() {
  int dev = 0;
  return cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < kMaxDevices ? dev : 0;
}

template <class KernT, int THREADS, int TOTAL, int KE, int NG>
int launch_persistent(KernT kern, DevCache& cache, const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  const int dev = current_device();
  int blocks_per_sm = cache[dev].load(std::memory_order_acquire);
  if (blocks_per_sm < 1) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TOTAL);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, THREADS, TOTAL);
    if (e != cudaSuccess) return set_cuda_error(e, "occupancy");
    if (b < 1) return set_error(BBDG_ERR_UNSUPPORTED, "tile kernel does not fit on an SM");
    blocks_per_sm = b;
    cache[dev].store(b, std::memory_order_release);
  }
  const Params<T>& p = *static_cast<const Params<T>*>(vp);
  const int64_t ntiles = (p.kend - p.kbeg + KE - 1) / KE;
  if (ntiles == 0) return BBDG_OK;
  const int64_t grid = std::min<int64_t>((ntiles + NG - 1) / NG, (int64_t)num_sms * blocks_per_sm);
  kern<<<(unsigned)grid, THREADS, TOTAL, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "tile kernel launch");
}

template <int OP, int FSR> int launch_opt(const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  using L = OptLayout<T, BBDG_N, OP, FSR>;
  static DevCache cache;
  return launch_persistent<decltype(&opt_kernel<T, BBDG_N, OP, FSR>), L::threads, L::total, L::KE, L::NG>(
      opt_kernel<T, BBDG_N, OP, FSR>, cache, vp, stream, num_sms);
}

#ifndef BBDG_EPT_MAX_N
#define BBDG_EPT_MAX_N 3   // element-per-thread register kernels for N <= this (bbdg_ept.cuh)
#endif
#ifndef BBDG_EPT_MAX_N64
#define BBDG_EPT_MAX_N64 2
#endif
constexpr bool kEpt = BBDG_N <= (sizeof(BBDG_T) == 4 ? BBDG_EPT_MAX_N : BBDG_EPT_MAX_N64);

// element-per-thread kernels: one warp per 32-element tile, W warps per CTA, one CTA per SM
template <int OP, int NN = BBDG_N> int launch_ept(const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  using L = EptLayout<T, NN>;   // (dependent: only the orders that dispatch here instantiate it)
  static DevCache attr;
  auto kern = ept_kernel<T, NN, OP>;
  const int dev = current_device();
  if (attr[dev].load(std::memory_order_acquire) == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute (ept)");
    attr[dev].store(1, std::memory_order_release);
  }
  const Params<T>& p = *static_cast<const Params<T>*>(vp);
  const int64_t ntiles = (p.kend - p.kbeg + L::KE - 1) / L::KE;
  if (ntiles == 0) return BBDG_OK;
  const int64_t grid = std::min<int64_t>((ntiles + L::W - 1) / L::W, (int64_t)num_sms);
  kern<<<(unsigned)grid, L::threads, L::total, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "ept kernel launch");
}

// nodal block-partitioned path: flux kernel (surface ops), then the tensor-core GEMM kernel
template <int OP> int launch_nodal(const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  using L = NodalLayout<T, BBDG_N>;
  const Params<T>& p = *static_cast<const Params<T>*>(vp);
  const int64_t nl = p.kend - p.kbeg;
  if (nl == 0) return BBDG_OK;
  if ((OP != OP_SURFACE && !p.bvol) || !p.blift || (sizeof(T) == 8 && !p.flux))
    return set_error(BBDG_ERR_UNSUPPORTED, "nodal MMA fragments not uploaded");
  if constexpr (OP != OP_VOLUME && sizeof(T) == 8) {
    const int64_t n = nl * 4 * Dims<BBDG_N>::Nfp;
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 8);
    nodal_flux_kernel<T, BBDG_N><<<(unsigned)grid, 256, 0, stream>>>(p);
  }
  static DevCache attr;
  const int dev = current_device();
  if constexpr (sizeof(T) == 4) {
    // fp32: tcgen05 kind::tf32 (3xTF32) with TMEM accumulators (bbdg_tc.cuh)
    using LT = TcLayout<BBDG_N>;
    auto kern = nodal_tc_kernel<BBDG_N, OP>;
    if (attr[dev].load(std::memory_order_acquire) == 0) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, LT::total);
      if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute (nodal tc)");
      attr[dev].store(1, std::memory_order_release);
    }
    if (!p.img_l || (OP != OP_SURFACE && !p.img_a))
      return set_error(BBDG_ERR_UNSUPPORTED, "tcgen05 operand images not allocated");
    const int64_t nsteps = (nl + LT::ST - 1) / LT::ST;
    // tf32 hi / lo images of the element chunks in the UMMA layout (the kernel streams them with TMA)
    const int pgrid = num_sms * 8;
    if constexpr (OP != OP_SURFACE)
      tc_pack_kernel<BBDG_N><<<pgrid, 256, 0, stream>>>(reinterpret_cast<const float*>(p.q + p.kbeg * LT::Np), p.K * LT::Np, LT::Np, LT::Np, LT::KV,
                                                        nl, static_cast<float*>(p.img_a));
    if constexpr (OP != OP_VOLUME) {
      const int64_t n = nl * 4 * LT::Nfp;
      tc_flux_kernel<BBDG_N><<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 8), 256, 0, stream>>>(
          reinterpret_cast<const Params<float>&>(p));
    }
    kern<<<(unsigned)std::min<int64_t>(nsteps, num_sms), LT::threads, LT::total, stream>>>(
        reinterpret_cast<const Params<float>&>(p));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "nodal tcgen05 kernel launch");
  }
  auto kern = nodal_mma_kernel<T, BBDG_N, OP>;
  if (attr[dev].load(std::memory_order_acquire) == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute (nodal)");
    attr[dev].store(1, std::memory_order_release);
  }
  const int64_t ntiles = (nl + L::ET - 1) / L::ET;
  kern<<<(unsigned)std::min<int64_t>(ntiles, num_sms), L::THREADS, L::total, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "nodal MMA kernel launch");
}

template <int OP, int LIFT, int BASIS> int launch(const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  if constexpr (BASIS == BASIS_NODAL && LIFT == LIFT_BLOCKED) {
    return launch_nodal<OP>(vp, stream, num_sms);
  } else if constexpr (BASIS == BASIS_BERNSTEIN && LIFT == LIFT_OPTIMAL) {   // also the "factorized" mode
    // field-plane stride residue (K Np) mod (16 / sizeof(T)) selects the smem field stride
    const Params<T>& p = *static_cast<const Params<T>*>(vp);
    constexpr int A = 16 / sizeof(T);
    const int fsr = (int)((p.K * Dims<BBDG_N>::Np) % A);
    if constexpr (kEpt && (OP == OP_STAGE || OP == OP_RHS)) {
      // 16-byte aligned field windows of every tile: the register kernel
      if (fsr == 0 && (p.kbeg * Dims<BBDG_N>::Np) % A == 0) return launch_ept<OP>(vp, stream, num_sms);
    }
    if constexpr (A == 4) {
      switch (fsr) {
        case 0: return launch_opt<OP, 0>(vp, stream, num_sms);
        case 1: return launch_opt<OP, 1>(vp, stream, num_sms);
        case 2: return launch_opt<OP, 2>(vp, stream, num_sms);
        default: return launch_opt<OP, 3>(vp, stream, num_sms);
      }
    } else {
      return fsr ? launch_opt<OP, 1>(vp, stream, num_sms) : launch_opt<OP, 0>(vp, stream, num_sms);
    }
  } else {
    static DevCache cache;
    using L = Layout<T, BBDG_N, OP, LIFT, BASIS>;
    return launch_persistent<decltype(&tile_kernel<T, BBDG_N, OP, LIFT, BASIS>), L::threads, L::total, L::KE, L::NG>(
        tile_kernel<T, BBDG_N, OP, LIFT, BASIS>, cache, vp, stream, num_sms);
  }
}

template <int OP, int LIFT, int BASIS> int64_t smem() {
  if constexpr (BASIS == BASIS_NODAL && LIFT == LIFT_BLOCKED) return NodalLayout<BBDG_T, BBDG_N>::total;
  else if constexpr (BASIS == BASIS_BERNSTEIN && LIFT == LIFT_OPTIMAL) return OptLayout<BBDG_T, BBDG_N, OP, 0>::total;
  else return Layout<BBDG_T, BBDG_N, OP, LIFT, BASIS>::total;
}

}  // namespace

#define BBDG_CAT_(a, b, c) a##_##b##_##c
#define BBDG_CAT(a, b, c) BBDG_CAT_(a, b, c)

KernelEntry BBDG_CAT(entry, BBDG_TNAME, BBDG_N)(int op, int lift, int basis) {
  KernelEntry k{nullptr, nullptr, OptLayout<BBDG_T, BBDG_N, OP_STAGE, 0>::KE};
#define BBDG_CASE(O, Lf, B)                            \
  if (op == O && lift == Lf && basis == B) {           \
    k.launch = &launch<O, Lf, B>;                      \
    k.smem = &smem<O, Lf, B>;                          \
    return k;                                          \
  }
  BBDG_CASE(OP_VOLUME, LIFT_OPTIMAL, BASIS_BERNSTEIN)
  BBDG_CASE(OP_SURFACE, LIFT_FACTORIZED, BASIS_BERNSTEIN)
  BBDG_CASE(OP_SURFACE, LIFT_OPTIMAL, BASIS_BERNSTEIN)
  BBDG_CASE(OP_SURFACE, LIFT_DENSE, BASIS_BERNSTEIN)
  BBDG_CASE(OP_RHS, LIFT_FACTORIZED, BASIS_BERNSTEIN)
  BBDG_CASE(OP_RHS, LIFT_OPTIMAL, BASIS_BERNSTEIN)
  BBDG_CASE(OP_RHS, LIFT_DENSE, BASIS_BERNSTEIN)
  BBDG_CASE(OP_STAGE, LIFT_FACTORIZED, BASIS_BERNSTEIN)
  BBDG_CASE(OP_STAGE, LIFT_OPTIMAL, BASIS_BERNSTEIN)
  BBDG_CASE(OP_STAGE, LIFT_DENSE, BASIS_BERNSTEIN)
  BBDG_CASE(OP_VOLUME, LIFT_DENSE, BASIS_NODAL)
  BBDG_CASE(OP_SURFACE, LIFT_DENSE, BASIS_NODAL)
  BBDG_CASE(OP_RHS, LIFT_DENSE, BASIS_NODAL)
  BBDG_CASE(OP_STAGE, LIFT_DENSE, BASIS_NODAL)
  BBDG_CASE(OP_VOLUME, LIFT_BLOCKED, BASIS_NODAL)
  BBDG_CASE(OP_SURFACE, LIFT_BLOCKED, BASIS_NODAL)
  BBDG_CASE(OP_RHS, LIFT_BLOCKED, BASIS_NODAL)
  BBDG_CASE(OP_STAGE, LIFT_BLOCKED, BASIS_NODAL)
#undef BBDG_CASE
  return k;
}

}  // namespace bbdg
