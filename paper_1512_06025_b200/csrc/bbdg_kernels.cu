// Instantiation unit: compiled once per (BBDG_T, BBDG_N) so the 2 x 9 degree /
// dtype combinations build in parallel.  Exposes a launcher table entry
// through a C++ symbol named after the pair.
#include "bbdg_internal.h"
#include "bbdg_tile.cuh"

#ifndef BBDG_T
#error "BBDG_T (float|double) must be defined"
#endif
#ifndef BBDG_N
#error "BBDG_N must be defined"
#endif

namespace bbdg {
namespace {

template <int OP, int LIFT, int BASIS> int launch(const void* vp, cudaStream_t stream, int num_sms) {
  using T = BBDG_T;
  using L = Layout<T, BBDG_N, OP, LIFT, BASIS>;
  static int blocks_per_sm = -1;
  auto kern = tile_kernel<T, BBDG_N, OP, LIFT, BASIS>;
  if (blocks_per_sm < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, L::threads, L::total);
    if (e != cudaSuccess) return set_cuda_error(e, "occupancy");
    if (b < 1) return set_error(BBDG_ERR_UNSUPPORTED, "tile kernel does not fit on an SM");
    blocks_per_sm = b;
  }
  const Params<T>& p = *static_cast<const Params<T>*>(vp);
  const int64_t ntiles = (p.kend - p.kbeg + L::KE - 1) / L::KE;
  if (ntiles == 0) return BBDG_OK;
  const int64_t grid = std::min<int64_t>((ntiles + L::NG - 1) / L::NG, (int64_t)num_sms * blocks_per_sm);
  kern<<<(unsigned)grid, L::threads, L::total, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "tile kernel launch");
}

template <int OP, int LIFT, int BASIS> int64_t smem() { return Layout<BBDG_T, BBDG_N, OP, LIFT, BASIS>::total; }

}  // namespace

#define BBDG_CAT_(a, b, c) a##_##b##_##c
#define BBDG_CAT(a, b, c) BBDG_CAT_(a, b, c)

KernelEntry BBDG_CAT(entry, BBDG_TNAME, BBDG_N)(int op, int lift, int basis) {
  KernelEntry k{nullptr, nullptr, group_elems<BBDG_N>()};
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
#undef BBDG_CASE
  return k;
}

}  // namespace bbdg
