// Internal glue between the C ABI (bbdg_capi.cu) and the per-(dtype, degree)
// instantiation units (bbdg_kernels.cu compiled 2 x kMaxDegree times).
#pragma once
#include <algorithm>
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/bbdg.h"

// One (mesh, degree, basis, dtype) context: immutable device tables after setup.
struct bbdg_ctx {
  int N, basis, dtype;
  int64_t K;
  int Np, Nfp;
  int num_sms;
  void* geo_vol = nullptr;   // T (K,12)  legacy records (tile / ELL / dense / nodal kernels); NULL when a
  void* geo_surf = nullptr;  // T (K,24)  box context was built with the fused record only
  void* geo = nullptr;       // T (K,36) fused record of the optimal-lift kernels (kGeoRec)
  int32_t* nbr = nullptr;    // (K,4)
  int32_t* code = nullptr;   // (K)
  void* el_vals = nullptr;   // T (Np,w)
  uint16_t* el_cols = nullptr;
  int el_w = 0;
  void* liftT = nullptr;     // T (4Nfp,Np)
  void* dT = nullptr;        // T (3,Np,Np)
  void* bvol = nullptr;      // nodal blocked: D_m^T MMA fragments
  void* blift = nullptr;     // nodal blocked: L^T MMA fragments
  void* flux = nullptr;      // nodal blocked / BB dense on the tensor cores: (4, K, 4 Nfp) face-flux scratch
  void* rhs_scratch = nullptr;   // BB dense fused stage: (4, K, Np) rhs (allocated on first use)
  void* stage_ring = nullptr;   // bbdg_step_pageable: pinned staging rings (cudaHostAlloc), in then out
  size_t stage_ring_bytes = 0;
  void* img_a = nullptr;     // fp32 tcgen05 path: packed tf32 hi/lo image of q (bbdg_tc.cuh, first use)
  void* img_l = nullptr;     // fp32 tcgen05 path: packed tf32 hi/lo image of the face fluxes
  const void* halo = nullptr;
  int64_t nhalo = 0;
};

namespace bbdg {

constexpr int kMaxDegree = 9;

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
void free_geometry(bbdg_ctx* c);

struct KernelEntry {
  int (*launch)(const void* params, cudaStream_t stream, int num_sms);
  int64_t (*smem)();
  int tile_elems;
};

#define BBDG_DECLARE(tn, n) KernelEntry entry_##tn##_##n(int op, int lift, int basis);
#define BBDG_DECLARE_ALL(tn) \
  BBDG_DECLARE(tn, 1) BBDG_DECLARE(tn, 2) BBDG_DECLARE(tn, 3) BBDG_DECLARE(tn, 4) BBDG_DECLARE(tn, 5) \
  BBDG_DECLARE(tn, 6) BBDG_DECLARE(tn, 7) BBDG_DECLARE(tn, 8) BBDG_DECLARE(tn, 9)
BBDG_DECLARE_ALL(f32)
BBDG_DECLARE_ALL(f64)
#undef BBDG_DECLARE_ALL
#undef BBDG_DECLARE

}  // namespace bbdg
