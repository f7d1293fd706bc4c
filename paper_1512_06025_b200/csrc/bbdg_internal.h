// Internal glue between the C ABI (bbdg_capi.cu) and the per-(dtype, degree)
// instantiation units (bbdg_kernels.cu compiled 2 x kMaxDegree times).
#pragma once
#include <algorithm>
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/bbdg.h"

namespace bbdg {

constexpr int kMaxDegree = 9;

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);

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
