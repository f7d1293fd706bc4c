// Does SHFL share the shared-memory data pipe with LDS on sm_100a?
// A: LDS only, B: SHFL only, C: both interleaved (same counts as A and B).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  __shared__ float s[1024 * 2];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
  __syncthreads();
  float a = threadIdx.x, b = 1.f, c = 2.f, d = 3.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0 || MODE == 2) { a += s[(idx + u * 32) & 2047]; b += s[(idx + u * 32 + 256) & 2047]; }
      if (MODE == 1 || MODE == 2) { c += __shfl_down_sync(0xffffffff, c, 1); d += __shfl_xor_sync(0xffffffff, d, 3); }
    }
    idx = (idx + 7) & 2047;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 2, 1024>>>(o, iters);
      if (mode == 1) k<1><<<148 * 2, 1024>>>(o, iters);
      if (mode == 2) k<2><<<148 * 2, 1024>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = 148.0 * 2 * 1024 / 32 * iters * 8 * 2;  // warp-instructions of each kind
      if (rep) printf("mode %d (%s): %.3f ms  -> %.2f warp-ops/clk/SM at 1.92GHz\n", mode,
                      mode == 0 ? "LDS" : mode == 1 ? "SHFL" : "LDS+SHFL", ms, ops / (ms * 1e-3) / 148 / 1.92e9);
    }
  }
  return 0;
}
