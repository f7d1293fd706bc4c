// tcgen05.mma kind::tf32 issue-rate probe: one CTA per SM issues `iters` MMAs (M=128, N, K=8) back
// to back from shared memory (no-swizzle K-major operands) into TMEM; prints cycles per MMA and the
// implied TF32 FLOP/s per SM.  Used to bound the nodal tcgen05 kernel (bbdg_tc.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1512_06025_b200/csrc -I include \
//        -o /tmp/umma tools/microbench/umma_tf32.cu && /tmp/umma
#include <cstdio>

#include "bbdg_tc.cuh"

using namespace bbdg;

template <int NN>
__global__ void probe(int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + NN) * 8; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&slot)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    const uint32_t a = smem_u32(sm), b = a + 128 * 8 * 4;
    const uint64_t da = umma_desc(a, 128, 256), db = umma_desc(b, 128, 256);
    const uint32_t idesc = umma_idesc_tf32(128, NN);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_tf32(slot, da, db, idesc, i > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "n"(256));
}

template <int NN> void run(int iters) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = (128 + NN) * 8 * 4;
  cudaFuncSetAttribute(probe<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<NN><<<148, 128, smem>>>(iters, d);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / iters;
  const double flops = 2.0 * 128 * NN * 8;
  printf("N=%3d: %.1f cycles per MMA, %.0f flop/cycle/SM = %.2f TFLOP/s per SM at 1.965 GHz (x148 = %.0f TF)  [%s]\n",
         NN, cyc, flops / cyc, flops / cyc * 1.965e9 / 1e12, flops / cyc * 1.965e9 * 148 / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64>(4096);
  run<128>(4096);
  run<192>(4096);
  run<256>(4096);
  return 0;
}
