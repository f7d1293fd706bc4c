// Operator-level entry points of the reference ops bundle, on the device:
//
//   bbdg_ops_grad     BernsteinRefOps.grad (bernstein.py:436-444): the four barycentric
//                     derivatives (<= 4 lanes per row, derivative_ops :182-218) by index
//                     arithmetic, combined as dr = (d1 - d0)/2, ds = (d2 - d0)/2, dt = (d3 - d0)/2
//   bbdg_ops_lift     lift_apply_factorized / lift_apply_optimal (bernstein.py:301-329): per face
//                     w = L0 flux_f, then N one-degree reductions, layer j scaled by ell_j
//                     (the factorised lift E_L L0 applied as sparse sweeps; E_L is never formed)
//   bbdg_dense_apply  opcount.dense_apply (opcount.py:38-43): y = x A^T, used for the dense lift
//                     (bernstein.py:332-347, nodal.py:236-241) and the nodal grad (nodal.py:220-225)
//
// These serve the reference's operator-level API (any degree 1..20, any batch), not the
// per-timestep hot path, which runs the fused mesh kernels of bbdg_opt.cuh.  Deterministic:
// each output is written by one thread in a fixed summation order.
#include <algorithm>

#include "bbdg_common.cuh"
#include "bbdg_internal.h"
#include "bbdg_tile.cuh"

namespace bbdg {
namespace {

constexpr int kOpsMaxDegree = 20;   // reference multiindex.MAX_DEGREE (multiindex.py:22)

// (D^i q)[alpha] = sum_j alpha_j q[alpha + e_i - e_j]   (lanes with alpha_j = 0 vanish)
template <typename T>
__global__ void ops_grad_kernel(int N, int64_t nb, const T* __restrict__ q, T* __restrict__ dr, T* __restrict__ ds,
                                T* __restrict__ dt) {
  const int Np = tet_dim(N);
  const int64_t total = nb * Np;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = x / Np;
    const int r = (int)(x - b * Np);
    int a0, a1, a2;
    decode3(N, r, a0, a1, a2);
    const int al[4] = {a0, a1, a2, N - a0 - a1 - a2};
    const T* qb = q + b * Np;
    T d[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      T s = T(0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (al[j] == 0) continue;
        int g[4] = {al[0], al[1], al[2], al[3]};
        g[i] += 1;
        g[j] -= 1;
        s += T(al[j]) * qb[pos3(N, g[0], g[1], g[2])];
      }
      d[i] = s;
    }
    const T h = T(0.5);
    dr[x] = h * (d[1] - d[0]);
    ds[x] = h * (d[2] - d[0]);
    dt[x] = h * (d[3] - d[0]);
  }
}

// one CTA per batch row: out (Np) = sum_f sum_j ell_j (R_j ... R_1 L0 flux_f) on layer j of face f
template <typename T>
__global__ void ops_lift_kernel(int N, int64_t nb, const T* __restrict__ flux, T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sraw[];
  const int Np = tet_dim(N), Nfp = tri_dim(N);
  T* so = reinterpret_cast<T*>(sraw);   // [Np]
  T* wa = so + Np;                      // [Nfp]
  T* wb = wa + Nfp;                     // [Nfp]
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    for (int i = threadIdx.x; i < Np; i += blockDim.x) so[i] = T(0);
    const T* fb = flux + b * 4 * Nfp;
    for (int f = 0; f < 4; ++f) {
      __syncthreads();
      // w = L0 flux_f: L0[c,c] = 1/2 sum_j (c_j+1)^2, L0[c, c+e_j-e_k] = 1/2 (c_j+1) c_k   (bernstein.py:221-229)
      for (int m = threadIdx.x; m < Nfp; m += blockDim.x) {
        int c0, c1;
        decode2(N, m, c0, c1);
        const int c[3] = {c0, c1, N - c0 - c1};
        T s = T(0.5 * double((c[0] + 1) * (c[0] + 1) + (c[1] + 1) * (c[1] + 1) + (c[2] + 1) * (c[2] + 1))) *
              fb[f * Nfp + m];
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k) {
            if (j == k || c[k] == 0) continue;
            int g[3] = {c[0], c[1], c[2]};
            g[j] += 1;
            g[k] -= 1;
            s += T(0.5 * double((c[j] + 1) * c[k])) * fb[f * Nfp + pos2(N, g[0], g[1])];
          }
        wa[m] = s;
      }
      T* w = wa;
      T* wn = wb;
      for (int j = 0; j <= N; ++j) {
        const int ml = N - j;   // degree of layer j's face space
        __syncthreads();
        if (j > 0) {
          // one-degree reduction (E^{ml+1}_{ml})^T: out[c] = sum_k (c_k+1)/(ml+1) w[c+e_k]   (bernstein.py:290-295)
          for (int m = threadIdx.x; m < tri_dim(ml); m += blockDim.x) {
            int c0, c1;
            decode2(ml, m, c0, c1);
            const int c[3] = {c0, c1, ml - c0 - c1};
            const T inv = T(1.0 / double(ml + 1));
            T s = T(0);
            for (int k = 0; k < 3; ++k) {
              int g[3] = {c[0], c[1], c[2]};
              g[k] += 1;
              s += T(c[k] + 1) * inv * w[pos2(ml + 1, g[0], g[1])];
            }
            wn[m] = s;
          }
          __syncthreads();
          T* t = w;
          w = wn;
          wn = t;
        }
        // layer j of face f: alpha with alpha_f = j, in the 2-D order of the other three indices
        const T ell = T(ell_of(N, j));
        for (int m = threadIdx.x; m < tri_dim(ml); m += blockDim.x) {
          int c0, c1;
          decode2(ml, m, c0, c1);
          const int c[3] = {c0, c1, ml - c0 - c1};
          int a[4], s = 0;
          for (int v = 0; v < 4; ++v) a[v] = (v == f) ? j : c[s++];
          const int pos = pos3(N, a[0], a[1], a[2]);
          so[pos] += j == 0 ? w[m] : ell * w[m];
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < Np; i += blockDim.x) out[b * Np + i] = so[i];
    __syncthreads();
  }
}

// y (nb, nr) = x (nb, nc) A^T with A (nr, nc) row-major: 32 x 32 output tiles, k tiles of 32
template <typename T>
__global__ void __launch_bounds__(256) dense_apply_kernel(int64_t nb, int nr, int nc, const T* __restrict__ A,
                                                          const T* __restrict__ x, T* __restrict__ y) {
  __shared__ T sx[32][33], sa[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 rows of 32 threads
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  T acc[4] = {T(0), T(0), T(0), T(0)};
  for (int c0 = 0; c0 < nc; c0 += 32) {
    for (int i = ty; i < 32; i += 8) {
      const int64_t b = b0 + i;
      const int c = c0 + tx;
      sx[i][tx] = (b < nb && c < nc) ? x[b * nc + c] : T(0);
      const int r = r0 + i;
      sa[i][tx] = (r < nr && c < nc) ? A[(int64_t)r * nc + c] : T(0);
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const T a = sa[tx][k];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += sx[ty + 8 * u][k] * a;
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t b = b0 + ty + 8 * u;
    const int r = r0 + tx;
    if (b < nb && r < nr) y[b * nr + r] = acc[u];
  }
}

int grid_for(int64_t work, int threads) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, (int64_t)sms * 16));
}

int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, what);
}

}  // namespace
}  // namespace bbdg

using namespace bbdg;

extern "C" {

int bbdg_ops_grad(int N, int dtype, int64_t nb, const void* q, void* dr, void* ds, void* dt, void* stream) {
  if (N < 1 || N > kOpsMaxDegree) return set_error(BBDG_ERR_UNSUPPORTED, "degree outside 1..20");
  if (nb < 0 || (nb > 0 && (!q || !dr || !ds || !dt))) return set_error(BBDG_ERR_ARG, "bad grad arguments");
  if (nb == 0) return BBDG_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(nb * tet_dim(N), 256);
  if (dtype == BBDG_F32)
    ops_grad_kernel<float><<<grid, 256, 0, s>>>(N, nb, static_cast<const float*>(q), static_cast<float*>(dr),
                                                static_cast<float*>(ds), static_cast<float*>(dt));
  else if (dtype == BBDG_F64)
    ops_grad_kernel<double><<<grid, 256, 0, s>>>(N, nb, static_cast<const double*>(q), static_cast<double*>(dr),
                                                 static_cast<double*>(ds), static_cast<double*>(dt));
  else
    return set_error(BBDG_ERR_ARG, "unknown dtype");
  return launch_status("grad launch");
}

int bbdg_ops_lift(int N, int dtype, int64_t nb, const void* flux, void* out, void* stream) {
  if (N < 1 || N > kOpsMaxDegree) return set_error(BBDG_ERR_UNSUPPORTED, "degree outside 1..20");
  if (nb < 0 || (nb > 0 && (!flux || !out))) return set_error(BBDG_ERR_ARG, "bad lift arguments");
  if (nb == 0) return BBDG_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<int64_t>(nb, 148 * 16);
  const size_t sz = dtype == BBDG_F32 ? 4 : 8;
  const size_t smem = (tet_dim(N) + 2 * tri_dim(N)) * sz;
  if (dtype == BBDG_F32)
    ops_lift_kernel<float><<<grid, 128, smem, s>>>(N, nb, static_cast<const float*>(flux), static_cast<float*>(out));
  else if (dtype == BBDG_F64)
    ops_lift_kernel<double><<<grid, 128, smem, s>>>(N, nb, static_cast<const double*>(flux),
                                                    static_cast<double*>(out));
  else
    return set_error(BBDG_ERR_ARG, "unknown dtype");
  return launch_status("lift launch");
}

int bbdg_dense_apply(int dtype, int64_t nb, int nrows, int ncols, const void* A, const void* x, void* y,
                     void* stream) {
  if (nb < 0 || nrows < 1 || ncols < 1 || (nb > 0 && (!A || !x || !y)))
    return set_error(BBDG_ERR_ARG, "bad dense apply arguments");
  if (nb == 0) return BBDG_OK;
  if ((nb + 31) / 32 > 0x7fffffff) return set_error(BBDG_ERR_ARG, "batch too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 grid((unsigned)((nb + 31) / 32), (unsigned)((nrows + 31) / 32));
  if (dtype == BBDG_F32)
    dense_apply_kernel<float><<<grid, 256, 0, s>>>(nb, nrows, ncols, static_cast<const float*>(A),
                                                   static_cast<const float*>(x), static_cast<float*>(y));
  else if (dtype == BBDG_F64)
    dense_apply_kernel<double><<<grid, 256, 0, s>>>(nb, nrows, ncols, static_cast<const double*>(A),
                                                    static_cast<const double*>(x), static_cast<double*>(y));
  else
    return set_error(BBDG_ERR_ARG, "unknown dtype");
  return launch_status("dense apply launch");
}

}  // extern "C"
