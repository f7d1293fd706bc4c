// Device-resident functionals: the discrete energy of the energy
// guard (reference solver.py:306-312, 233-238) and the L2 error of the
// standing-wave pressure (ErrorFunctional, solver.py:282-296), so integrate()
// and the finite-precision study never copy a state to the host.
//
// One CTA per element computes its contribution in float64 (states may be
// float32); a second single-CTA pass sums the per-element partials in a fixed
// order, so the result is deterministic.
#include <cmath>

#include "bbdg_common.cuh"
#include "bbdg_internal.h"

namespace bbdg {
namespace {

constexpr int kFuncThreads = 256;

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  __syncthreads();
  return s;
}

// partial[k] = sum_F c[F][k] q_F^T M q_F   (M symmetric, read column-wise = coalesced)
template <typename T>
__global__ void __launch_bounds__(kFuncThreads) energy_kernel(int64_t K, int Np, const T* __restrict__ q,
                                                              const double* __restrict__ M,
                                                              const double* __restrict__ coef,
                                                              double* __restrict__ partial) {
  extern __shared__ double sq[];   // [4][Np]
  __shared__ double red[kFuncThreads / 32];
  const int64_t k = blockIdx.x;
  for (int i = threadIdx.x; i < 4 * Np; i += blockDim.x) {
    const int F = i / Np, a = i - F * Np;
    sq[i] = (double)q[((int64_t)F * K + k) * Np + a];
  }
  __syncthreads();
  double acc = 0.0;
  for (int a = threadIdx.x; a < Np; a += blockDim.x) {
    double mq[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = 0; b < Np; ++b) {
      const double m = M[(int64_t)b * Np + a];
#pragma unroll
      for (int F = 0; F < 4; ++F) mq[F] += m * sq[F * Np + b];
    }
#pragma unroll
    for (int F = 0; F < 4; ++F) acc += coef[F * K + k] * sq[F * Np + a] * mq[F];
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[k] = s;
}

// partial[k] = jac_k sum_q w_q (p_h(x_q) - p_exact(x_q, tau))^2, p_h = E q_0, standing wave of
// exact_solution (solver.py:249-261): p = cos(pi x) cos(pi y) cos(pi z) cos(sqrt3 pi tau)
template <typename T>
__global__ void __launch_bounds__(kFuncThreads) error_kernel(int64_t K, int Np, int nq, const T* __restrict__ q0,
                                                             const double* __restrict__ ET,
                                                             const double* __restrict__ wq,
                                                             const double* __restrict__ lam,
                                                             const double* __restrict__ verts,
                                                             const double* __restrict__ jac, double ct,
                                                             double* __restrict__ partial) {
  extern __shared__ double sq[];   // [Np]
  __shared__ double red[kFuncThreads / 32];
  const int64_t k = blockIdx.x;
  for (int a = threadIdx.x; a < Np; a += blockDim.x) sq[a] = (double)q0[k * Np + a];
  __syncthreads();
  const double* X = verts + k * 12;
  const double pi = 3.14159265358979323846;
  double acc = 0.0;
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    double ph = 0.0;
    for (int a = 0; a < Np; ++a) ph += ET[(int64_t)a * nq + i] * sq[a];
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int d = 0; d < 3; ++d) x[d] += lam[i * 4 + v] * X[v * 3 + d];
    const double pe = cos(pi * x[0]) * cos(pi * x[1]) * cos(pi * x[2]) * ct;
    const double e = ph - pe;
    acc += wq[i] * e * e;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[k] = jac[k] * s;
}

// initial_state (solver.py:264-279) on the device: the standing wave of exact_solution at the
// element's nodal points x = sum_v lam[a][v] X_v, then coefficients c = Tmat values (Tmat =
// nodal_to_bernstein's matrix for the Bernstein basis, identity for nodal), float64 arithmetic
template <typename T>
__global__ void __launch_bounds__(kFuncThreads) project_kernel(int64_t K, int Np, const double* __restrict__ Tm,
                                                               const double* __restrict__ lam,
                                                               const double* __restrict__ verts, double tau,
                                                               T* __restrict__ q) {
  extern __shared__ double sv[];   // [4][Np] nodal values
  const int64_t k = blockIdx.x;
  const double* X = verts + k * 12;
  const double pi = 3.14159265358979323846, s3 = 1.7320508075688772;
  const double ct = cos(s3 * pi * tau), amp = sin(s3 * pi * tau) / s3;
  for (int a = threadIdx.x; a < Np; a += blockDim.x) {
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int d = 0; d < 3; ++d) x[d] += lam[a * 4 + v] * X[v * 3 + d];
    const double cx = cos(pi * x[0]), cy = cos(pi * x[1]), cz = cos(pi * x[2]);
    const double sx = sin(pi * x[0]), sy = sin(pi * x[1]), sz = sin(pi * x[2]);
    sv[a] = cx * cy * cz * ct;
    sv[Np + a] = sx * cy * cz * amp;
    sv[2 * Np + a] = cx * sy * cz * amp;
    sv[3 * Np + a] = cx * cy * sz * amp;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * Np; i += blockDim.x) {
    const int F = i / Np, a = i - F * Np;
    double c = 0.0;
    for (int b = 0; b < Np; ++b) c += Tm[(int64_t)a * Np + b] * sv[F * Np + b];
    q[((int64_t)F * K + k) * Np + a] = (T)c;
  }
}

__global__ void __launch_bounds__(kFuncThreads) sum_kernel(int64_t n, const double* __restrict__ partial,
                                                           double* __restrict__ out, int do_sqrt) {
  __shared__ double red[kFuncThreads / 32];
  // fixed assignment of indices to threads and fixed combination order: deterministic
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) *out = do_sqrt ? sqrt(s) : s;
}

template <typename T>
int energy_t(int64_t K, int Np, const void* q, const double* M, const double* coef, double* partial, double* out,
             cudaStream_t s) {
  const size_t sm = (size_t)4 * Np * sizeof(double);
  energy_kernel<T><<<(unsigned)K, kFuncThreads, sm, s>>>(K, Np, static_cast<const T*>(q), M, coef, partial);
  sum_kernel<<<1, kFuncThreads, 0, s>>>(K, partial, out, 0);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "energy kernels");
}

template <typename T>
int error_t(int64_t K, int Np, int nq, const void* q0, const double* ET, const double* wq, const double* lam,
            const double* verts, const double* jac, double ct, double* partial, double* out, cudaStream_t s) {
  const size_t sm = (size_t)Np * sizeof(double);
  error_kernel<T><<<(unsigned)K, kFuncThreads, sm, s>>>(K, Np, nq, static_cast<const T*>(q0), ET, wq, lam, verts,
                                                         jac, ct, partial);
  sum_kernel<<<1, kFuncThreads, 0, s>>>(K, partial, out, 1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "error kernels");
}

template <typename T>
int project_t(int64_t K, int Np, const double* Tm, const double* lam, const double* verts, double tau, void* q,
              cudaStream_t s) {
  project_kernel<T><<<(unsigned)K, kFuncThreads, (size_t)4 * Np * sizeof(double), s>>>(K, Np, Tm, lam, verts, tau,
                                                                                        static_cast<T*>(q));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "projection kernel");
}

}  // namespace
}  // namespace bbdg

using namespace bbdg;

extern "C" {

int bbdg_energy(int dtype, int64_t K, int Np, const void* q, const double* mass, const double* coef,
                double* partial, double* out, void* stream) {
  if (K < 1 || K >= (int64_t(1) << 31) || Np < 1 || !q || !mass || !coef || !partial || !out)
    return set_error(BBDG_ERR_ARG, "bad energy arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == BBDG_F32) return energy_t<float>(K, Np, q, mass, coef, partial, out, s);
  if (dtype == BBDG_F64) return energy_t<double>(K, Np, q, mass, coef, partial, out, s);
  return set_error(BBDG_ERR_ARG, "unknown dtype");
}

int bbdg_error_l2(int dtype, int64_t K, int Np, int nq, const void* q0, const double* eval_t, const double* wq,
                  const double* lam, const double* verts, const double* jac, double tau, double* partial,
                  double* out, void* stream) {
  if (K < 1 || K >= (int64_t(1) << 31) || Np < 1 || nq < 1 || !q0 || !eval_t || !wq || !lam || !verts || !jac ||
      !partial || !out)
    return set_error(BBDG_ERR_ARG, "bad error-functional arguments");
  const double ct = std::cos(std::sqrt(3.0) * 3.14159265358979323846 * tau);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == BBDG_F32) return error_t<float>(K, Np, nq, q0, eval_t, wq, lam, verts, jac, ct, partial, out, s);
  if (dtype == BBDG_F64) return error_t<double>(K, Np, nq, q0, eval_t, wq, lam, verts, jac, ct, partial, out, s);
  return set_error(BBDG_ERR_ARG, "unknown dtype");
}

int bbdg_project_standing_wave(int dtype, int64_t K, int Np, const double* tmat, const double* lam,
                               const double* verts, double tau, void* q, void* stream) {
  if (K < 1 || K >= (int64_t(1) << 31) || Np < 1 || !tmat || !lam || !verts || !q)
    return set_error(BBDG_ERR_ARG, "bad projection arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == BBDG_F32) return project_t<float>(K, Np, tmat, lam, verts, tau, q, s);
  if (dtype == BBDG_F64) return project_t<double>(K, Np, tmat, lam, verts, tau, q, s);
  return set_error(BBDG_ERR_ARG, "unknown dtype");
}

}  // extern "C"
