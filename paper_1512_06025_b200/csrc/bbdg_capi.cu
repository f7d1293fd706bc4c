// C ABI of libbbdg_cuda.so: context lifetime, table uploads, dispatch of the
// tile kernels, the stand-alone LSRK update and the halo packer.
#include <cstdio>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "bbdg_common.cuh"
#include "bbdg_geo.cuh"
#include "bbdg_internal.h"
#include "bbdg_nodal.cuh"
#include "bbdg_opt.cuh"
#include "bbdg_tc.cuh"

namespace bbdg {

static thread_local std::string g_err;

int set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
int set_cuda_error(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return BBDG_ERR_CUDA;
}

static KernelEntry lookup(int dtype, int N, int op, int lift, int basis) {
#define BBDG_SW(tn)                                  \
  switch (N) {                                       \
    case 1: return entry_##tn##_1(op, lift, basis);  \
    case 2: return entry_##tn##_2(op, lift, basis);  \
    case 3: return entry_##tn##_3(op, lift, basis);  \
    case 4: return entry_##tn##_4(op, lift, basis);  \
    case 5: return entry_##tn##_5(op, lift, basis);  \
    case 6: return entry_##tn##_6(op, lift, basis);  \
    case 7: return entry_##tn##_7(op, lift, basis);  \
    case 8: return entry_##tn##_8(op, lift, basis);  \
    case 9: return entry_##tn##_9(op, lift, basis);  \
  }
  if (dtype == BBDG_F32) { BBDG_SW(f32) }
  else { BBDG_SW(f64) }
#undef BBDG_SW
  return KernelEntry{nullptr, nullptr, 0};
}

void free_geometry(bbdg_ctx* c) {
  cudaFree(c->geo_vol);
  cudaFree(c->geo_surf);
  cudaFree(c->geo);
  cudaFree(c->nbr);
  cudaFree(c->code);
  c->geo_vol = c->geo_surf = c->geo = nullptr;
  c->nbr = c->code = nullptr;
}

template <typename T> static void* upload(const std::vector<T>& h, int* rc) {
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, std::max<size_t>(h.size(), 1) * sizeof(T));
  if (e == cudaSuccess && !h.empty()) e = cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    *rc = set_cuda_error(e, "table upload");
    if (d) cudaFree(d);
    return nullptr;
  }
  return d;
}

template <typename T> static std::vector<T> cast(const double* src, size_t n) {
  std::vector<T> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = static_cast<T>(src[i]);
  return v;
}

template <typename T>
static int set_geometry_t(bbdg_ctx* c, const double* rst_dx, const double* kappa, const double* inv_rho,
                          const double* normals, const double* face_scale, const double* tau_p,
                          const double* tau_u, const int32_t* nbr_elem, const int8_t* nbr_code) {
  const int64_t K = c->K;
  std::vector<T> gv((size_t)K * kGeoVol), gs((size_t)K * kGeoSurf), gr((size_t)K * kGeoRec);
  std::vector<int32_t> nb((size_t)K * 4), cd((size_t)K);
  for (int64_t k = 0; k < K; ++k) {
    int code[4];
    for (int f = 0; f < 4; ++f) {
      code[f] = static_cast<uint8_t>(nbr_code[k * 4 + f]);
      const int32_t n = nbr_elem[k * 4 + f];
      const bool halo = (code[f] >> 6) & 1, bnd = (code[f] >> 5) & 1;
      if (!bnd && !halo && (n < 0 || n >= K)) return set_error(BBDG_ERR_ARG, "neighbour element out of range");
    }
    pack_element<T>(rst_dx + k * 9, kappa[k], inv_rho[k], normals + k * 12, face_scale + k * 4, tau_p + k * 4,
                    tau_u + k * 4, nbr_elem + k * 4, code, &gr[k * kGeoRec], &gv[k * kGeoVol], &gs[k * kGeoSurf],
                    &nb[k * 4], &cd[k]);
  }
  int rc = BBDG_OK;
  free_geometry(c);
  c->geo = upload(gr, &rc);
  c->geo_vol = upload(gv, &rc);
  c->geo_surf = upload(gs, &rc);
  c->nbr = static_cast<int32_t*>(upload(nb, &rc));
  c->code = static_cast<int32_t*>(upload(cd, &rc));
  return rc;
}

// ---------------------------------------------------------------------------
// nodal blocked path: operator fragments in mma.sync lane order (bbdg_nodal.cuh)
// ---------------------------------------------------------------------------
// round-to-nearest (ties away) to tf32, as cvt.rna.tf32.f32
static float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// B(k, n) = Mats[m][n * kdim + k] (operator rows n = output node), per (m, k-step, n-tile, lane)
template <typename T>
static std::vector<T> mma_fragments(const double* const* mats, int nm, int Np, int kdim) {
  using MM = NodalMma<T>;
  const int KS = MM::KS, NT = MM::NT, nks = (kdim + KS - 1) / KS, ntl = (Np + NT - 1) / NT;
  const int per = sizeof(T) == 4 ? 4 : 1;
  std::vector<T> out((size_t)nm * nks * ntl * 32 * per, T(0));
  for (int m = 0; m < nm; ++m)
    for (int ks = 0; ks < nks; ++ks)
      for (int nt = 0; nt < ntl; ++nt)
        for (int lane = 0; lane < 32; ++lane) {
          const int g = lane >> 2, t = lane & 3, n = nt * NT + g;
          auto B = [&](int k) { return (n < Np && k < kdim) ? mats[m][(size_t)n * kdim + k] : 0.0; };
          T* o = &out[((((size_t)m * nks + ks) * ntl + nt) * 32 + lane) * per];
          if constexpr (sizeof(T) == 4) {
            const float b0 = (float)B(ks * KS + t), b1 = (float)B(ks * KS + t + 4);
            const float h0 = tf32_rna(b0), h1 = tf32_rna(b1);
            o[0] = h0;
            o[1] = h1;
            o[2] = tf32_rna(b0 - h0);
            o[3] = tf32_rna(b1 - h1);
          } else {
            o[0] = (T)B(ks * KS + t);
          }
        }
  return out;
}

// ---------------------------------------------------------------------------
// stand-alone LSRK update (K8) and halo pack
// ---------------------------------------------------------------------------
template <typename T>
__global__ void lsrk_update_kernel(int64_t n, T* __restrict__ q, T* __restrict__ res, const T* __restrict__ rhs,
                                   T a, T b, T dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T r = res[i] * a;
    r = r + dt * rhs[i];
    res[i] = r;
    q[i] = q[i] + b * r;
  }
}

// vectorised body: 16-byte lanes when all three arrays are aligned
template <typename T, typename V, int W>
__global__ void lsrk_update_vec_kernel(int64_t nv, V* __restrict__ q, V* __restrict__ res,
                                       const V* __restrict__ rhs, T a, T b, T dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    V r = res[i], k = __ldg(rhs + i), x = q[i];
    T* rr = reinterpret_cast<T*>(&r);
    const T* kk = reinterpret_cast<const T*>(&k);
    T* xx = reinterpret_cast<T*>(&x);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      rr[j] = rr[j] * a;
      rr[j] = rr[j] + dt * kk[j];
      xx[j] = xx[j] + b * rr[j];
    }
    res[i] = r;
    q[i] = x;
  }
}

template <typename T>
static int lsrk_update_t(int64_t n, void* q, void* res, const void* rhs, double a, double b, double dt,
                         cudaStream_t s, int num_sms) {
  if (n == 0) return BBDG_OK;
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int W = 16 / sizeof(T);
  const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(res) |
                         reinterpret_cast<uintptr_t>(rhs)) & 15) == 0;
  const int threads = 256;
  if (aligned) {
    const int64_t nv = n / W;
    if (nv) {
      const int64_t grid = std::min<int64_t>((nv + threads - 1) / threads, (int64_t)num_sms * 8);
      lsrk_update_vec_kernel<T, V, W><<<(unsigned)grid, threads, 0, s>>>(
          nv, static_cast<V*>(q), static_cast<V*>(res), static_cast<const V*>(rhs), T(a), T(b), T(dt));
    }
    const int64_t tail = n - nv * W;
    if (tail)
      lsrk_update_kernel<T><<<1, threads, 0, s>>>(tail, static_cast<T*>(q) + nv * W, static_cast<T*>(res) + nv * W,
                                                  static_cast<const T*>(rhs) + nv * W, T(a), T(b), T(dt));
  } else {
    const int64_t grid = std::min<int64_t>((n + threads - 1) / threads, (int64_t)num_sms * 8);
    lsrk_update_kernel<T><<<(unsigned)grid, threads, 0, s>>>(n, static_cast<T*>(q), static_cast<T*>(res),
                                                              static_cast<const T*>(rhs), T(a), T(b), T(dt));
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "lsrk update launch");
}

template <typename T>
__global__ void halo_pack_kernel(int N, int64_t K, int Np, int Nfp, const T* __restrict__ q, T* __restrict__ out,
                                 const int32_t* __restrict__ faces, int64_t n) {
  const int64_t total = n * Nfp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / Nfp;
    const int m = (int)(t % Nfp);
    const int64_t k = faces[2 * i];
    const int f = faces[2 * i + 1];
    int b0 = 0, r = m;
    while (r >= N - b0 + 1) { r -= N - b0 + 1; ++b0; }
    const int b[3] = {b0, r, N - b0 - r};
    int a[4], s = 0;
    for (int v = 0; v < 4; ++v) a[v] = (v == f) ? 0 : b[s++];
    const int pos = pos3(N, a[0], a[1], a[2]);
    for (int F = 0; F < 4; ++F) out[(F * n + i) * Nfp + m] = q[(F * K + k) * Np + pos];
  }
}

static int num_sms_of_current_device() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n;
}

template <typename T> static Params<T> make_params(const bbdg_ctx* c) {
  Params<T> p{};
  p.K = c->K;
  p.kbeg = 0;
  p.kend = c->K;
  p.geo_vol = static_cast<const T*>(c->geo_vol);
  p.geo_surf = static_cast<const T*>(c->geo_surf);
  p.geo = static_cast<const T*>(c->geo);
  p.nbr = c->nbr;
  p.code = c->code;
  p.halo = static_cast<const T*>(c->halo);
  p.nhalo = c->nhalo;
  p.el_vals = static_cast<const T*>(c->el_vals);
  p.el_cols = c->el_cols;
  p.el_w = c->el_w;
  p.liftT = static_cast<const T*>(c->liftT);
  p.dT = static_cast<const T*>(c->dT);
  p.flux = static_cast<T*>(c->flux);
  p.bvol = c->bvol;
  p.blift = c->blift;
  p.img_a = c->img_a;
  p.img_l = c->img_l;
  return p;
}

}  // namespace bbdg

using namespace bbdg;

static int check_ctx(const bbdg_ctx* c) {
  if (!c) return set_error(BBDG_ERR_ARG, "null context");
  if (!c->geo) return set_error(BBDG_ERR_UNSUPPORTED, "geometry not uploaded (bbdg_ctx_set_geometry)");
  return BBDG_OK;
}

// External lift ids (bbdg.h) -> kernel families.  "factorized" is the reference's default lift
// L = E_L L0 (bernstein.py:301-310); like "optimal" (:313-329) it runs as L0 + the one-degree
// reduction sweeps of the fused kernel (E_L is the composition of those sweeps, so the two modes
// differ by rounding only, <= 2.4e-16 in the reference itself).  "ell" keeps the paper's
// non-optimal Alg. 3 kernel that applies E_L as stored ELL rows (tile_kernel, LIFT_FACTORIZED).
static int internal_lift(int ext) {
  switch (ext) {
    case BBDG_LIFT_FACTORIZED: return LIFT_OPTIMAL;
    case BBDG_LIFT_OPTIMAL: return LIFT_OPTIMAL;
    case BBDG_LIFT_DENSE: return LIFT_DENSE;
    case BBDG_LIFT_BLOCKED: return LIFT_BLOCKED;
    case BBDG_LIFT_ELL: return LIFT_FACTORIZED;
  }
  return -1;
}

// validates the external lift id and turns it into the kernel family
static int check_lift(const bbdg_ctx* c, int& lift, bool surf) {
  if (c->basis == BBDG_BASIS_NODAL) {
    if (!c->geo_vol) return set_error(BBDG_ERR_UNSUPPORTED, "nodal kernels need the legacy geometry records");
    // WaveSystem forces "dense" for the nodal basis (solver.py:168-169); BLOCKED selects the
    // tensor-core (EPT) kernels for the same arithmetic
    if (lift == BBDG_LIFT_BLOCKED) {
      if (!c->bvol || !c->blift || (c->dtype == BBDG_F64 && !c->flux))
        return set_error(BBDG_ERR_UNSUPPORTED, "nodal MMA fragments not uploaded (set_nodal_ops + set_lift_tables)");
      lift = LIFT_BLOCKED;
      return BBDG_OK;
    }
    if (lift < 0 || lift > BBDG_LIFT_ELL) return set_error(BBDG_ERR_ARG, "unknown lift mode");
    lift = LIFT_DENSE;
    if (surf && !c->liftT) return set_error(BBDG_ERR_UNSUPPORTED, "nodal dense lift not uploaded");
    if (!c->dT) return set_error(BBDG_ERR_UNSUPPORTED, "nodal derivative matrices not uploaded");
    return BBDG_OK;
  }
  if (lift < 0 || lift > BBDG_LIFT_ELL || lift == BBDG_LIFT_BLOCKED)
    return set_error(BBDG_ERR_ARG, "unknown lift mode (blocked is nodal-only)");
  if (surf && lift == BBDG_LIFT_ELL && !c->el_vals)
    return set_error(BBDG_ERR_UNSUPPORTED, "E_L table not uploaded (bbdg_ctx_set_lift_tables)");
  if (surf && lift == BBDG_LIFT_DENSE && !c->liftT)
    return set_error(BBDG_ERR_UNSUPPORTED, "dense lift not uploaded (bbdg_ctx_set_lift_tables)");
  lift = internal_lift(lift);
  if (surf && lift != LIFT_OPTIMAL && !c->geo_vol)
    return set_error(BBDG_ERR_UNSUPPORTED, "this lift mode needs the legacy geometry records (box context built "
                                           "with the fused record only)");
  return BBDG_OK;
}

// the fused kernels stage field planes with 16-byte TMA bulk copies: the base pointers must be
// 16-byte aligned (every cudaMalloc / torch caching-allocator buffer is)
static int check_aligned(const void* a, const void* b = nullptr, const void* c = nullptr) {
  const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(c);
  return (m & 15) ? set_error(BBDG_ERR_ARG, "state arrays must be 16-byte aligned") : BBDG_OK;
}

static int ensure_scratch(void** ptr, size_t bytes, const char* what) {
  if (*ptr) return BBDG_OK;
  cudaError_t e = cudaMalloc(ptr, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return set_cuda_error(e, what);
  }
  return BBDG_OK;
}

template <typename T>
static int run(bbdg_ctx* c, int op, int lift, Params<T>& p, void* stream, int basis = -1) {
  if (lift == LIFT_BLOCKED && sizeof(T) == 4) {   // tcgen05 operand images (allocated on first use)
    const TcDims d = tc_dims(c->N);
    // zero-filled once: the K padding of the images is never written (the kernels write real entries only)
    if (op != OP_SURFACE && !c->img_a) {
      if (int rc = ensure_scratch(&c->img_a, tc_image_bytes(c->N, c->K, d.KV), "tcgen05 q image")) return rc;
      cudaMemset(c->img_a, 0, tc_image_bytes(c->N, c->K, d.KV));
      cudaDeviceSynchronize();   // one-time: ordered before any stream's use
    }
    if (op != OP_VOLUME && !c->img_l) {
      if (int rc = ensure_scratch(&c->img_l, tc_image_bytes(c->N, c->K, d.KL), "tcgen05 flux image")) return rc;
      cudaMemset(c->img_l, 0, tc_image_bytes(c->N, c->K, d.KL));
      cudaDeviceSynchronize();
    }
    p.img_a = c->img_a;
    p.img_l = c->img_l;
  }
  KernelEntry k = lookup(c->dtype, c->N, op, lift, basis < 0 ? c->basis : basis);
  if (!k.launch) return set_error(BBDG_ERR_UNSUPPORTED, "no kernel for this (op, lift, basis)");
  return k.launch(&p, static_cast<cudaStream_t>(stream), c->num_sms);
}

// res = a res + dt rhs;  q_out = q_in + b res  (the LSRK stage around a precomputed rhs, solver.py:211-213)
template <typename T>
__global__ void stage_update_kernel(int64_t n, const T* __restrict__ q_in, T* __restrict__ q_out, T* __restrict__ res,
                                    const T* __restrict__ rhs, T a, T b, T dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T r = res[i] * a;
    r = r + dt * rhs[i];
    res[i] = r;
    q_out[i] = q_in[i] + b * r;
  }
}

// The Bernstein "dense" lift (bernstein.py:332-347) on the tensor cores: the face fluxes
// (nodal_flux_kernel) times the dense (Np x 4 Nfp) lift as the lift GEMM of the block-partitioned
// kernels (tcgen05 kind::tf32 3xTF32 in fp32, DMMA in fp64; the material-scaled epilogue is
// basis-independent), on top of the Bernstein volume term of the fused kernel.  Whole-mesh calls
// only (ranges keep the node-per-thread tile kernel).  The flux (and, for the stage, an rhs) scratch
// is allocated on the first call.
template <typename T>
static int bb_dense_tc(bbdg_ctx* c, int op, const void* q, void* out, void* res, double a, double b, double dt,
                       int accumulate, void* stream) {
  const size_t sz = sizeof(T);
  if (sz == 8) {   // fp64 DMMA path: flux round trip (fp32 writes the tcgen05 flux image directly)
    if (int rc = ensure_scratch(&c->flux, (size_t)4 * c->K * 4 * c->Nfp * sz, "dense-lift flux scratch")) return rc;
  }
  Params<T> p = make_params<T>(c);
  p.q = static_cast<const T*>(q);
  T* rhs = static_cast<T*>(op == OP_STAGE ? nullptr : out);
  if (op == OP_STAGE) {
    if (int rc = ensure_scratch(&c->rhs_scratch, (size_t)4 * c->K * c->Np * sz, "dense-lift rhs scratch")) return rc;
    rhs = static_cast<T*>(c->rhs_scratch);
  }
  p.out = rhs;
  if (op != OP_SURFACE) {   // volume term first
    p.accumulate = 0;
    if (int rc = run<T>(c, OP_VOLUME, LIFT_OPTIMAL, p, stream)) return rc;
  }
  p.flux = static_cast<T*>(c->flux);
  p.accumulate = op == OP_SURFACE ? accumulate : 1;
  if (int rc = run<T>(c, OP_SURFACE, LIFT_BLOCKED, p, stream, BBDG_BASIS_NODAL)) return rc;
  if (op == OP_STAGE) {
    const int64_t n = (int64_t)4 * c->K * c->Np;
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)c->num_sms * 8);
    if (n > 0)
      stage_update_kernel<T><<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
          n, static_cast<const T*>(q), static_cast<T*>(out), static_cast<T*>(res), rhs, T(a), T(b), T(dt));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "stage update launch");
  }
  return BBDG_OK;
}

// (measured, cube_mesh(26): the GEMM wins from N = 6 -- fp32 N=9 2.19 vs 2.92 ms, N=7 0.96 vs 1.05; below, the
// flux round trip through HBM costs more than the node-per-thread kernel's scalar products)
static bool use_bb_dense_tc(const bbdg_ctx* c, int lift, int64_t k0, int64_t k1) {
  return c->basis == BBDG_BASIS_BERNSTEIN && lift == LIFT_DENSE && c->N >= 6 && c->blift && c->geo_vol && k0 == 0 &&
         k1 == c->K && c->nhalo == 0;
}

extern "C" {

int bbdg_version(void) { return 1; }
int bbdg_max_degree(void) { return kMaxDegree; }
const char* bbdg_last_error(void) { return g_err.c_str(); }

int bbdg_ctx_create(int N, int basis, int dtype, int64_t K, bbdg_ctx** out) {
  if (!out) return set_error(BBDG_ERR_ARG, "null output pointer");
  *out = nullptr;
  if (N < 1 || N > kMaxDegree) return set_error(BBDG_ERR_UNSUPPORTED, "degree outside the compiled range 1..9");
  if (basis != BBDG_BASIS_BERNSTEIN && basis != BBDG_BASIS_NODAL) return set_error(BBDG_ERR_ARG, "unknown basis");
  if (dtype != BBDG_F32 && dtype != BBDG_F64) return set_error(BBDG_ERR_ARG, "unknown dtype");
  if (K < 0 || K >= (int64_t(1) << 31)) return set_error(BBDG_ERR_ARG, "K must lie in [0, 2^31)");
  bbdg_ctx* c = new bbdg_ctx();
  c->N = N;
  c->basis = basis;
  c->dtype = dtype;
  c->K = K;
  c->Np = tet_dim(N);
  c->Nfp = tri_dim(N);
  c->num_sms = num_sms_of_current_device();
  *out = c;
  return BBDG_OK;
}

void bbdg_ctx_destroy(bbdg_ctx* c) {
  if (!c) return;
  free_geometry(c);
  cudaFree(c->el_vals);
  cudaFree(c->el_cols);
  cudaFree(c->liftT);
  cudaFree(c->dT);
  cudaFree(c->bvol);
  cudaFree(c->blift);
  cudaFree(c->flux);
  cudaFree(c->rhs_scratch);
  cudaFree(c->img_a);
  cudaFree(c->img_l);
  cudaFreeHost(c->stage_ring);
  delete c;
}

int bbdg_ctx_set_geometry(bbdg_ctx* c, const double* rst_dx, const double* kappa, const double* inv_rho,
                          const double* normals, const double* face_scale, const double* tau_p,
                          const double* tau_u, const int32_t* nbr_elem, const int8_t* nbr_code) {
  if (!c || !rst_dx || !kappa || !inv_rho || !normals || !face_scale || !tau_p || !tau_u || !nbr_elem || !nbr_code)
    return set_error(BBDG_ERR_ARG, "null argument");
  return c->dtype == BBDG_F32
             ? set_geometry_t<float>(c, rst_dx, kappa, inv_rho, normals, face_scale, tau_p, tau_u, nbr_elem, nbr_code)
             : set_geometry_t<double>(c, rst_dx, kappa, inv_rho, normals, face_scale, tau_p, tau_u, nbr_elem,
                                      nbr_code);
}

int bbdg_ctx_set_lift_tables(bbdg_ctx* c, const int32_t* el_cols, const double* el_vals, int width,
                             const double* dense_L) {
  if (!c) return set_error(BBDG_ERR_ARG, "null context");
  const int Np = c->Np, Nfp = c->Nfp;
  int rc = BBDG_OK;
  if (el_cols && el_vals) {
    if (width < 1 || width > 4 * Nfp) return set_error(BBDG_ERR_ARG, "bad E_L width");
    std::vector<uint16_t> cols((size_t)Np * width);
    for (size_t i = 0; i < cols.size(); ++i) {
      if (el_cols[i] < 0 || el_cols[i] >= 4 * Nfp) return set_error(BBDG_ERR_ARG, "E_L column out of range");
      cols[i] = static_cast<uint16_t>(el_cols[i]);
    }
    cudaFree(c->el_vals);
    cudaFree(c->el_cols);
    c->el_vals = c->dtype == BBDG_F32 ? upload(cast<float>(el_vals, cols.size()), &rc)
                                      : upload(cast<double>(el_vals, cols.size()), &rc);
    c->el_cols = static_cast<uint16_t*>(upload(cols, &rc));
    c->el_w = width;
  }
  if (dense_L) {
    std::vector<double> t((size_t)4 * Nfp * Np);
    for (int a = 0; a < Np; ++a)
      for (int j = 0; j < 4 * Nfp; ++j) t[(size_t)j * Np + a] = dense_L[(size_t)a * 4 * Nfp + j];
    cudaFree(c->liftT);
    c->liftT = c->dtype == BBDG_F32 ? upload(cast<float>(t.data(), t.size()), &rc)
                                    : upload(cast<double>(t.data(), t.size()), &rc);
    {
      // lift GEMM operator of the tensor-core kernels (nodal blocked path, and the BB "dense" mode)
      const double* m[1] = {dense_L};
      cudaFree(c->blift);
      cudaFree(c->flux);
      c->flux = nullptr;
      if (c->dtype == BBDG_F32) {   // tcgen05 operator images (bbdg_tc.cuh)
        std::vector<float> vol, lift;
        tc_operator_images(c->N, nullptr, dense_L, vol, lift, tf32_rna);
        c->blift = upload(lift, &rc);
      } else {
        c->blift = upload(mma_fragments<double>(m, 1, Np, 4 * Nfp), &rc);
      }
      if (c->basis == BBDG_BASIS_NODAL && c->dtype == BBDG_F64) {
        const size_t fb = (size_t)4 * c->K * 4 * Nfp * (c->dtype == BBDG_F32 ? 4 : 8);
        cudaError_t e = cudaMalloc(&c->flux, std::max<size_t>(fb, 16));
        if (e != cudaSuccess) {
          c->flux = nullptr;
          rc = set_cuda_error(e, "nodal flux scratch");
        }
      }
    }
  }
  return rc;
}

int bbdg_ctx_set_nodal_ops(bbdg_ctx* c, const double* Dr, const double* Ds, const double* Dt) {
  if (!c || !Dr || !Ds || !Dt) return set_error(BBDG_ERR_ARG, "null argument");
  const int Np = c->Np;
  std::vector<double> t((size_t)3 * Np * Np);
  const double* D[3] = {Dr, Ds, Dt};
  for (int d = 0; d < 3; ++d)
    for (int a = 0; a < Np; ++a)
      for (int b = 0; b < Np; ++b) t[((size_t)d * Np + b) * Np + a] = D[d][(size_t)a * Np + b];
  int rc = BBDG_OK;
  cudaFree(c->dT);
  c->dT = c->dtype == BBDG_F32 ? upload(cast<float>(t.data(), t.size()), &rc)
                               : upload(cast<double>(t.data(), t.size()), &rc);
  cudaFree(c->bvol);
  if (c->dtype == BBDG_F32) {   // tcgen05 operator images (bbdg_tc.cuh)
    std::vector<float> vol, lift;
    tc_operator_images(c->N, D, nullptr, vol, lift, tf32_rna);
    c->bvol = upload(vol, &rc);
  } else {
    c->bvol = upload(mma_fragments<double>(D, 3, Np, Np), &rc);
  }
  return rc;
}

int bbdg_ctx_set_halo(bbdg_ctx* c, const void* halo, int64_t nhalo) {
  if (!c || nhalo < 0 || (nhalo > 0 && !halo)) return set_error(BBDG_ERR_ARG, "bad halo");
  c->halo = halo;
  c->nhalo = nhalo;
  return BBDG_OK;
}

#define BBDG_DISPATCH(EXPR)                                                 \
  (c->dtype == BBDG_F32 ? [&]() { using T = float; EXPR; }() : [&]() { using T = double; EXPR; }())

int bbdg_volume(bbdg_ctx* c, const void* q, void* rhs, int accumulate, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  if (!q || !rhs) return set_error(BBDG_ERR_ARG, "null state pointer");
  if (q == rhs) return set_error(BBDG_ERR_ARG, "rhs must not alias q");
  if (int rc = check_aligned(q, rhs)) return rc;
  int lift = BBDG_LIFT_OPTIMAL;
  if (int rc = check_lift(c, lift, false)) return rc;
  return BBDG_DISPATCH({
    Params<T> p = make_params<T>(c);
    p.q = static_cast<const T*>(q);
    p.out = static_cast<T*>(rhs);
    p.accumulate = accumulate;
    return run<T>(c, OP_VOLUME, lift, p, stream);
  });
}

int bbdg_surface(bbdg_ctx* c, const void* q, void* rhs, int lift, int accumulate, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  if (!q || !rhs) return set_error(BBDG_ERR_ARG, "null state pointer");
  if (q == rhs) return set_error(BBDG_ERR_ARG, "rhs must not alias q (neighbour traces are read during the call)");
  if (int rc = check_aligned(q, rhs)) return rc;
  if (int rc = check_lift(c, lift, true)) return rc;
  if (use_bb_dense_tc(c, lift, 0, c->K))
    return BBDG_DISPATCH({ return bb_dense_tc<T>(c, OP_SURFACE, q, rhs, nullptr, 0, 0, 0, accumulate, stream); });
  return BBDG_DISPATCH({
    Params<T> p = make_params<T>(c);
    p.q = static_cast<const T*>(q);
    p.out = static_cast<T*>(rhs);
    p.accumulate = accumulate;
    return run<T>(c, OP_SURFACE, lift, p, stream);
  });
}

int bbdg_rhs(bbdg_ctx* c, const void* q, void* rhs, int lift, void* stream) {
  if (!c) return set_error(BBDG_ERR_ARG, "null context");
  return bbdg_rhs_range(c, q, rhs, lift, 0, c->K, stream);
}

int bbdg_rhs_range(bbdg_ctx* c, const void* q, void* rhs, int lift, int64_t k0, int64_t k1, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  if (k0 < 0 || k1 > c->K || k0 > k1) return set_error(BBDG_ERR_ARG, "element range outside [0, K]");
  if (!q || !rhs) return set_error(BBDG_ERR_ARG, "null state pointer");
  if (q == rhs) return set_error(BBDG_ERR_ARG, "rhs must not alias q");
  if (int rc = check_aligned(q, rhs)) return rc;
  if (int rc = check_lift(c, lift, true)) return rc;
  if (use_bb_dense_tc(c, lift, k0, k1))
    return BBDG_DISPATCH({ return bb_dense_tc<T>(c, OP_RHS, q, rhs, nullptr, 0, 0, 0, 0, stream); });
  return BBDG_DISPATCH({
    Params<T> p = make_params<T>(c);
    p.q = static_cast<const T*>(q);
    p.out = static_cast<T*>(rhs);
    p.kbeg = k0;
    p.kend = k1;
    return run<T>(c, OP_RHS, lift, p, stream);
  });
}

int bbdg_lsrk_stage(bbdg_ctx* c, const void* q_in, void* q_out, void* res, int lift, double rk_a, double rk_b,
                    double dt, void* stream) {
  if (!c) return set_error(BBDG_ERR_ARG, "null context");
  return bbdg_lsrk_stage_range(c, q_in, q_out, res, lift, rk_a, rk_b, dt, 0, c->K, stream);
}

int bbdg_lsrk_stage_range(bbdg_ctx* c, const void* q_in, void* q_out, void* res, int lift, double rk_a, double rk_b,
                          double dt, int64_t k0, int64_t k1, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  if (k0 < 0 || k1 > c->K || k0 > k1) return set_error(BBDG_ERR_ARG, "element range outside [0, K]");
  if (!q_in || !q_out || !res) return set_error(BBDG_ERR_ARG, "null state pointer");
  if (q_in == q_out) return set_error(BBDG_ERR_ARG, "q_out must not alias q_in");
  if (!(dt > 0.0)) return set_error(BBDG_ERR_ARG, "dt must be positive");
  if (int rc = check_aligned(q_in, q_out, res)) return rc;
  if (int rc = check_lift(c, lift, true)) return rc;
  if (use_bb_dense_tc(c, lift, k0, k1))
    return BBDG_DISPATCH({ return bb_dense_tc<T>(c, OP_STAGE, q_in, q_out, res, rk_a, rk_b, dt, 0, stream); });
  return BBDG_DISPATCH({
    Params<T> p = make_params<T>(c);
    p.q = static_cast<const T*>(q_in);
    p.out = static_cast<T*>(q_out);
    p.res = static_cast<T*>(res);
    p.rk_a = T(rk_a);
    p.rk_b = T(rk_b);
    p.dt = T(dt);
    p.kbeg = k0;
    p.kend = k1;
    return run<T>(c, OP_STAGE, lift, p, stream);
  });
}

int bbdg_lsrk_update(int dtype, int64_t n, void* q, void* res, const void* rhs, double rk_a, double rk_b, double dt,
                     void* stream) {
  if (n < 0 || (n > 0 && (!q || !res || !rhs))) return set_error(BBDG_ERR_ARG, "bad update arguments");
  if (!(dt > 0.0)) return set_error(BBDG_ERR_ARG, "dt must be positive");
  const int sms = num_sms_of_current_device();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == BBDG_F32) return lsrk_update_t<float>(n, q, res, rhs, rk_a, rk_b, dt, s, sms);
  if (dtype == BBDG_F64) return lsrk_update_t<double>(n, q, res, rhs, rk_a, rk_b, dt, s, sms);
  return set_error(BBDG_ERR_ARG, "unknown dtype");
}

// Carpenter-Kennedy five-stage LSRK4 coefficients (solver.py:25-51)
static const double kRK4A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                                -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
static const double kRK4B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                                1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                                2277821191437.0 / 14882151754819.0};

int bbdg_step(bbdg_ctx* c, void* q, void* q_tmp, void* res, double dt, int lift, void* stream) {
  return bbdg_step2(c, q, q_tmp, nullptr, res, dt, lift, stream);
}

// Five stages.  With a second scratch buffer they run q -> t1 -> t2 -> t1 -> t2 -> q, so the last
// stage writes the caller's q directly; with q_tmp2 == NULL they alternate q <-> q_tmp and one
// device copy moves the result (left in q_tmp by the odd stage count) back into q.
int bbdg_step2(bbdg_ctx* c, void* q, void* q_tmp, void* q_tmp2, void* res, double dt, int lift, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  if (!q || !q_tmp || !res) return set_error(BBDG_ERR_ARG, "null state pointer");
  if (q_tmp2 && (q_tmp2 == q || q_tmp2 == q_tmp || q_tmp2 == res))
    return set_error(BBDG_ERR_ARG, "scratch buffers must be distinct");
  if (!(dt > 0.0)) return set_error(BBDG_ERR_ARG, "dt must be positive");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = (size_t)4 * c->K * c->Np * (c->dtype == BBDG_F32 ? 4 : 8);
  cudaError_t e = cudaMemsetAsync(res, 0, bytes, s);
  if (e != cudaSuccess) return set_cuda_error(e, "res zeroing");
  void* seq[6];
  if (q_tmp2) {
    void* s6[6] = {q, q_tmp, q_tmp2, q_tmp, q_tmp2, q};
    std::memcpy(seq, s6, sizeof(seq));
  } else {
    void* s6[6] = {q, q_tmp, q, q_tmp, q, q_tmp};
    std::memcpy(seq, s6, sizeof(seq));
  }
  for (int st = 0; st < 5; ++st) {
    int rc = bbdg_lsrk_stage(c, seq[st], seq[st + 1], res, lift, kRK4A[st], kRK4B[st], dt, stream);
    if (rc) return rc;
  }
  if (q_tmp2) return BBDG_OK;
  e = cudaMemcpyAsync(q, q_tmp, bytes, cudaMemcpyDeviceToDevice, s);
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "final stage copy");
}

// lsrk4_step on a HOST state: the element range is cut into chunks whose neighbours lie within
// `reach` chunks (banded element numbering, e.g. cube_mesh's x-slabs).  Stage s of chunk i runs in
// slot t = i + reach (s-1), stages ascending within a slot: stage s-1 of chunks i-reach..i+reach
// then precedes it in stream order (the last of them, chunk i+reach, earlier in the same slot) --
// both its reads of q_{s-1} and the last reads of the q_{s-2} values it overwrites (ping-pong).
// Chunk i's H2D (h2d stream) gates stage 1 of chunk i-reach; chunk i's D2H (d2h stream) follows
// its stage 5, so both copy directions overlap the stages of the other chunks.  The result
// (stage 5 writes q_tmp) goes straight to the host array; the stream `stream` is joined with
// both copy streams before return, so work queued after the call sees host_q complete.
int bbdg_step_host(bbdg_ctx* c, void* host_q, void* q, void* q_tmp, void* res, double dt, int lift,
                   const int64_t* bounds, int nchunks, int reach, void* stream, void* h2d_stream, void* d2h_stream) {
  if (int rc = check_ctx(c)) return rc;
  if (!host_q || !q || !q_tmp || !res || !bounds) return set_error(BBDG_ERR_ARG, "null pointer");
  if (!(dt > 0.0)) return set_error(BBDG_ERR_ARG, "dt must be positive");
  if (nchunks < 1 || reach < 0 || bounds[0] != 0 || bounds[nchunks] != c->K)
    return set_error(BBDG_ERR_ARG, "chunk bounds must cover [0, K)");
  for (int i = 0; i < nchunks; ++i)
    if (bounds[i + 1] <= bounds[i]) return set_error(BBDG_ERR_ARG, "chunk bounds must increase");
  if (c->nhalo) return set_error(BBDG_ERR_ARG, "host-pipelined step on a partitioned context");
  cudaStream_t cs = static_cast<cudaStream_t>(stream), hs = static_cast<cudaStream_t>(h2d_stream),
               ds = static_cast<cudaStream_t>(d2h_stream);
  const size_t sz = c->dtype == BBDG_F32 ? 4 : 8, plane = (size_t)c->K * c->Np * sz;
  std::vector<cudaEvent_t> ev(2 * nchunks + 2, nullptr);
  int rc = BBDG_OK;
  auto fail = [&](cudaError_t e, const char* where) {
    rc = set_cuda_error(e, where);
    return rc;
  };
  for (auto& e : ev)
    if (cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) {
      fail(r, "event create");
      break;
    }
  cudaEvent_t* h2d_done = ev.data();
  cudaEvent_t* st5_done = ev.data() + nchunks;
  cudaEvent_t start = ev[2 * nchunks], d2h_all = ev[2 * nchunks + 1];
  auto copy_chunk = [&](char* dst, const char* src, int i, cudaMemcpyKind kind, cudaStream_t s) {
    const size_t off = (size_t)bounds[i] * c->Np * sz, len = (size_t)(bounds[i + 1] - bounds[i]) * c->Np * sz;
    for (int F = 0; F < 4 && rc == BBDG_OK; ++F)
      if (cudaError_t r = cudaMemcpyAsync(dst + F * plane + off, src + F * plane + off, len, kind, s))
        fail(r, "chunk copy");
  };
  // the copy streams start after the work already queued on `stream` (buffers may be in use)
  if (rc == BBDG_OK) {
    if (cudaError_t r = cudaEventRecord(start, cs)) fail(r, "event record");
    else if ((r = cudaStreamWaitEvent(hs, start, 0)) || (r = cudaStreamWaitEvent(ds, start, 0))) fail(r, "wait");
  }
  if (rc == BBDG_OK)
    if (cudaError_t r = cudaMemsetAsync(res, 0, 4 * plane, cs)) fail(r, "res zeroing");
  for (int i = 0; i < nchunks && rc == BBDG_OK; ++i) {
    copy_chunk(static_cast<char*>(q), static_cast<const char*>(host_q), i, cudaMemcpyHostToDevice, hs);
    if (rc == BBDG_OK)
      if (cudaError_t r = cudaEventRecord(h2d_done[i], hs)) fail(r, "event record");
  }
  void* buf[2] = {q, q_tmp};
  const int lag = reach, slots = nchunks + 4 * lag;
  for (int t = 0; t < slots && rc == BBDG_OK; ++t) {
    for (int s = 0; s < 5 && rc == BBDG_OK; ++s) {
      const int i = t - lag * s;
      if (i < 0 || i >= nchunks) continue;
      if (s == 0) {
        const int need = i + reach < nchunks ? i + reach : nchunks - 1;
        if (cudaError_t r = cudaStreamWaitEvent(cs, h2d_done[need], 0)) {
          fail(r, "wait");
          break;
        }
      }
      rc = bbdg_lsrk_stage_range(c, buf[s & 1], buf[(s + 1) & 1], res, lift, kRK4A[s], kRK4B[s], dt, bounds[i],
                                 bounds[i + 1], stream);
      if (rc == BBDG_OK && s == 4) {
        cudaError_t r = cudaEventRecord(st5_done[i], cs);
        if (!r) r = cudaStreamWaitEvent(ds, st5_done[i], 0);
        if (r) fail(r, "event");
        else copy_chunk(static_cast<char*>(host_q), static_cast<const char*>(q_tmp), i, cudaMemcpyDeviceToHost, ds);
      }
    }
  }
  if (rc == BBDG_OK) {
    cudaError_t r = cudaEventRecord(d2h_all, ds);
    if (!r) r = cudaStreamWaitEvent(cs, d2h_all, 0);
    if (r) fail(r, "join");
  }
  for (auto e : ev)
    if (e) cudaEventDestroy(e);   // released once the queued work that uses it completes
  return rc;
}

// Host copies of a pageable state through the pinned staging rings: the byte range of a job
// list split evenly over `nthreads` threads (memcpy of one thread is ~10 GB/s, PCIe ~55).
struct HostCopy {
  char* dst;
  const char* src;
  size_t len;
};
static void parallel_copy(const std::vector<HostCopy>& jobs, int nthreads) {
  size_t total = 0;
  for (const HostCopy& j : jobs) total += j.len;
  auto run = [&jobs](size_t b, size_t e) {
    size_t pos = 0;
    for (const HostCopy& j : jobs) {
      const size_t js = pos, je = pos + j.len;
      pos = je;
      const size_t lo = b > js ? b : js, hi = e < je ? e : je;
      if (lo < hi) std::memcpy(j.dst + (lo - js), j.src + (lo - js), hi - lo);
    }
  };
  if (nthreads <= 1 || total < ((size_t)1 << 22)) {
    run(0, total);
    return;
  }
  const size_t per = ((total + nthreads - 1) / nthreads + 4095) & ~(size_t)4095;
  std::vector<std::thread> pool;
  size_t done = per;   // [0, done) is this thread's; ranges whose thread could not start run here too
  try {
    for (int i = 1; i < nthreads && (size_t)i * per < total; ++i) {
      pool.emplace_back(run, (size_t)i * per, std::min(total, (size_t)(i + 1) * per));
      done = std::min(total, (size_t)(i + 1) * per);
    }
  } catch (...) {   // no more threads (std::system_error): copy the rest on this one
  }
  run(0, std::min(total, per));
  if (done < total) run(done, total);
  for (std::thread& t : pool) t.join();
}

int bbdg_step_pageable(bbdg_ctx* c, void* host_q, void* q, void* q_tmp, void* res, double dt, int lift,
                       const int64_t* bounds, int nchunks, int reach, int slots, int threads, void* stream,
                       void* h2d_stream, void* d2h_stream) {
  if (int rc = check_ctx(c)) return rc;
  if (!host_q || !q || !q_tmp || !res || !bounds) return set_error(BBDG_ERR_ARG, "null pointer");
  if (!(dt > 0.0)) return set_error(BBDG_ERR_ARG, "dt must be positive");
  if (nchunks < 1 || reach < 0 || bounds[0] != 0 || bounds[nchunks] != c->K)
    return set_error(BBDG_ERR_ARG, "chunk bounds must cover [0, K)");
  if (slots < 1 || slots > 16 || threads < 1 || threads > 256) return set_error(BBDG_ERR_ARG, "bad slots / threads");
  int64_t maxlen = 0;
  for (int i = 0; i < nchunks; ++i) {
    if (bounds[i + 1] <= bounds[i]) return set_error(BBDG_ERR_ARG, "chunk bounds must increase");
    maxlen = std::max<int64_t>(maxlen, bounds[i + 1] - bounds[i]);
  }
  if (c->nhalo) return set_error(BBDG_ERR_ARG, "host-pipelined step on a partitioned context");
  cudaStream_t cs = static_cast<cudaStream_t>(stream), hs = static_cast<cudaStream_t>(h2d_stream),
               ds = static_cast<cudaStream_t>(d2h_stream);
  const size_t sz = c->dtype == BBDG_F32 ? 4 : 8, plane = (size_t)c->K * c->Np * sz;
  const size_t slot_bytes = 4 * (size_t)maxlen * c->Np * sz, need = 2 * (size_t)slots * slot_bytes;
  if (c->stage_ring_bytes < need) {
    cudaFreeHost(c->stage_ring);
    c->stage_ring = nullptr;
    c->stage_ring_bytes = 0;
    if (cudaError_t e = cudaHostAlloc(&c->stage_ring, need, cudaHostAllocDefault)) {
      c->stage_ring = nullptr;
      return set_cuda_error(e, "pinned staging ring");
    }
    c->stage_ring_bytes = need;
  }
  char* const in_ring = static_cast<char*>(c->stage_ring);
  char* const out_ring = in_ring + (size_t)slots * slot_bytes;
  char* const hq = static_cast<char*>(host_q);
  auto chunk_off = [&](int i) { return (size_t)bounds[i] * c->Np * sz; };
  auto chunk_len = [&](int i) { return (size_t)(bounds[i + 1] - bounds[i]) * c->Np * sz; };

  std::vector<cudaEvent_t> ev(3 * nchunks + 1, nullptr);
  int rc = BBDG_OK;
  auto fail = [&](cudaError_t e, const char* where) {
    if (rc == BBDG_OK) rc = set_cuda_error(e, where);
    return rc;
  };
  for (auto& e : ev)
    if (cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) {
      fail(r, "event create");
      break;
    }
  cudaEvent_t* h2d_done = ev.data();
  cudaEvent_t* st5_done = ev.data() + nchunks;
  cudaEvent_t* d2h_done = ev.data() + 2 * nchunks;
  cudaEvent_t start = ev[3 * nchunks];
  if (rc == BBDG_OK) {
    if (cudaError_t r = cudaEventRecord(start, cs)) fail(r, "event record");
    else if ((r = cudaStreamWaitEvent(hs, start, 0)) || (r = cudaStreamWaitEvent(ds, start, 0))) fail(r, "wait");
  }
  if (rc == BBDG_OK)
    if (cudaError_t r = cudaMemsetAsync(res, 0, 4 * plane, cs)) fail(r, "res zeroing");

  // drainer: waits for each chunk's D2H into its out slot, then copies the slot into host_q
  std::mutex mu;
  std::condition_variable cv;
  int posted = 0, drained = 0;
  bool stop = false;
  auto drain = [&] {
    for (int i = 0; i < nchunks; ++i) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return posted > i || stop; });
        if (posted <= i) return;
      }
      cudaEventSynchronize(d2h_done[i]);
      const size_t off = chunk_off(i), len = chunk_len(i);
      const char* slot = out_ring + (size_t)(i % slots) * slot_bytes;
      std::vector<HostCopy> jobs;
      for (int F = 0; F < 4; ++F) jobs.push_back({hq + F * plane + off, slot + F * len, len});
      parallel_copy(jobs, threads);
      {
        std::lock_guard<std::mutex> lk(mu);
        drained = i + 1;
      }
      cv.notify_all();
    }
  };
  std::thread drainer;
  try {
    drainer = std::thread(drain);
  } catch (...) {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    return set_error(BBDG_ERR_CUDA, "could not start the staging drainer thread");
  }

  int fed = 0;
  auto feed = [&](int i) {
    const int sl = i % slots;
    if (i >= slots)
      if (cudaError_t r = cudaEventSynchronize(h2d_done[i - slots])) return fail(r, "staging slot wait");
    const size_t off = chunk_off(i), len = chunk_len(i);
    char* slot = in_ring + (size_t)sl * slot_bytes;
    std::vector<HostCopy> jobs;
    for (int F = 0; F < 4; ++F) jobs.push_back({slot + F * len, hq + F * plane + off, len});
    parallel_copy(jobs, threads);
    for (int F = 0; F < 4 && rc == BBDG_OK; ++F)
      if (cudaError_t r = cudaMemcpyAsync(static_cast<char*>(q) + F * plane + off, slot + F * len, len,
                                          cudaMemcpyHostToDevice, hs))
        fail(r, "chunk copy");
    if (rc == BBDG_OK)
      if (cudaError_t r = cudaEventRecord(h2d_done[i], hs)) fail(r, "event record");
    return rc;
  };
  void* buf[2] = {q, q_tmp};
  const int lag = reach, nslot_t = nchunks + 4 * lag;
  for (int t = 0; t < nslot_t && rc == BBDG_OK; ++t) {
    for (int s = 0; s < 5 && rc == BBDG_OK; ++s) {
      const int i = t - lag * s;
      if (i < 0 || i >= nchunks) continue;
      if (s == 0) {
        const int need_i = i + reach < nchunks ? i + reach : nchunks - 1;
        while (fed <= need_i && rc == BBDG_OK) feed(fed++);
        if (rc != BBDG_OK) break;
        if (cudaError_t r = cudaStreamWaitEvent(cs, h2d_done[need_i], 0)) {
          fail(r, "wait");
          break;
        }
      }
      rc = bbdg_lsrk_stage_range(c, buf[s & 1], buf[(s + 1) & 1], res, lift, kRK4A[s], kRK4B[s], dt, bounds[i],
                                 bounds[i + 1], stream);
      if (rc == BBDG_OK && s == 4) {
        cudaError_t r = cudaEventRecord(st5_done[i], cs);
        if (!r) r = cudaStreamWaitEvent(ds, st5_done[i], 0);
        if (r) {
          fail(r, "event");
          break;
        }
        if (i >= slots) {   // the out slot's previous chunk has been copied to host_q
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return drained >= i - slots + 1; });
        }
        const size_t off = chunk_off(i), len = chunk_len(i);
        char* slot = out_ring + (size_t)(i % slots) * slot_bytes;
        for (int F = 0; F < 4 && rc == BBDG_OK; ++F)
          if ((r = cudaMemcpyAsync(slot + F * len, static_cast<const char*>(q_tmp) + F * plane + off, len,
                                   cudaMemcpyDeviceToHost, ds)))
            fail(r, "chunk copy");
        if (rc == BBDG_OK && (r = cudaEventRecord(d2h_done[i], ds))) fail(r, "event record");
        if (rc == BBDG_OK) {
          std::lock_guard<std::mutex> lk(mu);
          posted = i + 1;
        }
        cv.notify_all();
      }
    }
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    stop = true;
  }
  cv.notify_all();
  drainer.join();
  if (rc == BBDG_OK)
    if (cudaError_t r = cudaStreamSynchronize(cs)) fail(r, "step");
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  return rc;
}

int bbdg_halo_pack(bbdg_ctx* c, const void* q, void* sendbuf, const int32_t* faces, int64_t n, void* stream) {
  if (!c || (n > 0 && (!q || !sendbuf || !faces))) return set_error(BBDG_ERR_ARG, "bad halo pack arguments");
  if (n == 0) return BBDG_OK;
  const int threads = 256;
  const int64_t grid = std::min<int64_t>((n * c->Nfp + threads - 1) / threads, (int64_t)c->num_sms * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->dtype == BBDG_F32)
    halo_pack_kernel<float><<<(unsigned)grid, threads, 0, s>>>(c->N, c->K, c->Np, c->Nfp, static_cast<const float*>(q),
                                                               static_cast<float*>(sendbuf), faces, n);
  else
    halo_pack_kernel<double><<<(unsigned)grid, threads, 0, s>>>(c->N, c->K, c->Np, c->Nfp,
                                                                static_cast<const double*>(q),
                                                                static_cast<double*>(sendbuf), faces, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "halo pack launch");
}

int bbdg_tile_elems(int N, int dtype) {
  KernelEntry k = lookup(dtype, N, OP_STAGE, LIFT_OPTIMAL, BASIS_BERNSTEIN);
  return k.launch ? k.tile_elems : -1;
}

int64_t bbdg_kernel_smem(int N, int dtype, int op, int lift, int basis) {
  KernelEntry k = lookup(dtype, N, op, lift, basis);
  return k.smem ? k.smem() : -1;
}

}  // extern "C"
