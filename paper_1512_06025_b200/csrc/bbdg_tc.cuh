// Block-partitioned nodal DG on the 5th-generation tensor cores (tcgen05.mma kind::tf32, TMEM
// accumulators) -- the fp32 comparison path the paper measures BB against ("EPT" nodal,
// SURVEY K6/K7; reference nodal.py:220-241 through WaveSystem, solver.py:139-190).  fp64 keeps
// the DMMA kernel of bbdg_nodal.cuh (tcgen05 has no f64 kind).
//
// A CTA tile is 32 elements x 4 fields = 128 GEMM rows (row 4e + F: the four fields of an element
// sit in adjacent TMEM lanes of one warp).  Per block of NB output nodes:
//   volume  C_v[row][(m, a)] = sum_b Q[row][b] D_m[a][b]      (N = 3 NB, K = Np)
//   lift    C_l[row][a]      = sum_c X[row][c] L[a][c]        (N = NB,   K = 4 Nfp)
// with X = (Fp, n1 Fu, n2 Fu, n3 Fu) from nodal_flux_kernel.  fp32 accuracy from 3xTF32: every
// k-step issues lo*hi + hi*lo + hi*hi (x = hi + lo split at tf32 precision, cvt.rna), so the
// products carry ~fp32 precision (TF32 alone: ~5e-4, SURVEY 7 "hard part 5").
//
// Operands stream through two shared-memory stages in the canonical no-swizzle K-major UMMA
// layout (8-row x 16-byte core matrices; LBO = 128 B between K-adjacent core matrices, SBO =
// KC/4 x 128 B between row groups).  The operator chunks are pre-arranged on the host in exactly
// that image (hi and lo), so they are plain 16-byte copies; the element tiles are split into
// hi / lo while being stored.  One elected thread issues the MMAs and commits them to an
// mbarrier per stage, so the loads of chunk c+1 overlap the MMAs of chunk c.  The epilogue reads
// the accumulators with tcgen05.ld (lane = row), combines the 3 derivative columns of the four
// field lanes of an element with warp shuffles (chain rule, solver.py:148-157), adds the material-
// scaled lift (solver.py:182-189) and writes the rhs or the LSRK stage (solver.py:211-213).
#pragma once
#include <vector>

#include "bbdg_opt.cuh"

namespace bbdg {

// tile geometry as a function of the degree (shared by the kernel and the host image builder)
struct TcDims {
  int Np, Nfp, KC, NB, NBLK, KV, KL, NV, SBO, BV_BYTES, BL_BYTES;
};
__host__ __device__ constexpr TcDims tc_dims(int N) {
  const int Np = (N + 1) * (N + 2) * (N + 3) / 6, Nfp = (N + 1) * (N + 2) / 2, KC = 32;
  const int NB = Np <= 16 ? 16 : (Np <= 32 ? 32 : 64);   // output nodes per block
  return TcDims{Np, Nfp, KC, NB, (Np + NB - 1) / NB, (Np + KC - 1) / KC, (4 * Nfp + KC - 1) / KC, 3 * NB,
                (KC / 4) * 128, 3 * NB * KC * 4, NB * KC * 4};
}

template <int N> struct TcLayout {
  static constexpr TcDims d = tc_dims(N);
  static constexpr int Np = d.Np, Nfp = d.Nfp;
  static constexpr int KE = 32;                 // elements per tile -> 128 rows
  static constexpr int M = 128;
  static constexpr int KC = d.KC;               // K per stage chunk (4 MMA k-steps of 8)
  static constexpr int NB = d.NB, NBLK = d.NBLK;
  static constexpr int KV = d.KV, KL = d.KL;    // volume / lift K chunks
  static constexpr int NV = d.NV;               // volume MMA N
  static constexpr int SBO = d.SBO;             // bytes between 8-row groups
  static constexpr int A_BYTES = M * KC * 4;    // one of hi / lo
  static constexpr int BV_BYTES = d.BV_BYTES;   // volume B chunk (hi or lo)
  static constexpr int BL_BYTES = d.BL_BYTES;
  static constexpr int B_BYTES = BV_BYTES > BL_BYTES ? BV_BYTES : BL_BYTES;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int total = 2 * STAGE + 64;          // + 2 mbarriers + TMEM slot
  static constexpr int threads = 128;
  static constexpr int TM_COLS = NV + NB <= 128 ? 128 : 256;   // power of two >= 32
  static_assert(NV + NB <= 256, "accumulators exceed the TMEM columns");
  static_assert(total <= 227 * 1024, "tcgen05 nodal tile does not fit in shared memory");
};

// byte offset of element (row, k) (k in the chunk) in the canonical no-swizzle K-major layout
__host__ __device__ constexpr int umma_off(int sbo, int row, int k) {
  return (row & 7) * 16 + (row >> 3) * sbo + (k >> 2) * 128 + (k & 3) * 4;
}

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// shared-memory matrix descriptor: no swizzle, K-major (PTX "tcgen05 shared memory descriptor",
// cute::UMMA::SmemDescriptor): start >> 4, LBO >> 4 at bit 16, SBO >> 4 at bit 32, version 1 at 46
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// instruction descriptor kind::tf32: F32 accumulator, TF32 A and B, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

template <int N, int OP>
__global__ void __launch_bounds__(128, 1) nodal_tc_kernel(const Params<float> p) {
  using L = TcLayout<N>;
  constexpr int Np = L::Np, Nfp = L::Nfp, KC = L::KC, NB = L::NB, NV = L::NV;
  constexpr bool VOL = OP != OP_SURFACE, SURF = OP != OP_VOLUME;
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * L::STAGE);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + 2 * L::STAGE + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tm_slot)),
                 "n"(L::TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tm_slot;
  const uint32_t tm_vol = tmem, tm_lift = tmem + NV;   // column offsets (lane 0)

  const int64_t fs = p.K * Np, nl = p.kend - p.kbeg;
  const int64_t ntiles = (nl + L::KE - 1) / L::KE;
  const float* bvh = static_cast<const float*>(p.bvol);                    // [blk][kc] chunks, hi then lo
  const float* blh = static_cast<const float*>(p.blift);
  constexpr int nchunk = (VOL ? L::KV : 0) + (SURF ? L::KL : 0);
  uint32_t c = 0;   // global chunk counter (stage = c & 1, its mbarrier phase = (c >> 1) & 1)

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t kt = p.kbeg + tile * L::KE;
    const int nv = (int)((p.kend - kt) < L::KE ? (p.kend - kt) : L::KE);
    for (int blk = 0; blk < L::NBLK; ++blk) {
      for (int ci = 0; ci < nchunk; ++ci, ++c) {
        const bool isvol = VOL && ci < (VOL ? L::KV : 0);
        const int kc = isvol ? ci : ci - (VOL ? L::KV : 0);
        const int st = c & 1;
        unsigned char* sbase = sm + st * L::STAGE;
        unsigned char* sa_hi = sbase;
        unsigned char* sa_lo = sbase + L::A_BYTES;
        unsigned char* sb_hi = sbase + 2 * L::A_BYTES;
        unsigned char* sb_lo = sb_hi + L::B_BYTES;
        if (c >= 2) mbar_wait(bars + st, ((c >> 1) - 1) & 1);   // the MMAs of chunk c-2 released this stage
        // ---- A chunk: 128 rows (4e + F) x KC, split into tf32 hi / lo in the UMMA layout
        const int kmax = isvol ? Np : 4 * Nfp;
        for (int u = tid; u < L::M * (KC / 4); u += 128) {
          const int row = u / (KC / 4), kq = (u - row * (KC / 4)) * 4;
          const int e = row >> 2, F = row & 3;
          float x[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = kc * KC + kq + j;
            x[j] = 0.f;
            if (e < nv && k < kmax)
              x[j] = isvol ? p.q[F * fs + (kt + e) * Np + k] : p.flux[(F * nl + (kt - p.kbeg + e)) * 4 * Nfp + k];
          }
          uint4 hi, lo;
          uint32_t* h = &hi.x;
          uint32_t* l = &lo.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            h[j] = tf32_bits(x[j]);
            l[j] = tf32_bits(x[j] - __uint_as_float(h[j]));
          }
          const int off = umma_off(L::SBO, row, kq);
          *reinterpret_cast<uint4*>(sa_hi + off) = hi;
          *reinterpret_cast<uint4*>(sa_lo + off) = lo;
        }
        // ---- B chunk: pre-arranged image (hi, lo), plain 16-byte copies
        {
          const int bytes = isvol ? L::BV_BYTES : L::BL_BYTES;
          const int nch = isvol ? L::KV : L::KL;
          const float* src = (isvol ? bvh : blh) + ((int64_t)(blk * nch + kc) * 2) * (bytes / 4);
          const uint4* s4 = reinterpret_cast<const uint4*>(src);
          for (int i = tid; i < 2 * bytes / 16; i += 128) {
            const uint4 v = __ldg(s4 + i);
            if (i < bytes / 16) reinterpret_cast<uint4*>(sb_hi)[i] = v;
            else reinterpret_cast<uint4*>(sb_lo)[i - bytes / 16] = v;
          }
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t ah = smem_u32(sa_hi), al = smem_u32(sa_lo), bh = smem_u32(sb_hi), bl = smem_u32(sb_lo);
          const uint32_t nrows = isvol ? NV : NB;
          const uint32_t idesc = isvol ? umma_idesc_tf32(128, NV) : umma_idesc_tf32(128, NB);
          const uint32_t d = isvol ? tm_vol : tm_lift;
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint32_t ko = ks * 256;   // two 16-byte K units per k-step
            const uint64_t dah = umma_desc(ah + ko, 128, L::SBO), dal = umma_desc(al + ko, 128, L::SBO);
            const uint64_t dbh = umma_desc(bh + ko, 128, L::SBO), dbl = umma_desc(bl + ko, 128, L::SBO);
            (void)nrows;
            umma_tf32(d, dal, dbh, idesc, (kc | ks) != 0);
            umma_tf32(d, dah, dbl, idesc, 1);
            umma_tf32(d, dah, dbh, idesc, 1);
          }
          umma_commit(bars + st);
        }
        if (ci == nchunk - 1) {
          // ---- epilogue of this node block: all accumulators complete
          mbar_wait(bars + st, (c >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const int row = warp * 32 + lane, e = row >> 2, F = row & 3, base = lane & ~3;
          const int64_t k = kt + e;
          const bool okr = e < nv;
          const float* gv = p.geo_vol + (okr ? k : kt) * kGeoVol;
          float G[9];
#pragma unroll
          for (int j = 0; j < 9; ++j) G[j] = gv[j];
          const float kap = gv[9], irho = gv[10];
          const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
#pragma unroll 1
          for (int a0 = 0; a0 < NB; a0 += 16) {
            uint32_t gr[16], gs[16], gt[16], li[16];
            if constexpr (VOL) {
              tm_ld<16>(tm_vol + lane_off + a0, gr);
              tm_ld<16>(tm_vol + lane_off + NB + a0, gs);
              tm_ld<16>(tm_vol + lane_off + 2 * NB + a0, gt);
            }
            if constexpr (SURF) tm_ld<16>(tm_lift + lane_off + a0, li);
            tm_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int a = blk * NB + a0 + j;
              float r = 0.f;
              if constexpr (VOL) {
                const float g0 = __uint_as_float(gr[j]), g1 = __uint_as_float(gs[j]), g2 = __uint_as_float(gt[j]);
                // the p row's derivatives (lane base) and the u rows' (base + 1..3) of this element
                const float p0 = __shfl_sync(0xffffffffu, g0, base), p1 = __shfl_sync(0xffffffffu, g1, base),
                            p2 = __shfl_sync(0xffffffffu, g2, base);
                float div = 0.f;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                  const float u0 = __shfl_sync(0xffffffffu, g0, base + 1 + i);
                  const float u1 = __shfl_sync(0xffffffffu, g1, base + 1 + i);
                  const float u2 = __shfl_sync(0xffffffffu, g2, base + 1 + i);
                  div += G[i] * u0 + G[3 + i] * u1 + G[6 + i] * u2;
                }
                if (F == 0) {
                  r = -kap * div;
                } else {
                  const int i = F - 1;
                  r = -irho * (G[i] * p0 + G[3 + i] * p1 + G[6 + i] * p2);
                }
              }
              if constexpr (SURF) {
                const float s = (F == 0 ? kap : irho) * __uint_as_float(li[j]);
                r = VOL ? r + s : s;
              }
              if (okr && a < Np) {
                const int64_t o = F * fs + k * Np + a;
                if constexpr (OP == OP_STAGE) {
                  float x = p.res[o] * p.rk_a;
                  x = x + p.dt * r;
                  p.res[o] = x;
                  p.out[o] = p.q[o] + p.rk_b * x;
                } else {
                  if (p.accumulate) p.out[o] += r;
                  else p.out[o] = r;
                }
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncthreads();   // accumulators read: the next block's MMAs may overwrite them
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(L::TM_COLS));
}

// Host-side image of the operator chunks for nodal_tc_kernel: for each node block and K chunk, the
// (rows x KC) B tile in the UMMA no-swizzle K-major layout, tf32 hi then lo.  Volume rows are
// (m, a) = m NB + a_local with B[(m,a)][b] = D_m[a][b]; lift rows a_local with B[a][c] = L[a][c].
inline void tc_operator_images(int N, const double* const* D, const double* Lmat, std::vector<float>& vol,
                               std::vector<float>& lift, float (*tf32)(float)) {
  const TcDims d = tc_dims(N);
  const int Np = d.Np, Nfp = d.Nfp, KC = d.KC, NB = d.NB;
  vol.assign((size_t)d.NBLK * d.KV * 2 * (d.BV_BYTES / 4), 0.f);
  lift.assign((size_t)d.NBLK * d.KL * 2 * (d.BL_BYTES / 4), 0.f);
  for (int blk = 0; blk < d.NBLK; ++blk) {
    for (int kc = 0; kc < d.KV && D; ++kc) {
      float* hi = &vol[((size_t)(blk * d.KV + kc) * 2) * (d.BV_BYTES / 4)];
      float* lo = hi + d.BV_BYTES / 4;
      for (int m = 0; m < 3; ++m)
        for (int al = 0; al < NB; ++al)
          for (int kk = 0; kk < KC; ++kk) {
            const int a = blk * NB + al, b = kc * KC + kk;
            const float v = (a < Np && b < Np) ? (float)D[m][(size_t)a * Np + b] : 0.f;
            const float h = tf32(v);
            const int o = umma_off(d.SBO, m * NB + al, kk) / 4;
            hi[o] = h;
            lo[o] = tf32(v - h);
          }
    }
    for (int kc = 0; kc < d.KL && Lmat; ++kc) {
      float* hi = &lift[((size_t)(blk * d.KL + kc) * 2) * (d.BL_BYTES / 4)];
      float* lo = hi + d.BL_BYTES / 4;
      for (int al = 0; al < NB; ++al)
        for (int kk = 0; kk < KC; ++kk) {
          const int a = blk * NB + al, cc = kc * KC + kk;
          const float v = (a < Np && cc < 4 * Nfp) ? (float)Lmat[(size_t)a * 4 * Nfp + cc] : 0.f;
          const float h = tf32(v);
          const int o = umma_off(d.SBO, al, kk) / 4;
          hi[o] = h;
          lo[o] = tf32(v - h);
        }
    }
  }
}

}  // namespace bbdg
