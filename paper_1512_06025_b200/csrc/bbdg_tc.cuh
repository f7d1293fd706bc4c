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

#include "bbdg_nodal.cuh"
#include "bbdg_opt.cuh"

namespace bbdg {

// tile geometry as a function of the degree (shared by the kernel and the host image builder)
struct TcDims {
  int Np, Nfp, KC, NB, NBLK, KV, KL, NV, SBO, BV_BYTES, BL_BYTES;
};
__host__ __device__ constexpr TcDims tc_dims(int N) {
  const int Np = (N + 1) * (N + 2) * (N + 3) / 6, Nfp = (N + 1) * (N + 2) / 2, KC = 8;
  const int NB = Np <= 16 ? 16 : (Np <= 32 ? 32 : 64);   // output nodes per block
  return TcDims{Np, Nfp, KC, NB, (Np + NB - 1) / NB, (Np + KC - 1) / KC, (4 * Nfp + KC - 1) / KC, 3 * NB,
                (KC / 4) * 128, 3 * NB * KC * 4, NB * KC * 4};
}

template <int N> struct TcLayout {
  static constexpr TcDims d = tc_dims(N);
  static constexpr int Np = d.Np, Nfp = d.Nfp;
  static constexpr int MT = 2;                  // 128-row sub-tiles sharing each operator chunk
  static constexpr int KE = 32;                 // elements per sub-tile -> 128 rows
  static constexpr int M = 128;
  static constexpr int KC = d.KC;               // K per stage chunk (KC / 8 MMA k-steps)
  static constexpr int NB = d.NB, NBLK = d.NBLK;
  static constexpr int KV = d.KV, KL = d.KL;    // volume / lift K chunks
  static constexpr int NV = d.NV;               // volume MMA N
  static constexpr int SBO = d.SBO;             // bytes between 8-row groups
  static constexpr int A_BYTES = M * KC * 4;    // one sub-tile, one of hi / lo
  static constexpr int BV_BYTES = d.BV_BYTES;   // volume B chunk (hi or lo)
  static constexpr int BL_BYTES = d.BL_BYTES;
  static constexpr int B_BYTES = BV_BYTES > BL_BYTES ? BV_BYTES : BL_BYTES;
  static constexpr int RAW_LD = KC + 4;         // padded fp32 row of the raw element chunk
  static constexpr int B_OFF = MT * 2 * A_BYTES, RAW_OFF = B_OFF + 2 * B_BYTES;
  static constexpr int STAGE = RAW_OFF + MT * M * RAW_LD * 4;
  static constexpr int NS = (227 * 1024 - 128) / STAGE < 6 ? (227 * 1024 - 128) / STAGE : 6;   // pipeline depth
  static constexpr int total = NS * STAGE + 128;                      // + mbarriers + TMEM slot
  static constexpr int threads = 512;          // 16 warps: 4 per TMEM lane quarter in the epilogue
  static constexpr int ACC = NV + NB;           // accumulator columns of one sub-tile
  static constexpr int TM_COLS = MT * ACC <= 128 ? 128 : (MT * ACC <= 256 ? 256 : 512);
  static_assert(MT * ACC <= 512, "accumulators exceed the TMEM columns");
  static_assert(total <= 227 * 1024, "tcgen05 nodal tile does not fit in shared memory");
};

// wait until at most `newer` cp.async groups are still pending (wait_group needs an immediate)
__device__ __forceinline__ void cp_async_wait_newer(int newer) {
  switch (newer) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
  }
}

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
__global__ void __launch_bounds__(TcLayout<N>::threads, 1) nodal_tc_kernel(const Params<float> p) {
  using L = TcLayout<N>;
  constexpr int Np = L::Np, Nfp = L::Nfp, KC = L::KC, NB = L::NB, NV = L::NV, MT = L::MT, NS = L::NS;
  constexpr bool VOL = OP != OP_SURFACE, SURF = OP != OP_VOLUME;
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NS * L::STAGE);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + NS * L::STAGE + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(bars + i, 1);
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

  const int64_t fs = p.K * Np, nl = p.kend - p.kbeg;
  constexpr int ST = MT * L::KE;                 // elements per CTA step (MT sub-tiles)
  const int64_t nsteps = (nl + ST - 1) / ST;
  const float* bvh = static_cast<const float*>(p.bvol);                    // [blk][kc] chunks, hi then lo
  const float* blh = static_cast<const float*>(p.blift);
  constexpr int nchunk = (VOL ? L::KV : 0) + (SURF ? L::KL : 0);
  constexpr int per_step = L::NBLK * nchunk;
  const int64_t my_steps = blockIdx.x < nsteps ? (nsteps - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int nC = (int)(my_steps * per_step);   // this CTA's chunk sequence (step, node block, K chunk)
  struct Chunk {
    int64_t kt;   // first element of the step
    int blk, ci, kc;
    bool isvol;
  };
  auto decode = [&](int c) {   // 32-bit index math: divisions by compile-time constants
    Chunk ch;
    const int t = c / per_step;
    const int r = c - t * per_step;
    ch.blk = r / nchunk;
    ch.ci = r - ch.blk * nchunk;
    ch.kt = p.kbeg + ((int64_t)blockIdx.x + (int64_t)t * gridDim.x) * ST;
    ch.isvol = VOL && ch.ci < (VOL ? L::KV : 0);
    ch.kc = ch.isvol ? ch.ci : ch.ci - (VOL ? L::KV : 0);
    return ch;
  };
  auto stage_ptr = [&](int st) { return sm + st * L::STAGE; };
  // cp.async prefetch of a chunk: the element rows of both sub-tiles (fp32, zero-filled outside the
  // mesh / K range) into the raw buffer, the operator image (hi, lo) straight into place
  auto prefetch = [&](int c) {
    const Chunk ch = decode(c);
    unsigned char* sb = stage_ptr(c % NS);
    const uint32_t raw = smem_u32(sb + L::RAW_OFF);
    const int kmax = ch.isvol ? Np : 4 * Nfp;
    if (!ch.isvol || Np % 4 == 0) {
      // 16-byte rows (every flux row, and the state rows when Np = 0 mod 4): one cp.async per
      // 4 values, the tail of a row zero-filled by the source size
      for (int i = tid; i < MT * L::M * (KC / 4); i += L::threads) {
        const int row = i / (KC / 4), k = (i - row * (KC / 4)) * 4, e = row >> 2, F = row & 3, kk = ch.kc * KC + k;
        const int64_t ke = ch.kt + e;
        const int nval = (ke < p.kend) ? (kmax - kk < 4 ? (kmax - kk > 0 ? kmax - kk : 0) : 4) : 0;
        const float* src = nval == 0 ? p.q
                           : ch.isvol ? p.q + F * fs + ke * Np + kk : p.flux + (F * nl + (ke - p.kbeg)) * 4 * Nfp + kk;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(raw + (row * L::RAW_LD + k) * 4),
                     "l"(src), "r"(4 * nval)
                     : "memory");
      }
    } else {
      for (int i = tid; i < MT * L::M * KC; i += L::threads) {
        const int row = i / KC, k = i - row * KC, e = row >> 2, F = row & 3, kk = ch.kc * KC + k;
        const int64_t ke = ch.kt + e;
        const bool ok = ke < p.kend && kk < kmax;
        stage_cp<float>(raw + (row * L::RAW_LD + k) * 4, ok ? p.q + F * fs + ke * Np + kk : p.q, ok);
      }
    }
    const int bytes = ch.isvol ? L::BV_BYTES : L::BL_BYTES;
    const int nch = ch.isvol ? L::KV : L::KL;
    const float* src = (ch.isvol ? bvh : blh) + ((int64_t)(ch.blk * nch + ch.kc) * 2) * (bytes / 4);
    const uint32_t bh = smem_u32(sb + L::B_OFF), bl = bh + L::B_BYTES;
    for (int i = tid; i < 2 * bytes / 16; i += L::threads)
      cp_async<16>(i < bytes / 16 ? bh + i * 16 : bl + (i - bytes / 16) * 16, src + 4 * i);
    cp_async_commit();
  };

  // prefetch distance NS - 2: the stage a prefetch overwrites was read by the MMAs of two chunks
  // back, which have long completed -- the MMAs of the previous chunk keep running meanwhile
  static_assert(NS >= 3, "pipeline needs three stages");
  for (int c = 0; c < NS - 2 && c < nC; ++c) prefetch(c);
  for (int c = 0; c < nC; ++c) {
    const Chunk ch = decode(c);
    const int st = c % NS;
    unsigned char* sbase = stage_ptr(st);
    const float* araw = reinterpret_cast<const float*>(sbase + L::RAW_OFF);
    // this chunk's copies landed (the newer prefetches may stay in flight)
    {
      // groups committed after chunk c's: min(NS - 2, nC - 1 - c)
      const int newer = (nC - 1 - c) < NS - 3 ? (nC - 1 - c) : NS - 3;
      cp_async_wait_newer(newer);
    }
    __syncthreads();
    // ---- split the element rows into tf32 hi / lo in the UMMA layout (consecutive threads:
    // consecutive 16-byte rows of a core matrix; raw rows padded -> both sides conflict-free)
    for (int u = tid; u < MT * L::M * (KC / 4); u += L::threads) {
      const int row = (u / (8 * (KC / 4))) * 8 + (u & 7), kq = ((u >> 3) % (KC / 4)) * 4;
      const float4 x4 = *reinterpret_cast<const float4*>(araw + row * L::RAW_LD + kq);
      const float x[4] = {x4.x, x4.y, x4.z, x4.w};
      uint4 hi, lo;
      uint32_t* h = &hi.x;
      uint32_t* l = &lo.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h[j] = tf32_bits(x[j]);
        l[j] = tf32_bits(x[j] - __uint_as_float(h[j]));
      }
      const int t = row >> 7, off = t * 2 * L::A_BYTES + umma_off(L::SBO, row & 127, kq);
      *reinterpret_cast<uint4*>(sbase + off) = hi;
      *reinterpret_cast<uint4*>(sbase + off + L::A_BYTES) = lo;
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t bh = smem_u32(sbase + L::B_OFF), bl = bh + L::B_BYTES;
      const uint32_t idesc = ch.isvol ? umma_idesc_tf32(128, NV) : umma_idesc_tf32(128, NB);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const uint32_t ah = smem_u32(sbase + t * 2 * L::A_BYTES), al = ah + L::A_BYTES;
        const uint32_t d = tmem + t * L::ACC + (ch.isvol ? 0 : NV);
#pragma unroll
        for (int ks = 0; ks < KC / 8; ++ks) {
          const uint32_t ko = ks * 256;   // two 16-byte K units per k-step
          const uint64_t dah = umma_desc(ah + ko, 128, L::SBO), dal = umma_desc(al + ko, 128, L::SBO);
          const uint64_t dbh = umma_desc(bh + ko, 128, L::SBO), dbl = umma_desc(bl + ko, 128, L::SBO);
          umma_tf32(d, dal, dbh, idesc, (ch.kc | ks) != 0);
          umma_tf32(d, dah, dbl, idesc, 1);
          umma_tf32(d, dah, dbh, idesc, 1);
        }
      }
      umma_commit(bars + st);
    }
    if (c + NS - 2 < nC) {
      // the stage of chunk c + NS - 2 was last read by chunk c - 2's MMAs
      if (c >= 2) mbar_wait(bars + (c - 2) % NS, (uint32_t)(((c - 2) / NS) & 1));
      prefetch(c + NS - 2);
    }
    if (ch.ci == nchunk - 1) {
      // ---- epilogue of this node block: all accumulators complete
      mbar_wait(bars + st, (uint32_t)((c / NS) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int wq = warp & 3, half = warp >> 2;   // TMEM lane quarter, column quarter
      const int row = wq * 32 + lane, F = row & 3, base = lane & ~3;
      const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
#pragma unroll 1
      for (int t = 0; t < MT; ++t) {
        const int64_t k = ch.kt + t * L::KE + (row >> 2);
        const bool okr = k < p.kend;
        const float* gv = p.geo_vol + (okr ? k : ch.kt) * kGeoVol;
        float G[9];
#pragma unroll
        for (int j = 0; j < 9; ++j) G[j] = gv[j];
        const float kap = gv[9], irho = gv[10];
        const uint32_t tv = tmem + t * L::ACC + lane_off, tl = tv + NV;
#pragma unroll 1
        for (int a0 = 16 * half; a0 < NB; a0 += 16 * (L::threads / 128)) {
          uint32_t gr[16], gs[16], gt[16], li[16];
          if constexpr (VOL) {
            tm_ld<16>(tv + a0, gr);
            tm_ld<16>(tv + NB + a0, gs);
            tm_ld<16>(tv + 2 * NB + a0, gt);
          }
          if constexpr (SURF) tm_ld<16>(tl + a0, li);
          tm_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int a = ch.blk * NB + a0 + j;
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
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncthreads();   // accumulators read: the next block's MMAs may overwrite them
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
