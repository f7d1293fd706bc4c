// Block-partitioned nodal DG on the 5th-generation tensor cores (tcgen05.mma kind::tf32, TMEM
// accumulators) -- the fp32 comparison path the paper measures BB against ("EPT" nodal,
// SURVEY K6/K7; reference nodal.py:220-241 through WaveSystem, solver.py:139-190).  fp64 keeps
// the DMMA kernel of bbdg_nodal.cuh (tcgen05 has no f64 kind).
//
// A 128-row sub-tile is 32 elements x 4 fields (row 4e + F: the four fields of an element sit in
// adjacent TMEM lanes of one warp).  Per block of NB output nodes:
//   volume  C_v[row][(m, a)] = sum_b Q[row][b] D_m[a][b]      (N = 3 NB, K = Np)
//   lift    C_l[row][a]      = sum_c X[row][c] L[a][c]        (N = NB,   K = 4 Nfp)
// with X = (Fp, n1 Fu, n2 Fu, n3 Fu), the face fluxes.  fp32 accuracy from 3xTF32: every k-step
// issues lo*hi + hi*lo + hi*hi (x = hi + lo split at tf32 precision, cvt.rna), so the products
// carry ~fp32 precision (TF32 alone: ~5e-4, SURVEY 7 "hard part 5").
//
// All operands are tf32 hi / lo images in the canonical no-swizzle K-major UMMA layout (8-row x
// 16-byte core matrices; LBO = 128 B between K-adjacent core matrices, SBO = KC/4 x 128 B between
// row groups): the operator chunks built once on the host (tc_operator_images), the element rows
// by tc_pack_kernel (q) and tc_flux_kernel (fluxes computed straight into the image) before the
// GEMM.  nodal_tc_kernel is warp-specialised: a producer warp streams (element chunk, operator
// chunk) pairs into NS stages with cp.async.bulk, one thread of the MMA warp issues the MMAs and
// commits each stage back to the producer and each finished node block to the epilogue, and four
// epilogue warps read the double-buffered accumulators with tcgen05.ld (lane = row), combine the
// 3 derivative columns of the element's four field lanes with shuffles (chain rule,
// solver.py:148-157), add the material-scaled lift (solver.py:182-189) and write the rhs or the
// LSRK stage (solver.py:211-213).
#pragma once
#include <vector>

#include "bbdg_nodal.cuh"
#include "bbdg_opt.cuh"

#ifndef BBDG_TC_KC
#define BBDG_TC_KC 0   // K per pipeline stage (multiple of 8); 0 = per order (8 up to N = 3, else 16)
#endif

namespace bbdg {

// tile geometry as a function of the degree (shared by the kernels and the host image builder)
struct TcDims {
  int Np, Nfp, KC, NB, NBLK, KV, KL, NV, SBO, BV_BYTES, BL_BYTES, MT;
};
__host__ __device__ constexpr TcDims tc_dims(int N) {
  // K per stage: 8 at N <= 3 (less padding of the short K extents: N=3 0.148 -> 0.139 ms), 16 above
  // (fewer stage round trips: N=9 1.94 ms at 8, 1.70 at 16, 1.73 at 32)
  const int Np = (N + 1) * (N + 2) * (N + 3) / 6, Nfp = (N + 1) * (N + 2) / 2,
            KC = BBDG_TC_KC ? BBDG_TC_KC : (N <= 3 ? 8 : 16);
  const int NB = Np <= 16 ? 16 : (Np <= 32 ? 32 : 64);   // output nodes per block
  // 128-row sub-tiles sharing each operator chunk: two while both accumulator sets of two sub-tiles
  // fit the 512 TMEM columns twice over (double buffering), else one
  const int MT = 2 * 2 * (4 * NB) <= 512 ? 2 : 1;
  return TcDims{Np, Nfp, KC, NB, (Np + NB - 1) / NB, (Np + KC - 1) / KC, (4 * Nfp + KC - 1) / KC, 3 * NB,
                (KC / 4) * 128, 3 * NB * KC * 4, NB * KC * 4, MT};
}

// bytes of a packed element image of nl elements with nk K chunks (TcLayout: 64 elements per step,
// both 128-row sub-tiles, tf32 hi and lo)
inline size_t tc_image_bytes(int N, int64_t nl, int nk) {
  const TcDims d = tc_dims(N);
  return (size_t)((nl + 32 * d.MT - 1) / (32 * d.MT)) * nk * (size_t)(d.MT * 2 * 128 * d.KC * 4);
}

template <int N> struct TcLayout {
  static constexpr TcDims d = tc_dims(N);
  static constexpr int Np = d.Np, Nfp = d.Nfp;
  static constexpr int MT = d.MT;               // 128-row sub-tiles sharing each operator chunk
  static constexpr int KE = 32;                 // elements per sub-tile -> 128 rows
  static constexpr int ST = MT * KE;            // elements per step
  static constexpr int M = 128;
  static constexpr int KC = d.KC;               // K per stage chunk (KC / 8 MMA k-steps)
  static constexpr int NB = d.NB, NBLK = d.NBLK;
  static constexpr int KV = d.KV, KL = d.KL;    // volume / lift K chunks
  static constexpr int NV = d.NV;               // volume MMA N
  static constexpr int SBO = d.SBO;             // bytes between 8-row groups
  static constexpr int A_BYTES = M * KC * 4;    // one sub-tile, one of hi / lo
  static constexpr int ABLK = MT * 2 * A_BYTES; // one packed element chunk (both sub-tiles, hi and lo)
  static constexpr int BV_BYTES = d.BV_BYTES;   // volume B chunk (hi or lo)
  static constexpr int BL_BYTES = d.BL_BYTES;
  static constexpr int B_BYTES = BV_BYTES > BL_BYTES ? BV_BYTES : BL_BYTES;
  static constexpr int B_OFF = ABLK;
  static constexpr int STAGE = B_OFF + 2 * B_BYTES;
  static constexpr int NS = (227 * 1024 - 256) / STAGE < 8 ? (227 * 1024 - 256) / STAGE : 8;   // pipeline depth
  static constexpr int total = NS * STAGE + 256;                      // + mbarriers + TMEM slot
  static constexpr int threads = 192;           // warp 0 producer, warp 1 MMA issuer, warps 2-5 epilogue
  static constexpr int ACC = NV + NB;           // accumulator columns of one sub-tile
  static constexpr int ABUF = MT * ACC;         // one accumulator buffer (double-buffered)
  static constexpr int TM_COLS = 2 * ABUF <= 128 ? 128 : (2 * ABUF <= 256 ? 256 : 512);
  static_assert(2 * ABUF <= 512, "accumulators exceed the TMEM columns");
  static_assert(NS >= 2 && total <= 227 * 1024, "tcgen05 nodal tile does not fit in shared memory");
  // packed element image: [step][kc][sub-tile][hi, lo][UMMA rows x KC] (tc_image_bytes)
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

// Pack element rows (row 4e + F of a 32-element sub-tile; row data at src + F plane + e ld) into the
// tcgen05 image: per (step, K chunk) one contiguous block [sub-tile][hi, lo][UMMA layout], the
// tf32 hi / lo split done here once (zero rows past the range, zero K past kmax).
template <int N>
__global__ void __launch_bounds__(256) tc_pack_kernel(const float* __restrict__ src, int64_t plane, int ld, int kmax,
                                                      int nk, int64_t nl, float* __restrict__ img) {
  using L = TcLayout<N>;
  constexpr int KC = L::KC, UPR = KC / 4;   // 16-byte units per row and chunk
  const int64_t nsteps = (nl + L::ST - 1) / L::ST;
  const int64_t units = nsteps * nk * L::MT * L::M * UPR;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units; u += (int64_t)gridDim.x * blockDim.x) {
    // u -> (step, kc, sub-tile, row, k-unit) with the unit fastest: reads run along a row
    const int kq = (int)(u % UPR) * 4;
    int64_t r = u / UPR;
    const int row = (int)(r % L::M);
    r /= L::M;
    const int t = (int)(r % L::MT);
    r /= L::MT;
    const int kc = (int)(r % nk);
    const int64_t step = r / nk;
    const int64_t e = step * L::ST + t * L::KE + (row >> 2);
    const int F = row & 3;
    float x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = kc * KC + kq + j;
      x[j] = (e < nl && k < kmax) ? src[F * plane + e * ld + k] : 0.f;
    }
    uint4 hi, lo;
    uint32_t* h = &hi.x;
    uint32_t* l = &lo.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[j] = tf32_bits(x[j]);
      l[j] = tf32_bits(x[j] - __uint_as_float(h[j]));
    }
    unsigned char* blk = reinterpret_cast<unsigned char*>(img) + (step * nk + kc) * (int64_t)L::ABLK + t * 2 * L::A_BYTES;
    const int off = umma_off(L::SBO, row, kq);
    *reinterpret_cast<uint4*>(blk + off) = hi;
    *reinterpret_cast<uint4*>(blk + L::A_BYTES + off) = lo;
  }
}

// The nodal face fluxes written straight into the tcgen05 flux image (tf32 hi / lo in the UMMA
// layout, row 4 e + F of the element's sub-tile, column f Nfp + m): no flux round trip through HBM.
// Column padding of the image stays zero from its allocation.
template <int N>
__global__ void __launch_bounds__(256) tc_flux_kernel(const Params<float> p) {
  using L = TcLayout<N>;
  constexpr int Nfp = L::Nfp;
  const int64_t nl = p.kend - p.kbeg;
  const int64_t total = nl * 4 * Nfp;
  unsigned char* img = static_cast<unsigned char*>(p.img_l);
  __shared__ uint16_t tab[FluxTab<N>::total];
  build_flux_tables<N>(tab);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / (4 * Nfp);
    const int fm = (int)(x - e * 4 * Nfp);
    float fl[4];
    nodal_face_flux<float, N>(p, tab, p.kbeg + e, fm, fl);
    const int64_t step = e / L::ST;
    const int el = (int)(e - step * L::ST), t = el / L::KE, kc = fm / L::KC;
    unsigned char* blk = img + (step * L::KL + kc) * (int64_t)L::ABLK + t * 2 * L::A_BYTES;
#pragma unroll
    for (int F = 0; F < 4; ++F) {
      const int off = umma_off(L::SBO, 4 * (el - t * L::KE) + F, fm - kc * L::KC);
      const uint32_t h = tf32_bits(fl[F]);
      *reinterpret_cast<uint32_t*>(blk + off) = h;
      *reinterpret_cast<uint32_t*>(blk + L::A_BYTES + off) = tf32_bits(fl[F] - __uint_as_float(h));
    }
  }
}

// Warp-specialised tcgen05 GEMM with the fused nodal epilogue.  Warp 0 streams the packed element
// chunks and the operator chunks into NS shared-memory stages with TMA bulk copies (full / empty
// mbarriers per stage), warp 1 issues the 3xTF32 MMAs for both sub-tiles and commits each stage back
// to the producer and each finished node block to the epilogue, warps 2-5 (one per TMEM lane
// quarter) read the accumulators and run the chain rule / lift / LSRK epilogue while the producer
// already streams the next block.
template <int N, int OP>
__global__ void __launch_bounds__(192, 1) nodal_tc_kernel(const Params<float> p) {
  using L = TcLayout<N>;
  constexpr int Np = L::Np, KC = L::KC, NB = L::NB, NV = L::NV, MT = L::MT, NS = L::NS;
  constexpr bool VOL = OP != OP_SURFACE, SURF = OP != OP_VOLUME;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * L::STAGE);
  uint64_t* empty = full + NS;
  uint64_t* acc_full = empty + NS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tm_slot)),
                 "n"(L::TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tm_slot;

  const int64_t fs = p.K * Np, nl = p.kend - p.kbeg;
  const int64_t nsteps = (nl + L::ST - 1) / L::ST;
  const int64_t my_steps = blockIdx.x < nsteps ? (nsteps - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  constexpr int nchunk = (VOL ? L::KV : 0) + (SURF ? L::KL : 0);
  const int nC = (int)(my_steps * L::NBLK * nchunk);
  const int nBlocks = (int)(my_steps * L::NBLK);

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const float* bvh = static_cast<const float*>(p.bvol);
      const float* blh = static_cast<const float*>(p.blift);
      // an element chunk is read once per node block: keep it in L2 until the last block's read
      const uint64_t keep = l2_policy(true), drop = l2_policy(false);
      for (int c = 0; c < nC; ++c) {
        const int st = c % NS;
        if (c >= NS) mbar_wait(empty + st, (uint32_t)(((c / NS) - 1) & 1));
        const int step_i = c / (L::NBLK * nchunk), r = c - step_i * (L::NBLK * nchunk);
        const int blk = r / nchunk, ci = r - blk * nchunk;
        const bool isvol = VOL && ci < (VOL ? L::KV : 0);
        const int kc = isvol ? ci : ci - (VOL ? L::KV : 0);
        const int64_t step = blockIdx.x + (int64_t)step_i * gridDim.x;
        const float* asrc = static_cast<const float*>(isvol ? p.img_a : p.img_l) +
                            (step * (isvol ? L::KV : L::KL) + kc) * (int64_t)(L::ABLK / 4);
        const int bbytes = isvol ? L::BV_BYTES : L::BL_BYTES;
        const float* bsrc = (isvol ? bvh : blh) + ((int64_t)(blk * (isvol ? L::KV : L::KL) + kc) * 2) * (bbytes / 4);
        unsigned char* sb = sm + st * L::STAGE;
        mbar_expect_tx(full + st, L::ABLK + 2 * bbytes);
        tma_bulk_g2s_hint(sb, asrc, L::ABLK, full + st, blk == L::NBLK - 1 ? drop : keep);
        tma_bulk_g2s_hint(sb + L::B_OFF, bsrc, 2 * bbytes, full + st, keep);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int blk_i = 0;
      for (int c = 0; c < nC; ++c) {
        const int st = c % NS;
        const int r = c % (L::NBLK * nchunk), ci = r % nchunk;
        const bool isvol = VOL && ci < (VOL ? L::KV : 0);
        const int kc = isvol ? ci : ci - (VOL ? L::KV : 0);
        const int buf = blk_i & 1;
        // the buffer's previous node block has been drained by the epilogue
        if (ci == 0 && blk_i >= 2) mbar_wait(acc_empty + buf, (uint32_t)(((blk_i >> 1) - 1) & 1));
        mbar_wait(full + st, (uint32_t)((c / NS) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        unsigned char* sb = sm + st * L::STAGE;
        const uint32_t bh = smem_u32(sb + L::B_OFF), bl = bh + (isvol ? L::BV_BYTES : L::BL_BYTES);
        const uint32_t idesc = isvol ? umma_idesc_tf32(128, NV) : umma_idesc_tf32(128, NB);
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const uint32_t ah = smem_u32(sb + t * 2 * L::A_BYTES), al = ah + L::A_BYTES;
          const uint32_t d = tmem + buf * L::ABUF + t * L::ACC + (isvol ? 0 : NV);
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint32_t ko = ks * 256;   // two 16-byte K units per k-step
            const uint64_t dah = umma_desc(ah + ko, 128, L::SBO), dal = umma_desc(al + ko, 128, L::SBO);
            const uint64_t dbh = umma_desc(bh + ko, 128, L::SBO), dbl = umma_desc(bl + ko, 128, L::SBO);
            umma_tf32(d, dal, dbh, idesc, (kc | ks) != 0);
            umma_tf32(d, dah, dbl, idesc, 1);
            umma_tf32(d, dah, dbh, idesc, 1);
          }
        }
        umma_commit(empty + st);                      // the stage is free once these MMAs complete
        if (ci == nchunk - 1) {
          umma_commit(acc_full + buf);                // the node block's accumulators are complete
          ++blk_i;
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-5)
    const int wq = warp & 3;                          // TMEM lane quarter of this warp
    const int row = wq * 32 + lane, F = row & 3, base = lane & ~3;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    for (int b = 0; b < nBlocks; ++b) {
      const int64_t step = blockIdx.x + (int64_t)(b / L::NBLK) * gridDim.x;
      const int blk = b % L::NBLK;
      const int buf = b & 1;
      mbar_wait(acc_full + buf, (uint32_t)((b >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
      for (int t = 0; t < MT; ++t) {
        const int64_t k = p.kbeg + step * L::ST + t * L::KE + (row >> 2);
        const bool okr = k < p.kend;
        const float* gv = p.geo_vol + (okr ? k : p.kbeg) * kGeoVol;
        // chain-rule coefficients of this row's field: u_i rows (F = i + 1) use column i of the
        // metric, G[3 m + i] (m = r, s, t); the p row uses none (its share of the divergence is 0)
        float Gc[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) Gc[m] = F == 0 ? 0.f : gv[3 * m + (F == 0 ? 0 : F - 1)];
        const float mat = F == 0 ? gv[9] : gv[10];   // kappa for p, 1 / rho for u_i
        const uint32_t tv = tmem + buf * L::ABUF + t * L::ACC + lane_off, tl = tv + NV;
        float* outp = p.out + F * fs + k * Np;
        float* resp = OP == OP_STAGE ? p.res + F * fs + k * Np : nullptr;
        const float* qp = OP == OP_STAGE ? p.q + F * fs + k * Np : nullptr;
#pragma unroll 1
        for (int a0 = 0; a0 < NB; a0 += 16) {
          uint32_t gr[16], gs[16], gt[16], li[16];
          if constexpr (VOL) {
            tm_ld<16>(tv + a0, gr);
            tm_ld<16>(tv + NB + a0, gs);
            tm_ld<16>(tv + 2 * NB + a0, gt);
          }
          if constexpr (SURF) tm_ld<16>(tl + a0, li);
          tm_wait_ld();
          float r[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float x = 0.f;
            if constexpr (VOL) {
              const float d0 = __uint_as_float(gr[j]), d1 = __uint_as_float(gs[j]), d2 = __uint_as_float(gt[j]);
              // u_i rows: own share of div u, and grad_i p from the p row's derivatives (lane base)
              const float c = Gc[0] * d0 + Gc[1] * d1 + Gc[2] * d2;
              const float p0 = __shfl_sync(0xffffffffu, d0, base), p1 = __shfl_sync(0xffffffffu, d1, base),
                          p2 = __shfl_sync(0xffffffffu, d2, base);
              const float g = Gc[0] * p0 + Gc[1] * p1 + Gc[2] * p2;
              float dv = c + __shfl_xor_sync(0xffffffffu, c, 1);
              dv += __shfl_xor_sync(0xffffffffu, dv, 2);   // div u over the element's four rows
              x = F == 0 ? dv : g;
            }
            // rhs = material (lift - chain rule): -kappa div u + kappa L f_p, -grad_i p / rho + L f_ui / rho
            r[j] = SURF ? mat * (__uint_as_float(li[j]) - x) : -mat * x;
          }
          const int a = blk * NB + a0;
          if (!okr || a >= Np) continue;
          if (Np % 4 == 0 && a + 16 <= Np) {   // 16-byte aligned rows: vector accesses
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              float4 v = make_float4(r[j], r[j + 1], r[j + 2], r[j + 3]);
              if constexpr (OP == OP_STAGE) {
                float4 rs = *reinterpret_cast<const float4*>(resp + a + j);
                const float4 qv = *reinterpret_cast<const float4*>(qp + a + j);
                rs.x = rs.x * p.rk_a + p.dt * v.x;
                rs.y = rs.y * p.rk_a + p.dt * v.y;
                rs.z = rs.z * p.rk_a + p.dt * v.z;
                rs.w = rs.w * p.rk_a + p.dt * v.w;
                *reinterpret_cast<float4*>(resp + a + j) = rs;
                *reinterpret_cast<float4*>(outp + a + j) =
                    make_float4(qv.x + p.rk_b * rs.x, qv.y + p.rk_b * rs.y, qv.z + p.rk_b * rs.z, qv.w + p.rk_b * rs.w);
              } else {
                if (p.accumulate) {
                  const float4 o = *reinterpret_cast<const float4*>(outp + a + j);
                  v.x += o.x;
                  v.y += o.y;
                  v.z += o.z;
                  v.w += o.w;
                }
                *reinterpret_cast<float4*>(outp + a + j) = v;
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (a + j >= Np) break;
              if constexpr (OP == OP_STAGE) {
                float x = resp[a + j] * p.rk_a;
                x = x + p.dt * r[j];
                resp[a + j] = x;
                outp[a + j] = qp[a + j] + p.rk_b * x;
              } else {
                outp[a + j] = p.accumulate ? outp[a + j] + r[j] : r[j];
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + buf);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
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
