// Block-partitioned nodal DG on the tensor cores (reference
// nodal.py:220-241 through WaveSystem, solver.py:139-190): the comparison path
// the paper measures BB against ("EPT" nodal).
//
// Every element tile is a small GEMM batch.  With Q_F = the (elements x Np)
// coefficients of field F, the volume is G_{m,F} = Q_F D_m^T (m = r, s, t) and
// the lift is L_F = X_F L^T where X = (Fp, n1 Fu, n2 Fu, n3 Fu) are the face
// fluxes (elements x 4 Nfp), written by nodal_flux_kernel.  One warp-level MMA
// accumulator fragment holds the same (element, node) positions for all 4
// fields, 3 derivative matrices and the lift, so the chain rule and material
// scaling (solver.py:150-158, 182-186) and the LSRK update are applied straight
// from the accumulators:
//   du_i = -(1/rho) sum_m G[m][i] g_m(p) + (1/rho) L(n_i Fu)
//   dp   = -kappa sum_m sum_i G[m][i] g_m(u_i) + kappa L(Fp)
//
// Arithmetic: fp64 uses DMMA (mma.sync m8n8k4 f64, IEEE fp64 products);
// fp32 uses 3xTF32 (mma.sync m16n8k8: hi*hi + hi*lo + lo*hi, with x = hi + lo
// split at tf32 precision), which keeps fp32-level accuracy.  The operator
// fragments (D_m^T, L^T) are pre-arranged on the host in per-lane fragment
// order (hi and lo parts pre-split), so one coalesced LDG feeds each MMA; the
// element tile (q and flux) is staged in shared memory with a row pitch that
// makes the A-fragment loads bank-conflict free.
#pragma once
#include "bbdg_tile.cuh"

namespace bbdg {

template <typename T> struct NodalMma;

// fp32: m16n8k8 tf32, 3 products per step
template <> struct NodalMma<float> {
  static constexpr int MT = 16, KS = 8, NT = 8;   // rows (elements), k per step, n per tile
  static constexpr int AR = 4, BR = 2, CR = 4;    // fragment registers per lane (A, B half, C)
  using BFrag = float4;                            // (hi b0, hi b1, lo b0, lo b1)
  __device__ static uint32_t tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
  }
  __device__ static void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  // A fragment of rows (g, g+8), cols (t, t+4) of a tile at `a` with row pitch ld; hi/lo split
  __device__ static void load_a(const float* a, int ld, int g, int t, uint32_t* hi, uint32_t* lo) {
    const float x[4] = {a[g * ld + t], a[(g + 8) * ld + t], a[g * ld + t + 4], a[(g + 8) * ld + t + 4]};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      hi[i] = tf32(x[i]);
      lo[i] = tf32(x[i] - __uint_as_float(hi[i]));
    }
  }
  __device__ static void step(float* c, const uint32_t* ahi, const uint32_t* alo, const BFrag& b) {
    const uint32_t bh0 = __float_as_uint(b.x), bh1 = __float_as_uint(b.y);
    const uint32_t bl0 = __float_as_uint(b.z), bl1 = __float_as_uint(b.w);
    mma(c, alo, bh0, bh1);
    mma(c, ahi, bl0, bl1);
    mma(c, ahi, bh0, bh1);
  }
  // C element i of this lane: row g + 8 (i >> 1), col 2t + (i & 1)
  __device__ static int crow(int g, int i) { return g + 8 * (i >> 1); }
  __device__ static int ccol(int t, int i) { return 2 * t + (i & 1); }
};

// fp64: m8n8k4 DMMA
template <> struct NodalMma<double> {
  static constexpr int MT = 8, KS = 4, NT = 8;
  static constexpr int AR = 1, BR = 1, CR = 2;
  using BFrag = double;
  __device__ static void load_a(const double* a, int ld, int g, int t, double* hi, double* lo) {
    hi[0] = a[g * ld + t];
    (void)lo;
  }
  __device__ static void step(double* c, const double* a, const double* alo, const BFrag& b) {
    (void)alo;
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a[0]), "d"(b));
  }
  __device__ static int crow(int g, int i) { return g; }
  __device__ static int ccol(int t, int i) { return 2 * t + i; }
};

// 4/8-byte cp.async with zero fill (src-size 0) for padding
template <typename T> __device__ __forceinline__ void stage_cp(uint32_t dst, const T* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(src), "n"(sizeof(T)),
               "r"(ok ? (int)sizeof(T) : 0)
               : "memory");
}

template <typename T, int N> struct NodalLayout {
  using M = NodalMma<T>;
  using D = Dims<N>;
  static constexpr int Np = D::Np, Nfp = D::Nfp;
  static constexpr int KQ = (Np + M::KS - 1) / M::KS;        // k-steps of the volume GEMM
  static constexpr int KF = (4 * Nfp + M::KS - 1) / M::KS;   // k-steps of the lift GEMM
  static constexpr int NTL = (Np + M::NT - 1) / M::NT;       // n-tiles (output nodes)
  // smem row pitch (elements): >= k extent and == 4 (mod 32 words / element size), so the A-fragment
  // addresses g * ld + t of a (half-)warp hit distinct banks
  static constexpr int pitch(int n) {
    const int m = 32 / ((int)sizeof(T) / 4);
    int x = n;
    while (x % m != 4) ++x;
    return x;
  }
  static constexpr int LQ = pitch(KQ * M::KS), LF = pitch(KF * M::KS);
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  // element M-tiles per CTA: enough that every warp has an (M-tile, n-tile) pair at low order
  static constexpr int R = NTL >= WARPS ? 1 : WARPS / NTL;
  static constexpr int WPM = WARPS / R;                        // warps per M-tile
  static constexpr int ET = R * M::MT;                         // elements per CTA tile
  static constexpr int sq = 0, sf = 4 * ET * LQ;               // [4][ET][LQ], [4][ET][LF]
  static constexpr int total = (sf + 4 * ET * LF) * (int)sizeof(T);
};

// Face-point position tables of the nodal flux kernels, built per CTA in shared memory:
//   own[f Nfp + m]            node of face f's point m (own canonical order)
//   nbt[(f2 6 + s) Nfp + m]   node of the neighbour's face f2 matching point m under vertex
//                             permutation s (multiindex.PERMS3)
//   hpt[s Nfp + m]            point index in a halo face's canonical order under permutation s
template <int N> struct FluxTab {
  static constexpr int Nfp = Dims<N>::Nfp;
  static constexpr int own = 0, nbt = 4 * Nfp, hpt = 28 * Nfp, total = 34 * Nfp;   // uint16 entries
};
template <int N> __device__ void build_flux_tables(uint16_t* t) {
  using TB = FluxTab<N>;
  constexpr int Nfp = TB::Nfp;
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int i = threadIdx.x; i < TB::total; i += blockDim.x) {
    const int r = i < TB::nbt ? i : (i < TB::hpt ? i - TB::nbt : i - TB::hpt);
    const int key = r / Nfp, m = r - key * Nfp;
    int b0, b1;
    decode2(N, m, b0, b1);
    const int b[3] = {b0, b1, N - b0 - b1};
    int v;
    if (i < TB::nbt) {   // own: face key, point m
      int a[4], s = 0;
      for (int x = 0; x < 4; ++x) a[x] = (x == key) ? 0 : b[s++];
      v = pos3(N, a[0], a[1], a[2]);
    } else {
      const int f2 = i < TB::hpt ? key / 6 : 0, sp = i < TB::hpt ? key % 6 : key;
      int c[3];
      for (int kk = 0; kk < 3; ++kk) c[perms[sp][kk]] = b[kk];
      if (i < TB::hpt) {
        int a2[4], s3 = 0;
        for (int x = 0; x < 4; ++x) a2[x] = (x == f2) ? 0 : c[s3++];
        v = pos3(N, a2[0], a2[1], a2[2]);
      } else {
        v = pos2(N, c[0], c[1]);
      }
    }
    t[i] = (uint16_t)v;
  }
  __syncthreads();
}

// Face flux of the nodal path at face point fm = f Nfp + m of element k:
// fl = (Fp, n1 Fu, n2 Fu, n3 Fu)   (solver.py:166-185); tab from build_flux_tables
template <typename T, int N>
__device__ __forceinline__ void nodal_face_flux(const Params<T>& p, const uint16_t* tab, int64_t k, int fm, T fl[4]) {
  using TB = FluxTab<N>;
  constexpr int Np = Dims<N>::Np, Nfp = TB::Nfp;
  const int64_t fs = p.K * Np;
  const int f = fm / Nfp, m = fm - f * Nfp;
  const int pos = tab[TB::own + fm];
  const T* gs = p.geo_surf + k * kGeoSurf + f * 6;
  const int cd = (p.code[k] >> (8 * f)) & 0xff;
  const bool bnd = (cd >> 5) & 1;
  T loc[4], nb[4];
#pragma unroll
  for (int F = 0; F < 4; ++F) loc[F] = p.q[F * fs + k * Np + pos];
  if (bnd) {
#pragma unroll
    for (int F = 0; F < 4; ++F) nb[F] = loc[F];
  } else {
    const int s2 = (cd >> 2) & 7, f2 = cd & 3;
    const int64_t k2 = p.nbr[k * 4 + f];
    if ((cd >> 6) & 1) {
      const int m2 = tab[TB::hpt + s2 * Nfp + m];
#pragma unroll
      for (int F = 0; F < 4; ++F) nb[F] = p.halo[(F * p.nhalo + k2) * Nfp + m2];
    } else {
      const int pos2n = tab[TB::nbt + (f2 * 6 + s2) * Nfp + m];
#pragma unroll
      for (int F = 0; F < 4; ++F) nb[F] = p.q[F * fs + k2 * Np + pos2n];
    }
  }
  const T jp = bnd ? T(-2) * loc[0] : nb[0] - loc[0];
  const T jun = gs[0] * (nb[1] - loc[1]) + gs[1] * (nb[2] - loc[2]) + gs[2] * (nb[3] - loc[3]);
  const T Fp = T(0.5) * (gs[4] * jp - jun) * gs[3];
  const T Fu = T(0.5) * (gs[5] * jun - jp) * gs[3];
  fl[0] = Fp;
  fl[1] = gs[0] * Fu;
  fl[2] = gs[1] * Fu;
  fl[3] = gs[2] * Fu;
}

// Face fluxes of the nodal path, one thread per (element, face, point):
// flux[F][k][f Nfp + m] = (Fp, n1 Fu, n2 Fu, n3 Fu)
template <typename T, int N>
__global__ void __launch_bounds__(256) nodal_flux_kernel(const Params<T> p) {
  constexpr int Nfp = Dims<N>::Nfp;
  const int64_t nl = p.kend - p.kbeg;
  const int64_t total = nl * 4 * Nfp;
  __shared__ uint16_t tab[FluxTab<N>::total];
  build_flux_tables<N>(tab);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / (4 * Nfp);
    const int fm = (int)(x - e * 4 * Nfp);
    T fl[4];
    nodal_face_flux<T, N>(p, tab, p.kbeg + e, fm, fl);
    T* o = p.flux + e * 4 * Nfp + fm;
    const int64_t ps = nl * 4 * Nfp;
#pragma unroll
    for (int F = 0; F < 4; ++F) o[F * ps] = fl[F];
  }
}

// The tensor-core GEMM + fused chain-rule / lift / LSRK epilogue.  Persistent CTAs of
// 8 warps loop over tiles of MT elements; warp w owns n-tiles w, w + 8, ...
template <typename T, int N, int OP>
__global__ void __launch_bounds__(NodalLayout<T, N>::THREADS, 1) nodal_mma_kernel(const Params<T> p) {
  using L = NodalLayout<T, N>;
  using M = NodalMma<T>;
  using AT = typename std::conditional<sizeof(T) == 4, uint32_t, double>::type;
  constexpr int Np = L::Np, Nfp = L::Nfp, MT = M::MT, KS = M::KS, NT = M::NT;
  constexpr int KQ = L::KQ, KF = L::KF, NTL = L::NTL, LQ = L::LQ, LF = L::LF;
  constexpr bool VOL = OP != OP_SURFACE, SURF = OP != OP_VOLUME;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sq = reinterpret_cast<T*>(smraw) + L::sq;
  T* sf = reinterpret_cast<T*>(smraw) + L::sf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int64_t fs = p.K * Np, nl = p.kend - p.kbeg;
  const int64_t ntiles = (nl + L::ET - 1) / L::ET;
  const auto* bvol = static_cast<const typename M::BFrag*>(p.bvol);
  const auto* blift = static_cast<const typename M::BFrag*>(p.blift);

  constexpr int ET = L::ET;
  const int mr = warp / L::WPM;          // this warp's M-tile within the CTA tile
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t kt = p.kbeg + tile * ET;
    const int nvt = (int)((p.kend - kt) < ET ? (p.kend - kt) : ET);
    // stage the tile with cp.async (non-blocking; zero fill beyond Np / 4 Nfp and the last element)
    if constexpr (VOL) {
      const uint32_t sb = smem_u32(sq);
      for (int i = tid; i < 4 * ET * LQ; i += L::THREADS) {
        const int F = i / (ET * LQ), r = i - F * ET * LQ, e = r / LQ, c = r - e * LQ;
        const bool ok = e < nvt && c < Np;
        stage_cp<T>(sb + i * (int)sizeof(T), ok ? p.q + F * fs + (kt + e) * Np + c : p.q, ok);
      }
    }
    if constexpr (SURF) {
      const uint32_t sb = smem_u32(sf);
      for (int i = tid; i < 4 * ET * LF; i += L::THREADS) {
        const int F = i / (ET * LF), r = i - F * ET * LF, e = r / LF, c = r - e * LF;
        const bool ok = e < nvt && c < 4 * Nfp;
        stage_cp<T>(sb + i * (int)sizeof(T), ok ? p.flux + (F * nl + (kt - p.kbeg + e)) * 4 * Nfp + c : p.flux, ok);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    const int64_t k0 = kt + mr * MT;
    const int nv = (int)(nvt - mr * MT < 0 ? 0 : (nvt - mr * MT < MT ? nvt - mr * MT : MT));
    const T* sqm = sq + mr * MT * LQ;    // this M-tile's rows (field stride ET LQ)
    const T* sfm = sf + mr * MT * LF;
    // geometry of this lane's accumulator rows (elements)
    T G[2][9], kap[2], irho[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = M::crow(g, 2 * h);
      const int64_t k = e < nv ? k0 + e : kt;
      const T* gv = p.geo_vol + k * kGeoVol;
#pragma unroll
      for (int j = 0; j < 9; ++j) G[h][j] = gv[j];
      kap[h] = gv[9];
      irho[h] = gv[10];
    }
    for (int nt = warp % L::WPM; nt < NTL && nv > 0; nt += L::WPM) {
      T acc[3][4][M::CR], accl[4][M::CR];
#pragma unroll
      for (int i = 0; i < M::CR; ++i) {
#pragma unroll
        for (int F = 0; F < 4; ++F) {
          accl[F][i] = T(0);
#pragma unroll
          for (int m = 0; m < 3; ++m) acc[m][F][i] = T(0);
        }
      }
      if constexpr (VOL) {
#pragma unroll 2
        for (int ks = 0; ks < KQ; ++ks) {
          AT ah[4][M::AR], al[4][M::AR];
#pragma unroll
          for (int F = 0; F < 4; ++F) M::load_a(sqm + F * ET * LQ + ks * KS, LQ, g, t, ah[F], al[F]);
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const typename M::BFrag b = __ldg(bvol + (((int64_t)m * KQ + ks) * NTL + nt) * 32 + lane);
#pragma unroll
            for (int F = 0; F < 4; ++F) M::step(acc[m][F], ah[F], al[F], b);
          }
        }
      }
      if constexpr (SURF) {
#pragma unroll 2
        for (int ks = 0; ks < KF; ++ks) {
          const typename M::BFrag b = __ldg(blift + ((int64_t)ks * NTL + nt) * 32 + lane);
#pragma unroll
          for (int F = 0; F < 4; ++F) {
            AT ah[M::AR], al[M::AR];
            M::load_a(sfm + F * ET * LF + ks * KS, LF, g, t, ah, al);
            M::step(accl[F], ah, al, b);
          }
        }
      }
      // epilogue: chain rule + lift + material scaling (+ LSRK stage) per (element, node)
#pragma unroll
      for (int i = 0; i < M::CR; ++i) {
        const int e = M::crow(g, i), a = nt * NT + M::ccol(t, i);
        const int h = (sizeof(T) == 4) ? (i >> 1) : 0;
        if (e >= nv || a >= Np) continue;
        T r[4];
        if constexpr (VOL) {
          T div = T(0);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            r[1 + c] = -irho[h] * (G[h][c] * acc[0][0][i] + G[h][3 + c] * acc[1][0][i] + G[h][6 + c] * acc[2][0][i]);
            div += G[h][c] * acc[0][1 + c][i] + G[h][3 + c] * acc[1][1 + c][i] + G[h][6 + c] * acc[2][1 + c][i];
          }
          r[0] = -kap[h] * div;
        }
        if constexpr (SURF) {
          const T s0 = kap[h] * accl[0][i], s1 = irho[h] * accl[1][i], s2 = irho[h] * accl[2][i],
                  s3 = irho[h] * accl[3][i];
          if constexpr (VOL) {
            r[0] += s0;
            r[1] += s1;
            r[2] += s2;
            r[3] += s3;
          } else {
            r[0] = s0;
            r[1] = s1;
            r[2] = s2;
            r[3] = s3;
          }
        }
        const int64_t o = (k0 + e) * Np + a;
        if constexpr (OP == OP_STAGE) {
#pragma unroll
          for (int F = 0; F < 4; ++F) {
            T x = p.res[F * fs + o] * p.rk_a;
            x = x + p.dt * r[F];
            p.res[F * fs + o] = x;
            p.out[F * fs + o] = p.q[F * fs + o] + p.rk_b * x;
          }
        } else {
#pragma unroll
          for (int F = 0; F < 4; ++F) {
            if (p.accumulate) p.out[F * fs + o] += r[F];
            else p.out[F * fs + o] = r[F];
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace bbdg
