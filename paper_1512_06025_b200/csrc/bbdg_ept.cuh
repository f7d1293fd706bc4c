// Element-per-thread (EPT) Bernstein-Bezier kernels for the low orders -- the fused LSRK stage
// and the rhs (reference solver.py:139-214) with every operator applied in REGISTERS.
//
// At N <= 3 an element's whole state (4 fields x Np <= 80 values) fits in one thread's registers,
// so each lane of a warp owns one element of a 32-element tile and applies the volume stencils,
// the upwind flux, L0 and the reduction sweeps of the factorised lift with compile-time indices:
// every shared-memory value is read ONCE (the cooperative kernels of bbdg_opt.cuh re-read each
// value from shared memory for every stencil lane: ~10x the HBM bytes at N = 2, 3, which made them
// shared-memory-bound).  Per warp (independent pipelines, no CTA barriers):
//
//   TMA bulk copies (cp.async.bulk + mbarrier) of the tile's 4 state planes, LSRK register and
//   geometry records into one of two stage buffers, issued one tile ahead;
//   neighbour face traces gathered with cp.async (lanes over face points, so a warp instruction
//   touches few neighbour blocks) into one of two trace buffers, one tile ahead, from the
//   connectivity loaded into registers two tiles ahead;
//   per lane: q -> registers; volume (Delta_m at degree N-1 contracted with dr/dx, elevated back
//   with weights alpha_j); per face: flux, L0 (<= 7 taps), N one-degree reductions, each layer
//   accumulated with ell_j (the lift E_L L0 as sweeps); rhs -> shared memory;
//   cooperative epilogue over contiguous words: res = A res + dt rhs; q_out = q + B res
//   (coalesced 16-byte streaming stores).
//
// Requires 16-byte aligned field windows (K Np = 0 mod 16/sizeof(T) and a tile start aligned),
// which the dispatcher checks; other layouts run the cooperative kernel.
#pragma once
#include "bbdg_opt.cuh"

namespace bbdg {

// ---------------------------------------------------------------- compile-time index algebra
struct CA4 {
  int a[4];
};
constexpr int cpos2(int m, int b0, int b1) { return b0 * (m + 1) - (b0 * (b0 - 1)) / 2 + b1; }
constexpr int ctet(int m) { return (m + 1) * (m + 2) * (m + 3) / 6; }
constexpr int ctri(int m) { return (m + 1) * (m + 2) / 2; }
constexpr int cpos3(int m, int a0, int a1, int a2) { return ctet(m) - ctet(m - a0) + cpos2(m - a0, a1, a2); }
constexpr CA4 cdec3(int m, int i) {
  int r = i, a0 = 0;
  while (r >= ctri(m - a0)) r -= ctri(m - a0), ++a0;
  int a1 = 0;
  while (r >= m - a0 - a1 + 1) r -= m - a0 - a1 + 1, ++a1;
  return CA4{{a0, a1, r, m - a0 - a1 - r}};
}
constexpr CA4 cdec2(int m, int i) {   // (b0, b1, b2)
  int r = i, b0 = 0;
  while (r >= m - b0 + 1) r -= m - b0 + 1, ++b0;
  return CA4{{b0, r, m - b0 - r, 0}};
}
// volume position of the face-f point with 2-D exponents (c0, c1, c2) on layer j (alpha_f = j)
constexpr int cface_pos(int N, int f, int j, int c0, int c1, int c2) {
  int a[4] = {0, 0, 0, 0}, s = 0;
  const int c[3] = {c0, c1, c2};
  for (int v = 0; v < 4; ++v) a[v] = (v == f) ? j : c[s++];
  return cpos3(N, a[0], a[1], a[2]);
}

template <typename T, int N> struct EptLayout {
  using D = Dims<N>;
  static constexpr int Np = D::Np, Nfp = D::Nfp, Npm = D::Npm;
  static constexpr int sz = (int)sizeof(T);
  static constexpr int A = 16 / sz;                       // elements per 16 bytes
  static constexpr int KE = 32;                           // elements per warp tile (one per lane)
  // trace buffer: [F][e][4 faces x Nfp]; a lane reads its faces with FV-element vectors (the widest
  // that keeps every face 8/16-byte aligned), and the element stride ES makes those accesses
  // conflict-free: ES / FV odd (a 4-, 8- or 16-byte access phase covers 32, 16 or 8 lanes)
  static constexpr int NFS = Nfp;
  static constexpr int FV = (Nfp % A == 0) ? A : ((Nfp % 2 == 0 && sz == 4) ? 2 : 1);
  static constexpr int es_pick() {
    int e = 4 * Nfp;
    while (e % FV != 0 || ((e / FV) % 2) == 0) ++e;
    return e;
  }
  static constexpr int ES = es_pick();
  // vector width (elements) of the per-lane state loads: Np words per element
  static constexpr int QV = (Np % A == 0) ? A : ((Np % 2 == 0 && sz == 4) ? 2 : 1);
  // per-warp stage buffer (units of T): q [4][KE Np], res [4][KE Np], geometry [KE][kGeoRec]
  static constexpr int rnd(int n) { return (n + A - 1) / A * A; }
  static constexpr int FQ = rnd(KE * Np);                 // field plane stride in the stage
  static constexpr int s_q = 0, s_res = 4 * FQ, s_geo = 8 * FQ, stage_T = rnd(s_geo + KE * kGeoRec);
  static constexpr int nb_T = rnd(4 * KE * ES);           // trace buffer (one: refilled mid-tile)
  static constexpr int w_stage0 = 0, w_nb0 = 2 * stage_T, w_conn = w_nb0 + nb_T;   // units of T
  static constexpr int w_bar = rnd(w_conn + (KE * 5 * 4 + sz - 1) / sz);                 // 2 mbarriers
  static constexpr int warp_bytes = (w_bar + 16 / sz) * sz;
  static constexpr int o_tr2 = 0;                                   // u16 [4 f2][6 perm][Nfp]
  static constexpr int o_ptab = align16(o_tr2 + 2 * 24 * Nfp);      // u16 [6][Nfp] (halo faces)
  static constexpr int tables = align16(o_ptab + 2 * 6 * Nfp);
  // W warp PAIRS per CTA (one 32-element tile pipeline each), at most 16 warps
  static constexpr int W = ((227 * 1024 - tables) / warp_bytes) < 8 ? ((227 * 1024 - tables) / warp_bytes) : 8;
  static_assert(W >= 1, "EPT tile does not fit in shared memory");
  static constexpr int threads = 64 * W;
  static constexpr int total = tables + W * warp_bytes;
};

template <typename T, int W> __device__ __forceinline__ void ld_vec(const T* s, T* r) {
  if constexpr (W == 4) {
    const V4<T> v = *reinterpret_cast<const V4<T>*>(s);
    r[0] = v.x, r[1] = v.y, r[2] = v.z, r[3] = v.w;
  } else if constexpr (W == 2) {
    const P2<T> v = *reinterpret_cast<const P2<T>*>(s);
    r[0] = v.x, r[1] = v.y;
  } else {
    r[0] = s[0];
  }
}
template <typename T, int W> __device__ __forceinline__ void st_vec(T* s, const T* r) {
  if constexpr (W == 4) {
    *reinterpret_cast<V4<T>*>(s) = V4<T>{r[0], r[1], r[2], r[3]};
  } else if constexpr (W == 2) {
    *reinterpret_cast<P2<T>*>(s) = P2<T>{r[0], r[1]};
  } else {
    s[0] = r[0];
  }
}

// Named barrier of a warp pair (ids 1.., 64 threads).
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(1 + pair) : "memory");
}

// One warp PAIR per 32-element tile, lane e of both warps on element e.  The two warps split the
// element's equations (reference solver.py:148-157, 182-189) so each holds half of the state in
// registers and the SM runs twice as many warps:
//   role 0: dp = -kappa div u + kappa L(Fp)       (u1, u2, u3 in registers; own p traces from smem)
//   role 1: du_i = -(1/rho) dp/dx_i + (1/rho) L(n_i Fu)   (p in registers; own u traces from smem)
// Both evaluate the upwind flux at every face point (Fp needs the u jump, Fu the p jump).
template <int ROLE> struct EptRole {
  static constexpr int NF = ROLE == 0 ? 3 : 1;   // fields held in registers
  static constexpr int F0 = ROLE == 0 ? 1 : 0;   // first of them
  static constexpr int NR = ROLE == 0 ? 1 : 3;   // rhs fields produced
};

// volume term (solver.py:139-158) added to r
template <int ROLE, typename T, int N, class L>
__device__ __forceinline__ void ept_volume(const T* __restrict__ gr, const T (&qv)[EptRole<ROLE>::NF][L::Np],
                                           T (&r)[EptRole<ROLE>::NR][L::Np]) {
  constexpr int Np = L::Np, Npm = L::Npm;
  constexpr int NF = EptRole<ROLE>::NF, NR = EptRole<ROLE>::NR;
  const T kap = gr[24], irho = gr[25];
  {
    T G[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) G[j] = gr[26 + j];   // rst_dx[m][i] = G[3m+i]
    // w(beta), beta of degree N-1: Delta_m = q[beta + e_{m+1}] - q[beta + e_0] contracted with dr/dx
    T w[NR][Npm > 0 ? Npm : 1];
    static_for<0, Npm>([&](auto B) {
      constexpr int b = decltype(B)::value;
      constexpr CA4 be = cdec3(N - 1, b);
      constexpr int c0 = cpos3(N, be.a[0] + 1, be.a[1], be.a[2]), c1 = cpos3(N, be.a[0], be.a[1] + 1, be.a[2]);
      constexpr int c2 = cpos3(N, be.a[0], be.a[1], be.a[2] + 1), c3 = cpos3(N, be.a[0], be.a[1], be.a[2]);
      T d[NF][3];
#pragma unroll
      for (int F = 0; F < NF; ++F) {
        d[F][0] = qv[F][c1] - qv[F][c0];
        d[F][1] = qv[F][c2] - qv[F][c0];
        d[F][2] = qv[F][c3] - qv[F][c0];
      }
      if constexpr (ROLE == 0) {
        T div = T(0);
#pragma unroll
        for (int c = 0; c < 3; ++c) div += G[c] * d[c][0] + G[3 + c] * d[c][1] + G[6 + c] * d[c][2];
        w[0][b] = (T(-0.5) * kap) * div;
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          w[c][b] = (T(-0.5) * irho) * (G[c] * d[0][0] + G[3 + c] * d[0][1] + G[6 + c] * d[0][2]);
      }
    });
    // rhs[alpha] = sum_j alpha_j w(alpha - e_j)   (exactly 0 for constant states)
    static_for<0, Np>([&](auto I) {
#pragma unroll
      for (int F = 0; F < NR; ++F) {
        T acc = T(0);
        static_for<0, 4>([&](auto J) {
          constexpr int j = decltype(J)::value;
          constexpr CA4 al = cdec3(N, decltype(I)::value);
          if constexpr (al.a[j] > 0) {
            constexpr int bj = cpos3(N - 1, al.a[0] - (j == 0), al.a[1] - (j == 1), al.a[2] - (j == 2));
            acc += T(al.a[j]) * w[F][bj];
          }
        });
        r[F][decltype(I)::value] += acc;
      }
    });
  }
}

// surface term (solver.py:166-190) added to r
template <int ROLE, typename T, int N, class L>
__device__ __forceinline__ void ept_surface(const T* __restrict__ sq, const T* __restrict__ gr,
                                            const T* __restrict__ snb, int lane,
                                            const T (&qv)[EptRole<ROLE>::NF][L::Np], T (&r)[EptRole<ROLE>::NR][L::Np]) {
  constexpr int Np = L::Np, Nfp = L::Nfp, KE = L::KE, ES = L::ES, NFS = L::NFS;
  constexpr int NR = EptRole<ROLE>::NR;
  const T kap = gr[24], irho = gr[25];
  static_for<0, 4>([&](auto FF) {
    constexpr int f = decltype(FF)::value;
    const V4<T> nf = *reinterpret_cast<const V4<T>*>(gr + 4 * f);
    const T bs = nf.w, ab = fabs(bs);
    const T cf = ROLE == 0 ? gr[16 + 2 * f] : gr[17 + 2 * f];   // tau_p (Fp) or C = tau_u |Bs| (Fu)
    T nbv[4][NFS];
#pragma unroll
    for (int F = 0; F < 4; ++F)
#pragma unroll
      for (int m = 0; m < NFS; m += L::FV) ld_vec<T, L::FV>(snb + F * KE * ES + lane * ES + f * NFS + m, &nbv[F][m]);
    // upwind flux: Fp = tau_p |Bs| jp - |Bs| jun (role 0), Fu = C jun - |Bs| jp (role 1)
    T Fx[Nfp];
    static_for<0, Nfp>([&](auto M) {
      constexpr int m = decltype(M)::value;
      constexpr CA4 b = cdec2(N, m);
      constexpr int own = cface_pos(N, decltype(FF)::value, 0, b.a[0], b.a[1], b.a[2]);
      T lp, l1, l2, l3;
      if constexpr (ROLE == 0) {
        lp = sq[lane * Np + own];
        l1 = qv[0][own], l2 = qv[1][own], l3 = qv[2][own];
      } else {
        lp = qv[0][own];
        l1 = sq[L::FQ + lane * Np + own], l2 = sq[2 * L::FQ + lane * Np + own], l3 = sq[3 * L::FQ + lane * Np + own];
      }
      const T u = bs * nbv[0][m] - ab * lp;
      const T jun = nf.x * (nbv[1][m] - l1) + nf.y * (nbv[2][m] - l2) + nf.z * (nbv[3][m] - l3);
      if constexpr (ROLE == 0) Fx[m] = cf * u - ab * jun;
      else Fx[m] = cf * jun - u;
    });
    // L0 (bernstein.py:221-229): diag 1/2 sum (b_j+1)^2, lane (j,k): 1/2 (b_j+1) b_k at b + e_j - e_k
    T wx[Nfp];
    static_for<0, Nfp>([&](auto M) {
      constexpr int m = decltype(M)::value;
      constexpr CA4 b = cdec2(N, m);
      constexpr double dg = 0.5 * ((b.a[0] + 1) * (b.a[0] + 1) + (b.a[1] + 1) * (b.a[1] + 1) + (b.a[2] + 1) * (b.a[2] + 1));
      T sx = T(dg) * Fx[m];
      static_for<0, 9>([&](auto JK) {
        constexpr int j = decltype(JK)::value / 3, k = decltype(JK)::value % 3;
        constexpr CA4 bb = cdec2(N, decltype(M)::value);
        if constexpr (j != k && bb.a[k] >= 1) {
          constexpr int gm = cpos2(N, bb.a[0] + (j == 0) - (k == 0), bb.a[1] + (j == 1) - (k == 1));
          sx += T(0.5 * (bb.a[j] + 1) * bb.a[k]) * Fx[gm];
        }
      });
      wx[m] = sx;
    });
    // material / normal scalings of this role's outputs
    T sc[NR];
    if constexpr (ROLE == 0) {
      sc[0] = kap;
    } else {
      sc[0] = irho * nf.x, sc[1] = irho * nf.y, sc[2] = irho * nf.z;
    }
    static_for<0, Nfp>([&](auto M) {   // layer 0: the face's own trace positions
      constexpr int m = decltype(M)::value;
      constexpr CA4 b = cdec2(N, m);
      constexpr int pos = cface_pos(N, decltype(FF)::value, 0, b.a[0], b.a[1], b.a[2]);
#pragma unroll
      for (int F = 0; F < NR; ++F) r[F][pos] += sc[F] * wx[m];
    });
    // layers j = 1..N: one-degree reduction (E^{ml+1}_{ml})^T, out[c] = sum_k (c_k+1)/(ml+1) w[c+e_k],
    // scaled by ell_j onto alpha_f = j   (lift_apply_optimal, bernstein.py:313-329)
    static_for<1, N + 1>([&](auto JJ) {
      T sl[NR];
#pragma unroll
      for (int F = 0; F < NR; ++F) sl[F] = T(ell_of(N, decltype(JJ)::value)) * sc[F];
      static_for<0, ctri(N - decltype(JJ)::value)>([&](auto M) {
        constexpr int m = decltype(M)::value;
        constexpr int j = decltype(JJ)::value, ml = N - j;
        constexpr double inv = 1.0 / double(ml + 1);
        constexpr CA4 c = cdec2(ml, m);
        constexpr int t0 = cpos2(ml + 1, c.a[0] + 1, c.a[1]), t1 = cpos2(ml + 1, c.a[0], c.a[1] + 1);
        constexpr int t2 = cpos2(ml + 1, c.a[0], c.a[1]);
        const T v = T((c.a[0] + 1) * inv) * wx[t0] + T((c.a[1] + 1) * inv) * wx[t1] + T((c.a[2] + 1) * inv) * wx[t2];
        wx[m] = v;   // in place: level j item m only reads level j-1 items >= m
        constexpr int pos = cface_pos(N, decltype(FF)::value, j, c.a[0], c.a[1], c.a[2]);
#pragma unroll
        for (int F = 0; F < NR; ++F) r[F][pos] += sl[F] * v;
      });
    });
  });
}

template <typename T, int W> __device__ __forceinline__ void st_global_vec(T* g, const T* r) {
  if constexpr (W == 4) {
    __stcs(reinterpret_cast<float4*>(g), make_float4(r[0], r[1], r[2], r[3]));
  } else if constexpr (W == 2 && sizeof(T) == 4) {
    __stcs(reinterpret_cast<float2*>(g), make_float2(r[0], r[1]));
  } else if constexpr (W == 2) {
    __stcs(reinterpret_cast<double2*>(g), make_double2(r[0], r[1]));
  } else {
    __stcs(g, r[0]);
  }
}

template <typename T, int N, int OP>
__global__ void __launch_bounds__(EptLayout<T, N>::threads, 1) ept_kernel(const Params<T> p) {
  using L = EptLayout<T, N>;
  constexpr int Np = L::Np, Nfp = L::Nfp, KE = L::KE, A = L::A, ES = L::ES, NFS = L::NFS;
  constexpr int sz = (int)sizeof(T);
  constexpr bool STAGE = OP == OP_STAGE;
  static_assert(OP == OP_STAGE || OP == OP_RHS, "EPT kernels: fused stage and rhs");
  extern __shared__ __align__(128) unsigned char sm[];
  const uint16_t* tr2 = reinterpret_cast<const uint16_t*>(sm + L::o_tr2);
  const uint16_t* ptab = reinterpret_cast<const uint16_t*>(sm + L::o_ptab);

  // CTA tables: neighbour trace positions per (neighbour face, orientation, point)
  for (int m = threadIdx.x; m < Nfp; m += blockDim.x) {
    int b0, b1;
    decode2(N, m, b0, b1);
    const int b[3] = {b0, b1, N - b0 - b1};
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int s2 = 0; s2 < 6; ++s2) {
      int nb[3];
      for (int k = 0; k < 3; ++k) nb[perms[s2][k]] = b[k];
      reinterpret_cast<uint16_t*>(sm + L::o_ptab)[s2 * Nfp + m] = pos2(N, nb[0], nb[1]);
      const int c[3] = {nb[0], nb[1], N - nb[0] - nb[1]};
      for (int f2 = 0; f2 < 4; ++f2) {
        int a[4], s = 0;
        for (int v = 0; v < 4; ++v) a[v] = (v == f2) ? 0 : c[s++];
        reinterpret_cast<uint16_t*>(sm + L::o_tr2)[(f2 * 6 + s2) * Nfp + m] = pos3(N, a[0], a[1], a[2]);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pair = warp >> 1, role = warp & 1;
  T* wb = reinterpret_cast<T*>(sm + L::tables + pair * L::warp_bytes);
  int32_t* sconn = reinterpret_cast<int32_t*>(wb + L::w_conn);   // [KE][5]: nbr[4], code
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + L::w_bar);
  auto stage_ptr = [&](int st) { return wb + L::w_stage0 + st * L::stage_T; };
  auto nb_ptr = [&](int st) { return wb + L::w_nb0 + st * L::nb_T; };
  if (role == 1 && lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int64_t fs = p.K * Np;
  const T* __restrict__ q = p.q;
  const int64_t ntiles = (p.kend - p.kbeg + KE - 1) / KE;
  const int64_t stride = (int64_t)gridDim.x * L::W;
  auto tile_k0 = [&](int64_t t) { return p.kbeg + t * KE; };
  auto tile_nv = [&](int64_t t) {
    const int64_t r = p.kend - tile_k0(t);
    return (int)(r < KE ? r : KE);
  };

  // role 1 issues the TMA windows (4 q planes, 4 res planes, geometry; a window running past the
  // end of its array leaves its last sub-16-byte piece to plain copies before the arrive)
  constexpr int NCH = STAGE ? 9 : 5;
  auto issue_state = [&](int64_t k0, int nv, int st) {
    T* s = stage_ptr(st);
    uint64_t* bar = bars + st;
    const unsigned char* src = nullptr;
    T* dst = nullptr;
    uint32_t len = 0;
    if (lane < NCH - 1) {
      const int F = lane & 3;
      const bool isq = lane < 4;
      const T* arr = isq ? q : p.res;
      src = reinterpret_cast<const unsigned char*>(arr + F * fs + k0 * Np);
      dst = s + (isq ? L::s_q : L::s_res) + F * L::FQ;
      len = (uint32_t)((nv * Np * sz + 15) & ~15);
      const unsigned char* end = reinterpret_cast<const unsigned char*>(arr + 4 * fs);
      if (src + len > end) {
        len -= 16;
        const T* tb = reinterpret_cast<const T*>(src + len);
        T* td = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(dst) + len);
        for (const T* x = tb; reinterpret_cast<const unsigned char*>(x) < end; ++x) td[x - tb] = *x;
      }
    } else if (lane == NCH - 1) {
      src = reinterpret_cast<const unsigned char*>(p.geo + k0 * kGeoRec);
      dst = s + L::s_geo;
      len = (uint32_t)(nv * kGeoRec * sz);
    }
    if (len) mbar_expect_tx_only(bar, len);
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
    if (len) tma_bulk_g2s(dst, src, len, bar);
  };
  // role 0 (the lighter arithmetic) gathers the neighbour traces: connectivity of its lane's element in registers (two tiles
  // ahead), items i = (e 4 + f) Nfp + m over the warp's lanes -> nb[F][e][f NFS + m]
  int32_t cn[5];
  auto load_conn = [&](int64_t k0, int nv) {
    const int64_t k = k0 + (lane < nv ? lane : 0);
    const int4 nb4 = __ldg(reinterpret_cast<const int4*>(p.nbr) + k);
    cn[0] = nb4.x, cn[1] = nb4.y, cn[2] = nb4.z, cn[3] = nb4.w;
    cn[4] = __ldg(p.code + k);
  };
  auto issue_nb = [&](int64_t k0, int nv, int st) {
#pragma unroll
    for (int k = 0; k < 5; ++k) sconn[lane * 5 + k] = cn[k];
    __syncwarp();
    const uint32_t sn = smem_u32(nb_ptr(st));
#pragma unroll 4
    for (int i = lane; i < 4 * KE * Nfp; i += 32) {
      const int ef = i / Nfp, m = i - ef * Nfp, e = ef >> 2, f = ef & 3;
      if (e < nv) {
        const int cd = (sconn[e * 5 + 4] >> (8 * f)) & 0xff;
        const int nbe = sconn[e * 5 + f];
        const T* src;
        int64_t fstride = fs;
        if (!(cd & 64)) {
          const bool bnd = cd & 32;   // boundary: own trace (the mirror sign lives in Bs)
          const int key = bnd ? f * 6 : (cd & 3) * 6 + ((cd >> 2) & 7);
          const int64_t k2 = bnd ? k0 + e : (int64_t)nbe;
          src = q + k2 * Np + tr2[key * Nfp + m];
        } else {
          src = p.halo + (int64_t)nbe * Nfp + ptab[((cd >> 2) & 7) * Nfp + m];
          fstride = p.nhalo * Nfp;
        }
        const uint32_t d = sn + (uint32_t)((e * ES + f * NFS + m) * sz);
#pragma unroll
        for (int F = 0; F < 4; ++F) cp_async<sz>(d + F * KE * ES * sz, src + F * fstride);
      }
    }
    cp_async_commit();
    __syncwarp();   // sconn reads done before the next tile's writes
  };

  int64_t tile = (int64_t)blockIdx.x * L::W + pair;
  if (tile < ntiles) {
    if (role == 1) {
      issue_state(tile_k0(tile), tile_nv(tile), 0);
    } else {
      load_conn(tile_k0(tile), tile_nv(tile));
      issue_nb(tile_k0(tile), tile_nv(tile), 0);
      const int64_t tn = tile + stride;
      if (tn < ntiles) load_conn(tile_k0(tn), tile_nv(tn));
    }
  }
  using R0 = EptRole<0>;
  using R1 = EptRole<1>;
  for (int it = 0; tile < ntiles; tile += stride, ++it) {
    const int st = it & 1;
    const int64_t k0 = tile_k0(tile);
    const int nv = tile_nv(tile);
    const int64_t tn = tile + stride, tn2 = tn + stride;
    if (role == 1 && tn < ntiles) {
      fence_proxy_async();
      issue_state(tile_k0(tn), tile_nv(tn), st ^ 1);
    }
    if (role == 0) cp_async_wait_all();   // this tile's traces landed
    mbar_wait(bars + st, (it >> 1) & 1);
    pair_sync(pair);   // the state (TMA) and the traces (role 0's cp.async) are visible to both warps

    const T* sq = stage_ptr(st) + L::s_q;
    const T* sres = stage_ptr(st) + L::s_res;
    const T* gr = stage_ptr(st) + L::s_geo + lane * kGeoRec;
    const T* snb = nb_ptr(0);
    // surface first: the trace buffer is then free for the next tile's gather, which overlaps the
    // volume term and the epilogue of this one
    auto finish = [&](auto role_c, auto& qv, auto& r) {
      constexpr int RL = decltype(role_c)::value;
      using RR = EptRole<RL>;
      ept_surface<RL, T, N, L>(sq, gr, snb, lane, qv, r);
      pair_sync(pair);
      if (RL == 0 && tn < ntiles) {
        issue_nb(tile_k0(tn), tile_nv(tn), 0);
        if (tn2 < ntiles) load_conn(tile_k0(tn2), tile_nv(tn2));
      }
      ept_volume<RL, T, N, L>(gr, qv, r);
      // epilogue per lane (element), 8/16-byte streaming stores straight from registers
      if (lane < nv) {
#pragma unroll
        for (int F = 0; F < RR::NR; ++F) {
          const int Fg = RL == 0 ? 0 : 1 + F;
          const int64_t o = Fg * fs + (k0 + lane) * Np;
#pragma unroll
          for (int i = 0; i < Np; i += L::QV) {
            T x[L::QV], y[L::QV];
            if constexpr (STAGE) {
              T ss[L::QV], qq[L::QV];
              ld_vec<T, L::QV>(sres + Fg * L::FQ + lane * Np + i, ss);
              ld_vec<T, L::QV>(sq + Fg * L::FQ + lane * Np + i, qq);
#pragma unroll
              for (int u = 0; u < L::QV; ++u) {
                x[u] = ss[u] * p.rk_a;
                x[u] = x[u] + p.dt * r[F][i + u];
                y[u] = qq[u] + p.rk_b * x[u];
              }
              st_global_vec<T, L::QV>(p.res + o + i, x);
              st_global_vec<T, L::QV>(p.out + o + i, y);
            } else {
#pragma unroll
              for (int u = 0; u < L::QV; ++u) y[u] = p.accumulate ? p.out[o + i + u] + r[F][i + u] : r[F][i + u];
              st_global_vec<T, L::QV>(p.out + o + i, y);
            }
          }
        }
      }
    };
    if (role == 0) {
      T qv[R0::NF][Np], r[R0::NR][Np];
#pragma unroll
      for (int F = 0; F < R0::NF; ++F)
#pragma unroll
        for (int i = 0; i < Np; i += L::QV) ld_vec<T, L::QV>(sq + (R0::F0 + F) * L::FQ + lane * Np + i, &qv[F][i]);
#pragma unroll
      for (int i = 0; i < Np; ++i) r[0][i] = T(0);
      finish(std::integral_constant<int, 0>{}, qv, r);
    } else {
      T qv[R1::NF][Np], r[R1::NR][Np];
#pragma unroll
      for (int i = 0; i < Np; i += L::QV) ld_vec<T, L::QV>(sq + lane * Np + i, &qv[0][i]);
#pragma unroll
      for (int F = 0; F < R1::NR; ++F)
#pragma unroll
        for (int i = 0; i < Np; ++i) r[F][i] = T(0);
      finish(std::integral_constant<int, 1>{}, qv, r);
    }
    pair_sync(pair);   // this stage buffer is free for the tile after next
  }
}

}  // namespace bbdg
