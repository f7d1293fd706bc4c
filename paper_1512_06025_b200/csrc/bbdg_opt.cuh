// Bernstein-Bezier fused kernels for the optimal lift (reference lift_mode
// "optimal", bernstein.py:313-329) -- the bench's hot path.
//
// Same per-tile algorithm as tile_kernel (bbdg_tile.cuh: S1 flux, S2 L0,
// S3 one-degree reduction cascade, V1/V2 factored volume, fused LSRK
// epilogue), laid out so that the instruction stream is almost only
// shared-memory loads and FMAs:
//
//  * TMA bulk staging (cp.async.bulk + mbarrier) of the next tile's state
//    planes, LSRK register and geometry.  A bulk copy moves a 16-byte aligned
//    window, so each field lands at its own sub-16-byte shift; the smem field
//    stride S is chosen congruent to the global plane stride K*Np modulo
//    16/sizeof(T) (template parameter FSR), which makes every field's shift
//    equal to field 0's.  All four fields (and res) of a tile then sit at
//    compile-time distances from one per-tile base: a stencil load is one LDS
//    with an immediate offset.
//  * Per-thread work is fixed across tiles (a persistent group always
//    processes KE-element tiles), so every stencil offset / table index of a
//    thread's items is computed once in the prologue and kept in registers
//    (u16 pairs) for the whole launch.  Slots that are full for every thread
//    are unguarded at compile time (no divergence bookkeeping).
//  * The neighbour face traces of the next tile are gathered with cp.async
//    into shared memory while the current tile computes (connectivity words
//    are loaded a phase earlier); one smem table maps (neighbour face,
//    orientation, point) to the neighbour's trace position.
//  * One 36-word geometry record per element (kGeoRec) replaces the 12 +
//    24-word volume / surface records; the boundary mirror condition
//    (jp = -2 p, solver.py:173) is folded into the sign of the face scale.
//
// Phases per group tile (reference solver.py:139-214):
//   S1  upwind flux at every face point (warp-local faces)   solver.py:166-184
//   S2  L0 on (Fp, Fu), <=7 closed-form lanes                bernstein.py:221-229
//   S3  N reduction sweeps (Alg. 1), factorial-scaled         bernstein.py:313-329
//   V1  Delta_m (degree N-1) contracted with rst_dx           solver.py:139-158
//   --- group barrier
//   V2  one-degree elevation; gather of the 4 lifted faces; epilogue
//       (rhs store/accumulate, or res = A res + dt rhs; q_out = q + B res)
//   --- group barrier
#pragma once
#include "bbdg_tile.cuh"

namespace bbdg {

// Per-element geometry record (dtype T), built by bbdg_ctx_set_geometry:
//   [4f+0..2] outward normal of face f      [4f+3] Bs_f = +-face_scale_f / 2 (negative on boundary faces)
//   [16+2f]   tau_p of face f               [17+2f] C_f = tau_u face_scale_f / 2
//   [24] kappa   [25] 1/rho   [26+3m+i] rst_dx[m][i]   [35] 0
// With jp = sgn(Bs) p+ - p- (p+ = own trace on boundary faces):
//   Fp = tau_p |Bs| jp - |Bs| jun,  Fu = C jun - |Bs| jp
// i.e. solver.py:175-181 (Fp = (tau_p jp - jun) fs/2, Fu = (tau_u jun - jp) fs/2).
constexpr int kGeoRec = 36;

template <typename T> struct alignas(2 * sizeof(T)) P2 {
  T x, y;
};

// ----------------------------------------------------------------------------
// cp.async (LDGSTS) helpers
// ----------------------------------------------------------------------------
template <int B> __device__ __forceinline__ void cp_async(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst), "l"(src), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ----------------------------------------------------------------------------
// configuration: elements per group tile; groups per CTA (4 warps per group)
// ----------------------------------------------------------------------------
// (tuning builds may override the tables: -DBBDG_OPT_KE4=0,32,... etc.)
#ifndef BBDG_OPT_KE4
#define BBDG_OPT_KE4 0, 32, 16, 12, 6, 4, 3, 3, 2, 1   // (N=2: KE 16 -> 4 groups, +5.6 %; N=7: KE 3, +4 % with 4 groups)
#endif
#ifndef BBDG_OPT_KE8
#define BBDG_OPT_KE8 0, 16, 12, 6, 4, 2, 2, 2, 1, 1   // (N=6: KE 2 -> 4 groups, +7 % with res from HBM)
#endif
#ifndef BBDG_OPT_NG4
#define BBDG_OPT_NG4 0, 4, 4, 4, 4, 4, 4, 4, 3, 4
#endif
#ifndef BBDG_OPT_NG8
#define BBDG_OPT_NG8 0, 4, 4, 4, 4, 4, 4, 4, 4, 4
#endif
template <int N, int SZ> __host__ __device__ constexpr int opt_ke() {
  constexpr int k4[10] = {BBDG_OPT_KE4};
  constexpr int k8[10] = {BBDG_OPT_KE8};
  return SZ == 4 ? k4[N] : k8[N];
}
#ifndef BBDG_OPT_NG_VOL
#define BBDG_OPT_NG_VOL 8   // volume-only kernels hoist few offsets: more groups for latency hiding
#endif
#ifndef BBDG_OPT_NG_SURF
#define BBDG_OPT_NG_SURF 4
#endif
// cascade levels whose parent level spans <= this many slots read their children by shuffles
// (per order; measured: more than one slot loses in fp32 -- 3 slots: sweep 136 -> 127 GDOF/s --
// and wins only at N = 7, 9 in fp64)
#ifndef BBDG_OPT_SHF4
#define BBDG_OPT_SHF4 0, 1, 1, 1, 1, 1, 1, 1, 1, 1
#endif
#ifndef BBDG_OPT_SHF8
#define BBDG_OPT_SHF8 0, 1, 1, 1, 1, 1, 1, 2, 1, 2
#endif
template <int N, int SZ> __host__ __device__ constexpr int opt_shf_slots() {
  constexpr int s4[10] = {BBDG_OPT_SHF4};
  constexpr int s8[10] = {BBDG_OPT_SHF8};
  return SZ == 4 ? s4[N] : s8[N];
}
#ifndef BBDG_OPT_TMEM
#define BBDG_OPT_TMEM 1
#endif
#ifndef BBDG_OPT_NG_TMEM
#define BBDG_OPT_NG_TMEM 5   // groups of the fused fp32 kernels whose hoisted tables live in TMEM
#endif
#ifndef BBDG_OPT_NGT4
// per order (fp32 fused stage / rhs in TMEM mode); measured on the HBM-filling boxes (same box,
// interleaved A/B): 4 groups at N = 6, 7 +5.3 % / +4.0 % (with KE 3 at N = 7), other orders neutral or worse
#define BBDG_OPT_NGT4 0, 5, 5, 5, 5, 5, 4, 4, 5, 5
#endif
// per order: the stage reads the LSRK register straight from HBM in the epilogue instead of
// staging it (frees shared memory for more groups where shared memory caps them)
#ifndef BBDG_OPT_RESG4
#define BBDG_OPT_RESG4 0, 0, 0, 0, 0, 0, 0, 0, 0, 0
#endif
#ifndef BBDG_OPT_RESG8
#define BBDG_OPT_RESG8 0, 0, 0, 1, 1, 1, 1, 1, 1, 1   // (measured: N = 1, 2 lose 3-9 %; not smem-bound)
#endif
// per order: faces whose neighbour lies inside the tile (and boundary faces) read the neighbour
// trace from the staged state instead of gathering it (measured A/B on the HBM-filling boxes,
// fp32: N=5 +2.5 %, N=8 +8.7 %, N=4, 6, 7, 9 lose 2-6 % to the divergent S1 path; fp64: N=3
// +8.6 %, N=6 +1.2 %, the others lose up to 2.6 %)
#ifndef BBDG_OPT_LOCNB4
#define BBDG_OPT_LOCNB4 0, 0, 0, 0, 0, 1, 0, 0, 1, 0
#endif
#ifndef BBDG_OPT_LOCNB8
#define BBDG_OPT_LOCNB8 0, 0, 0, 1, 0, 0, 1, 0, 0, 0
#endif
template <int N, int SZ> __host__ __device__ constexpr bool opt_local_nb() {
  constexpr int l4[10] = {BBDG_OPT_LOCNB4};
  constexpr int l8[10] = {BBDG_OPT_LOCNB8};
  return (SZ == 4 ? l4[N] : l8[N]) != 0;
}
template <int N, int SZ> __host__ __device__ constexpr bool opt_res_global() {
  constexpr int r4[10] = {BBDG_OPT_RESG4};
  constexpr int r8[10] = {BBDG_OPT_RESG8};
  return (SZ == 4 ? r4[N] : r8[N]) != 0;
}
#ifndef BBDG_OPT_TMEM64
#define BBDG_OPT_TMEM64 1   // fp64 fused kernels park their offset tables in TMEM too (coefficients stay in smem)
#endif
#ifndef BBDG_OPT_NGT8
#define BBDG_OPT_NGT8 0, 4, 4, 5, 4, 5, 4, 4, 4, 4   // fp64 TMEM-mode groups (measured: 5 win at N=3, 5)
#endif
#ifndef BBDG_OPT_TMEM64_MIN_N
#define BBDG_OPT_TMEM64_MIN_N 3
#endif
#ifndef BBDG_OPT_TMEM_MIN_N
#define BBDG_OPT_TMEM_MIN_N 4   // (measured: no gain below N = 4, where registers do not bind)
#endif
template <int N, int SZ, int OP> __host__ __device__ constexpr int opt_max_groups() {
  constexpr int g4[10] = {BBDG_OPT_NG4};
  constexpr int g8[10] = {BBDG_OPT_NG8};
  if constexpr (OP == 0) return BBDG_OPT_NG_VOL;   // OP_VOLUME
  if constexpr (OP == 1) return (BBDG_OPT_TMEM && SZ == 4 && N >= BBDG_OPT_TMEM_MIN_N) ? BBDG_OPT_NG_TMEM
                                                                                     : BBDG_OPT_NG_SURF;  // OP_SURFACE
  constexpr int gt4[10] = {BBDG_OPT_NGT4};
  if constexpr (BBDG_OPT_TMEM && SZ == 4 && N >= BBDG_OPT_TMEM_MIN_N) return gt4[N];
  constexpr int gt8[10] = {BBDG_OPT_NGT8};
  if constexpr (BBDG_OPT_TMEM && BBDG_OPT_TMEM64 && SZ == 8 && N >= BBDG_OPT_TMEM64_MIN_N) return gt8[N];
  return SZ == 4 ? g4[N] : g8[N];
}

template <typename T, int N, int OP, int FSR> struct OptLayout {
  using D = Dims<N>;
  static constexpr int Np = D::Np, Nfp = D::Nfp, Npm = D::Npm;
  static constexpr int sz = (int)sizeof(T);
  static constexpr int A = 16 / sz;          // elements per 16 bytes
  static_assert(FSR >= 0 && FSR < A, "FSR = (K Np) mod (16 / sizeof(T))");
  static constexpr int KE = opt_ke<N, sz>();
  static constexpr int GW = 4, GT = 32 * GW;
  static constexpr bool VOL = OP != OP_SURFACE, SURF = OP != OP_VOLUME, RES = OP == OP_STAGE;
  // res not staged (coalesced streaming loads in the epilogue instead): frees the shared
  // memory of two res tiles per group (fp64: one more group at N = 6, 7, 9)
  static constexpr bool RESG = RES && opt_res_global<N, sz>();
  static constexpr bool RESS = RES && !RESG;   // res staged by TMA with the state
  static constexpr int PPW = 4 * KE / GW;   // faces per warp
  static_assert((4 * KE) % GW == 0, "faces must split evenly over the warps");
  static constexpr int NFS = odd_up(Nfp), NPS = odd_up(Np), NWS = Npm + 1;
  static constexpr int NQ = KE * Np;        // values per field per tile
  static constexpr int NB = 4 * KE * NFS;   // face-point slots per field (nb / flux buffers)
  // slot counts (items per thread, rounded up); a slot is "full" if every thread has an item
  static constexpr int NS_ITEMS = PPW * Nfp;
  static constexpr int SS = SURF ? (NS_ITEMS + 31) / 32 : 0;
  static constexpr bool TMH = BBDG_OPT_TMEM && OP != OP_VOLUME &&
                              ((sz == 4 && N >= BBDG_OPT_TMEM_MIN_N) ||
                               (sz == 8 && BBDG_OPT_TMEM64 && OP == OP_STAGE && N >= BBDG_OPT_TMEM64_MIN_N));
  // per-point coefficient tables in TMEM too (fp32 only: they are stored as 32-bit words)
  static constexpr bool TMC = TMH && sz == 4;
  static constexpr int FW = sz / 4;   // 32-bit words per T (the V1/V2 scale factors stay exact)
  // L0 lane offsets hoisted (registers, or TMEM in TMEM mode) -- else one LDS.128 per item
  static constexpr bool HOIST_L0 = SS <= 2 || TMH;
  static constexpr int SV1 = VOL ? (KE * Npm + GT - 1) / GT : 0;
  static constexpr int SV2 = (KE * Np + GT - 1) / GT;
  // cascade items are single-field: 2 PPW face-fields x tri_dim(N-j) per warp at level j
  static constexpr int s3_items(int j) { return 2 * PPW * tri_dim(N - j); }
  static constexpr int s3_slots(int j) { return (s3_items(j) + 31) / 32; }
  static constexpr int s3_base(int j) {
    int o = 0;
    for (int jj = 1; jj < j; ++jj) o += s3_slots(jj);
    return o;
  }
  static constexpr int S3T = SURF ? s3_base(N + 1) : 0;
  static constexpr int cas_u(int j) {   // largest u = 2 pw (ml+2) + 2 b0 of a cascade item at level j
    return 2 * (PPW - 1) * (N - j + 2) + 2 * (N - j);
  }
  static_assert(cas_u(1) < 256, "8-bit cascade item offsets");
  // CTA tables (bytes)
  static constexpr int o_tr2 = 0;                                      // u16 [4 f2][6 perm][Nfp] neighbour trace pos
  static constexpr int o_ptab = align16(o_tr2 + 2 * 24 * Nfp);         // u16 [6][Nfp] (halo faces)
  static constexpr int o_l0c = align16(o_ptab + 2 * 6 * Nfp);          // V4<T> [Nfp] (d, c0, c1, c2)
  static constexpr int o_ffac = align16(o_l0c + 4 * sz * Nfp);         // T [Nfp] face-point b!
  static constexpr int o_gfac = align16(o_ffac + sz * Nfp);            // V4<T> [Np]
  static constexpr int o_l0p = align16(o_gfac + 4 * sz * Np);          // u16 [Nfp][8] L0 lane positions
  static constexpr int tables = align16(o_l0p + 16 * Nfp);
  // stage (units of T; every block 16-byte aligned).  Field stride S = FSR (mod A).
  static constexpr int rnd(int n) { return (n + A - 1) / A * A; }
  static constexpr int S = rnd(NQ + 2 * A) + FSR;
  static constexpr int t_q = 0;                                   // [4][S] + shift slack
  static constexpr int t_res = rnd(t_q + 4 * S + 2 * A);          // same shape (RES)
  static constexpr int t_geo = rnd(t_res + (RESS ? 4 * S + 2 * A : 0));   // [KE][36]
  static constexpr int t_nb = rnd(t_geo + KE * kGeoRec);          // [4][NB]
  // per face of the tile: neighbour inside the tile ((k2 - k0) << 16 | trace key; read from the
  // staged state instead of gathered) or ~0 (gathered into t_nb)
  static constexpr bool LOCNB = SURF && opt_local_nb<N, sz>();
  static constexpr int t_loc = rnd(t_nb + (SURF ? 4 * NB : 0));
  static constexpr int t_bar = rnd(t_loc + (LOCNB ? (16 * KE + sz - 1) / sz : 0));   // mbarrier (8 bytes)
  static constexpr int stage_T = rnd(t_bar + 8 / sz + 1);
  static constexpr int RQ = t_res - t_q;                          // res distance from q (elements)
  // group block (units of T)
  static constexpr int g_flux = 2 * stage_T;                      // [2][NB]
  static constexpr int g_W = rnd(g_flux + (SURF ? 2 * NB : 0));   // [layer j][4KE face][tri(N-j)][p,u]
  // V1 output: fp32 4-field vectors V4 [KE][NWS] (one 16-byte load per V2 parent: quarter-warp
  // conflict domains), fp64 planar [4][KE][NWS] (a 32-byte vector would cost two loads + registers)
  static constexpr bool WAOS = sz == 4 && N >= 4;   // (measured: planar wins below N = 4)
  static constexpr int g_w = rnd(g_W + (SURF ? 8 * KE * Np : 0));
  static constexpr int group_T = rnd(g_w + (VOL ? 4 * KE * NWS : 0));
  static constexpr int group_bytes = group_T * sz;
  static constexpr int ng_fit(int budget) {
    for (int n = opt_max_groups<N, sz, OP>(); n >= 1; --n)
      if (tables + n * group_bytes <= budget) return n;
    return 0;
  }
  static constexpr int NG = ng_fit(227 * 1024) >= 1 ? ng_fit(227 * 1024) : 1;
  // hoisted per-thread tables parked in TMEM (fused fp32 kernels at high order, where
  // registers cap the group count): flat 32-bit word offsets of each table
  static constexpr int SSa_ = SS > 0 ? SS : 1, SV1a_ = SV1 > 0 ? SV1 : 1;
  static constexpr int C3W = (S3T + 1) / 2 > 0 ? (S3T + 1) / 2 : 1;
  static constexpr int H_SOF = 0, H_SEF = SSa_, H_SL0 = 2 * SSa_, H_C3 = H_SL0 + (HOIST_L0 ? 3 * SSa_ : 3);
  static constexpr int H_V1C = H_C3 + C3W, H_V1W = H_V1C + 2 * SV1a_, H_V1F = H_V1W + SV1a_;
  static constexpr int H_V2P = H_V1F + FW * SV1a_, H_V2G = H_V2P + 2 * SV2, H_V2M = H_V2G + 2 * SV2;
  static constexpr int H_V2F = H_V2M + SV2;
  // per-point coefficients (TMEM mode only): L0 4-vector + b! per S slot, gather 1/beta! 4-vector per V2 slot
  static constexpr int H_L0C = H_V2F + FW * SV2, H_FF = H_L0C + 4 * SSa_, H_GF = H_FF + SSa_;
  static constexpr int NH = TMC ? H_GF + 4 * SV2 : H_L0C;
  static_assert(!TMH || NG * NH <= 512, "TMEM-parked tables exceed the 512 TMEM columns of an SM");
  static constexpr int tm_cols() {
    int c = 32;
    while (c < NG * NH) c *= 2;
    return c;
  }
  static constexpr int threads = NG * GT;
  static constexpr int total = tables + NG * group_bytes;
  static_assert(4 * KE * NPS < 65536 && KE * Np < 65536, "u16 offsets");
};

// L0 lane positions of face point m (lane order (j,k), j != k); missing lanes -> m
template <int N> __device__ __forceinline__ void l0_lanes(int m, int pp[6]) {
  int b0, b1;
  decode2(N, m, b0, b1);
  const int b[3] = {b0, b1, N - b0 - b1};
  int l = 0;
  for (int j = 0; j < 3; ++j)
    for (int k = 0; k < 3; ++k) {
      if (j == k) continue;
      int g[3] = {b[0], b[1], b[2]};
      g[j] += 1;
      g[k] -= 1;
      pp[l++] = b[k] >= 1 ? pos2(N, g[0], g[1]) : m;
    }
}

template <typename T, int N, class L> __device__ void build_opt_tables(unsigned char* sm, int tid, int nthreads) {
  constexpr int Np = L::Np, Nfp = L::Nfp;
  uint16_t* tr2 = reinterpret_cast<uint16_t*>(sm + L::o_tr2);
  uint16_t* ptab = reinterpret_cast<uint16_t*>(sm + L::o_ptab);
  V4<T>* l0c = reinterpret_cast<V4<T>*>(sm + L::o_l0c);
  V4<T>* gfac = reinterpret_cast<V4<T>*>(sm + L::o_gfac);
  for (int i = tid; i < Np; i += nthreads) {
    int a0, a1, a2;
    decode3(N, i, a0, a1, a2);
    const int a[4] = {a0, a1, a2, N - a0 - a1 - a2};
    T gf[4];
    for (int f = 0; f < 4; ++f) {
      double d = 1.0;
      for (int v = 0; v < 4; ++v)
        if (v != f) d *= factorial(a[v]);
      gf[f] = T(1.0 / d);
    }
    gfac[i] = V4<T>{gf[0], gf[1], gf[2], gf[3]};
  }
  for (int m = tid; m < Nfp; m += nthreads) {
    int b0, b1;
    decode2(N, m, b0, b1);
    const int b[3] = {b0, b1, N - b0 - b1};
    // PERMS3 order (multiindex.py): neighbour slot sig[k] holds local vertex k
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int s2 = 0; s2 < 6; ++s2) {
      int nb[3];
      for (int k = 0; k < 3; ++k) nb[perms[s2][k]] = b[k];
      const int m2 = pos2(N, nb[0], nb[1]);
      ptab[s2 * Nfp + m] = m2;
      const int c[3] = {nb[0], nb[1], N - nb[0] - nb[1]};
      for (int f2 = 0; f2 < 4; ++f2) {
        int a[4], s = 0;
        for (int v = 0; v < 4; ++v) a[v] = (v == f2) ? 0 : c[s++];
        tr2[(f2 * 6 + s2) * Nfp + m] = pos3(N, a[0], a[1], a[2]);
      }
    }
    // L0 (bernstein.py:221-229; diag 1/2 sum (b_j+1)^2, lane (j,k) 1/2 (b_j+1) b_k at b+e_j-e_k) in
    // factorial-scaled variables: with F^[g] = g! F[g], b! (L0 F)[b] = d F^[b] + sum_k c_k sum_{j!=k} F^[b+e_j-e_k],
    // d = 1/2 sum_j (b_j+1)^2, c_k = 1/2 b_k^2 (zero exactly where the lane b+e_j-e_k does not exist)
    l0c[m] = V4<T>{T(0.5 * double((b[0] + 1) * (b[0] + 1) + (b[1] + 1) * (b[1] + 1) + (b[2] + 1) * (b[2] + 1))),
                   T(0.5 * b[0] * b[0]), T(0.5 * b[1] * b[1]), T(0.5 * b[2] * b[2])};
    reinterpret_cast<T*>(sm + L::o_ffac)[m] = T(factorial(b[0]) * factorial(b[1]) * factorial(b[2]));
    int pp[6];
    l0_lanes<N>(m, pp);
    uint16_t* l0p = reinterpret_cast<uint16_t*>(sm + L::o_l0p) + 8 * m;
    for (int x = 0; x < 6; ++x) l0p[x] = pp[x];
    l0p[6] = l0p[7] = 0;
  }
}

// ----------------------------------------------------------------------------
// TMEM as a per-lane store for the hoisted per-thread tables (tcgen05.ld/st, 32x32b shape:
// thread t of warp w owns TMEM lane 32 (w % 4) + t).  The tables are written once after the
// prologue and re-read phase by phase, so they do not occupy registers across the tile loop.
// ----------------------------------------------------------------------------
template <int C> __device__ __forceinline__ void tm_st(uint32_t ta, const uint32_t* r) {
  if constexpr (C >= 16) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
    tm_st<C - 16>(ta + 16, r + 16);
  } else if constexpr (C >= 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    tm_st<C - 8>(ta + 8, r + 8);
  } else if constexpr (C >= 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(ta), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
    tm_st<C - 4>(ta + 4, r + 4);
  } else if constexpr (C >= 2) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(ta), "r"(r[0]), "r"(r[1]) : "memory");
    tm_st<C - 2>(ta + 2, r + 2);
  } else if constexpr (C == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(ta), "r"(r[0]) : "memory");
  }
}
template <int C> __device__ __forceinline__ void tm_ld(uint32_t ta, uint32_t* r) {
  if constexpr (C >= 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
    tm_ld<C - 8>(ta + 8, r + 8);
  } else if constexpr (C >= 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(ta)
                 : "memory");
    tm_ld<C - 4>(ta + 4, r + 4);
  } else if constexpr (C >= 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(ta) : "memory");
    tm_ld<C - 2>(ta + 2, r + 2);
  } else if constexpr (C == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r[0]) : "r"(ta) : "memory");
  }
}
// a T as 32-bit TMEM words (doubles as two words, bit-exact)
template <typename T> __device__ __forceinline__ void put_words(uint32_t* w, T v) {
  if constexpr (sizeof(T) == 4) {
    w[0] = __float_as_uint((float)v);
  } else {
    const unsigned long long b = (unsigned long long)__double_as_longlong((double)v);
    w[0] = (uint32_t)b;
    w[1] = (uint32_t)(b >> 32);
  }
}
template <typename T> __device__ __forceinline__ T get_words(const uint32_t* w) {
  if constexpr (sizeof(T) == 4) return (T)__uint_as_float(w[0]);
  else return (T)__longlong_as_double((long long)(((unsigned long long)w[1] << 32) | w[0]));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t lo16(uint32_t x) { return x & 0xffffu; }
__device__ __forceinline__ uint32_t hi16(uint32_t x) { return x >> 16; }
__device__ __forceinline__ uint32_t pk(uint32_t a, uint32_t b) { return a | (b << 16); }

// value of item x (in slot x / 32, lane x % 32) of a level held one slot per register:
// one shuffle per slot, the owning slot's result kept (all lanes must call it)
template <int PS, typename T> __device__ __forceinline__ T warp_gather(const T* v, int x) {
  T r = __shfl_sync(0xffffffffu, v[0], x & 31);
#pragma unroll
  for (int s = 1; s < PS; ++s) {
    const T t = __shfl_sync(0xffffffffu, v[s], x & 31);
    if ((x >> 5) == s) r = t;
  }
  return r;
}

// run f() for slot K of a phase with `count` items spread over `width` threads;
// full slots are unguarded at compile time
template <int K, int WIDTH, int COUNT, class F> __device__ __forceinline__ void slot(int idx, F&& f) {
  if constexpr ((K + 1) * WIDTH <= COUNT) {
    f();
  } else if constexpr (K * WIDTH < COUNT) {
    if (idx + K * WIDTH < COUNT) f();
  }
}

template <typename T, int N, int OP, int FSR>
__global__ void __launch_bounds__(OptLayout<T, N, OP, FSR>::threads, 1) opt_kernel(const Params<T> p) {
  using L = OptLayout<T, N, OP, FSR>;
  constexpr int Np = L::Np, Nfp = L::Nfp, Npm = L::Npm, KE = L::KE, NG = L::NG, GT = L::GT, A = L::A;
  constexpr int NPS = L::NPS, NFS = L::NFS, NWS = L::NWS, NB = L::NB, PPW = L::PPW, S = L::S;
  constexpr int SS = L::SS, SV1 = L::SV1, SV2 = L::SV2, NSI = L::NS_ITEMS;
  constexpr int sz = (int)sizeof(T);
  extern __shared__ __align__(128) unsigned char sm[];

  const uint16_t* tr2 = reinterpret_cast<const uint16_t*>(sm + L::o_tr2);
  const uint16_t* ptab = reinterpret_cast<const uint16_t*>(sm + L::o_ptab);
  const V4<T>* l0c = reinterpret_cast<const V4<T>*>(sm + L::o_l0c);
  const V4<T>* gfac = reinterpret_cast<const V4<T>*>(sm + L::o_gfac);
  const T* ffac = reinterpret_cast<const T*>(sm + L::o_ffac);

  const int tid = threadIdx.x;
  const int g = tid / GT;
  const int gtid = tid - g * GT;
  // logical warp role, rotated per group: warp w of every group sits on SMSP w, so rotating
  // the roles gives each scheduler one warp of every role (the roles' work differs)
  const int lane = tid & 31, wg = ((gtid >> 5) + g) % L::GW;
  const int ltid = wg * 32 + lane;   // logical thread index within the group
  T* gbase = reinterpret_cast<T*>(sm + L::tables + g * L::group_bytes);
  T* sflux = gbase + L::g_flux;   // [2][NB]: F^p, F^u (flux times the face point's b!)
  T* sW = gbase + L::g_W;   // [layer j][4KE face][tri(N-j)][p,u], ell- and factorial-scaled
  T* swp = gbase + L::g_w;   // V1 output, slot Npm = 0 (see OptLayout::WAOS)
  V4<T>* sw = reinterpret_cast<V4<T>*>(swp);
  auto stage_ptr = [&](int st) { return gbase + st * L::stage_T; };
  auto stage_bar = [&](int st) { return reinterpret_cast<uint64_t*>(stage_ptr(st) + L::t_bar); };

  build_opt_tables<T, N, L>(sm, tid, L::threads);
  if constexpr (L::VOL) {
    if constexpr (L::WAOS) {
      for (int i = gtid; i < KE; i += GT) sw[i * NWS + Npm] = V4<T>{T(0), T(0), T(0), T(0)};   // V2 sentinels
    } else {
      for (int i = gtid; i < 4 * KE; i += GT) swp[i * NWS + Npm] = T(0);
    }
  }
  if (ltid == 0) {
    mbar_init(stage_bar(0), 1);
    mbar_init(stage_bar(1), 1);
    fence_barrier_init();
  }
  __syncthreads();

  // ---------------------------------------------------------------- prologue: hoisted per-thread offsets
  constexpr int SSa = SS > 0 ? SS : 1;
  uint32_t s_of[SSa];   // own-trace offset | face-point slot (flux / nb buffers)
  uint32_t s_ef[SSa];   // m | f << 8 | e << 10  (bits 8.. = face index ef = 4e + f)
  uint32_t s_l0[L::HOIST_L0 ? SSa : 1][3];   // six L0 lane offsets in the flux buffer
#pragma unroll
  for (int k = 0; k < SS; ++k) {
    const int i = lane + 32 * k;
    const bool ok = i < NSI;
    const int pw = ok ? i / Nfp : 0, m = ok ? i - pw * Nfp : 0;
    const int ef = wg * PPW + pw, e = ef >> 2, f = ef & 3;
    s_of[k] = pk(e * Np + tr2[(f * 6) * Nfp + m], ef * NFS + m);
    s_ef[k] = m | (f << 8) | (e << 10);
    if constexpr (L::HOIST_L0) {
      int pp[6];
      l0_lanes<N>(m, pp);
      s_l0[k][0] = pk(ef * NFS + pp[0], ef * NFS + pp[1]);
      s_l0[k][1] = pk(ef * NFS + pp[2], ef * NFS + pp[3]);
      s_l0[k][2] = pk(ef * NFS + pp[4], ef * NFS + pp[5]);
    }
  }
  // cascade items (level j, single field), 16 bits each, two per register: u | v << 8 with
  // u = 2 pw (ml+2) + 2 b0, v = 2 b0 (tri(ml+1) - tri(ml) = ml+2).  Item i of the warp writes W at Bw_j + i and reads its
  // children at Br_j + i + u + {0, 2} and Br_j + i + u - v + 2 (ml+2)   (see S3 below)
  uint32_t c3[(L::S3T + 1) / 2 > 0 ? (L::S3T + 1) / 2 : 1];
  if constexpr (L::SURF) {
#pragma unroll
    for (int x = 0; x < (L::S3T + 1) / 2; ++x) c3[x] = 0;
    static_for<1, N + 1>([&](auto J) {
      constexpr int j = decltype(J)::value;
      constexpr int ml = N - j, nlo = tri_dim(ml);
#pragma unroll
      for (int k = 0; k < L::s3_slots(j); ++k) {
        const int i = lane + 32 * k;
        const bool ok = i < L::s3_items(j);
        const int pi = ok ? i >> 1 : 0;
        const int pw = pi / nlo, ii = pi - pw * nlo;
        int b0, b1;
        decode2(ml, ii, b0, b1);
        const uint32_t v = (uint32_t)(2 * pw * (ml + 2) + 2 * b0) | ((uint32_t)(2 * b0) << 8);
        const int x = L::s3_base(j) + k;
        c3[x >> 1] |= v << (16 * (x & 1));
      }
    });
  }
  constexpr int SV1a = SV1 > 0 ? SV1 : 1;
  uint32_t v1c[SV1a][2], v1w[SV1a];
  T v1f[SV1a];
#pragma unroll
  for (int k = 0; k < SV1; ++k) {
    const int i = ltid + GT * k;
    const bool ok = i < KE * Npm;
    const int e = ok ? i / Npm : 0, b = ok ? i - e * Npm : 0;
    int b0, b1, b2;
    decode3(N - 1, b, b0, b1, b2);
    const int b3 = N - 1 - b0 - b1 - b2;
    v1c[k][0] = pk(e * Np + pos3(N, b0 + 1, b1, b2), e * Np + pos3(N, b0, b1 + 1, b2));
    v1c[k][1] = pk(e * Np + pos3(N, b0, b1, b2 + 1), e * Np + pos3(N, b0, b1, b2));
    v1w[k] = pk(e * NWS + b, e);
    v1f[k] = T(0.5 / (factorial(b0) * factorial(b1) * factorial(b2) * factorial(b3)));
  }
  uint32_t v2p[SV2][2], v2g[SV2][2], v2m[SV2];
  T v2f[SV2];
#pragma unroll
  for (int k = 0; k < SV2; ++k) {
    const int i = ltid + GT * k;
    const bool ok = i < KE * Np;
    const int e = ok ? i / Np : 0, a = ok ? i - e * Np : 0;
    int a0, a1, a2;
    decode3(N, a, a0, a1, a2);
    const int al[4] = {a0, a1, a2, N - a0 - a1 - a2};
    // V2 parents alpha - e_j in degree N-1 (lanes with alpha_j = 0 read the zero slot Npm)
    const int q0 = al[0] ? pos3(N - 1, a0 - 1, a1, a2) : Npm, q1 = al[1] ? pos3(N - 1, a0, a1 - 1, a2) : Npm;
    const int q2 = al[2] ? pos3(N - 1, a0, a1, a2 - 1) : Npm, q3 = al[3] ? pos3(N - 1, a0, a1, a2) : Npm;
    v2p[k][0] = pk(e * NWS + q0, e * NWS + q1);
    v2p[k][1] = pk(e * NWS + q2, e * NWS + q3);
    uint32_t li[4];
    for (int f = 0; f < 4; ++f) {
      int bb[3], s = 0;
      for (int v = 0; v < 4; ++v)
        if (v != f) bb[s++] = al[v];
      // (p, u) pair index of alpha in face f's cascade output
      li[f] = 4 * KE * layer_off(N, al[f]) + (e * 4 + f) * tri_dim(N - al[f]) + pos2(N - al[f], bb[0], bb[1]);
    }
    v2g[k][0] = pk(li[0], li[1]);
    v2g[k][1] = pk(li[2], li[3]);
    v2m[k] = pk(ok ? i : 0, (e << 10) | a);
    v2f[k] = T(factorial(al[0]) * factorial(al[1]) * factorial(al[2]) * factorial(al[3]));
  }

  // ---------------------------------------------------------------- park the tables in TMEM
  __shared__ uint32_t tm_slot;
  uint32_t ta = 0;
  if constexpr (L::TMH) {
    const int pw_id = tid >> 5;
    if (pw_id == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tm_slot)),
                   "n"(L::tm_cols()));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    ta = tm_slot + ((uint32_t)(32 * (pw_id & 3)) << 16) + (uint32_t)((pw_id >> 2) * L::NH);
    uint32_t hx[L::NH];
#pragma unroll
    for (int x = 0; x < L::NH; ++x) hx[x] = 0;
#pragma unroll
    for (int k = 0; k < SS; ++k) {
      hx[L::H_SOF + k] = s_of[k];
      hx[L::H_SEF + k] = s_ef[k];
      if constexpr (L::HOIST_L0) {
        hx[L::H_SL0 + 3 * k] = s_l0[k][0];
        hx[L::H_SL0 + 3 * k + 1] = s_l0[k][1];
        hx[L::H_SL0 + 3 * k + 2] = s_l0[k][2];
      }
    }
#pragma unroll
    for (int x = 0; x < L::C3W; ++x) hx[L::H_C3 + x] = c3[x];
#pragma unroll
    for (int k = 0; k < SV1; ++k) {
      hx[L::H_V1C + 2 * k] = v1c[k][0];
      hx[L::H_V1C + 2 * k + 1] = v1c[k][1];
      hx[L::H_V1W + k] = v1w[k];
      put_words<T>(hx + L::H_V1F + L::FW * k, v1f[k]);
    }
#pragma unroll
    for (int k = 0; k < SV2; ++k) {
      hx[L::H_V2P + 2 * k] = v2p[k][0];
      hx[L::H_V2P + 2 * k + 1] = v2p[k][1];
      hx[L::H_V2G + 2 * k] = v2g[k][0];
      hx[L::H_V2G + 2 * k + 1] = v2g[k][1];
      hx[L::H_V2M + k] = v2m[k];
      put_words<T>(hx + L::H_V2F + L::FW * k, v2f[k]);
    }
#pragma unroll
    for (int k = 0; k < (L::TMC ? SS : 0); ++k) {
      const int m = s_ef[k] & 0xff;
      const V4<T> c = l0c[m];
      hx[L::H_L0C + 4 * k] = __float_as_uint((float)c.x);
      hx[L::H_L0C + 4 * k + 1] = __float_as_uint((float)c.y);
      hx[L::H_L0C + 4 * k + 2] = __float_as_uint((float)c.z);
      hx[L::H_L0C + 4 * k + 3] = __float_as_uint((float)c.w);
      hx[L::H_FF + k] = __float_as_uint((float)ffac[m]);
    }
#pragma unroll
    for (int k = 0; k < (L::TMC ? SV2 : 0); ++k) {
      const V4<T> gf = gfac[hi16(v2m[k]) & 1023];
      hx[L::H_GF + 4 * k] = __float_as_uint((float)gf.x);
      hx[L::H_GF + 4 * k + 1] = __float_as_uint((float)gf.y);
      hx[L::H_GF + 4 * k + 2] = __float_as_uint((float)gf.z);
      hx[L::H_GF + 4 * k + 3] = __float_as_uint((float)gf.w);
    }
    tm_st<L::NH>(ta, hx);
    tm_wait_st();
  }
  // per-point coefficients, from TMEM in TMEM mode (filled by the phase loads below)
  V4<T> tl0[L::TMC ? SSa : 1], tgf[L::TMC ? SV2 : 1];
  T tff[L::TMC ? SSa : 1];
  // reload one phase's tables from TMEM (no-op when they stay in registers)
  auto tm_load_s = [&] {
    if constexpr (L::TMH) {
      uint32_t t[2 * SSa];
      tm_ld<2 * SSa>(ta + L::H_SOF, t);
      uint32_t u[3 * SSa];
      if constexpr (L::HOIST_L0) tm_ld<3 * SSa>(ta + L::H_SL0, u);
      uint32_t cf[5 * SSa];
      if constexpr (L::TMC) tm_ld<5 * SSa>(ta + L::H_L0C, cf);
      tm_wait_ld();
#pragma unroll
      for (int k = 0; k < (L::TMC ? SS : 0); ++k) {
        tl0[k] = V4<T>{(T)__uint_as_float(cf[4 * k]), (T)__uint_as_float(cf[4 * k + 1]),
                       (T)__uint_as_float(cf[4 * k + 2]), (T)__uint_as_float(cf[4 * k + 3])};
        tff[k] = (T)__uint_as_float(cf[4 * SSa + k]);
      }
#pragma unroll
      for (int k = 0; k < SS; ++k) {
        s_of[k] = t[k];
        s_ef[k] = t[SSa + k];
        if constexpr (L::HOIST_L0) {
          s_l0[k][0] = u[3 * k];
          s_l0[k][1] = u[3 * k + 1];
          s_l0[k][2] = u[3 * k + 2];
        }
      }
    }
  };
  auto tm_load_c3 = [&] {
    if constexpr (L::TMH) {
      tm_ld<L::C3W>(ta + L::H_C3, c3);
      tm_wait_ld();
    }
  };
  auto tm_load_v1 = [&] {
    if constexpr (L::TMH) {
      uint32_t t[(3 + L::FW) * SV1a];
      tm_ld<(3 + L::FW) * SV1a>(ta + L::H_V1C, t);
      tm_wait_ld();
#pragma unroll
      for (int k = 0; k < SV1; ++k) {
        v1c[k][0] = t[2 * k];
        v1c[k][1] = t[2 * k + 1];
        v1w[k] = t[2 * SV1a + k];
        v1f[k] = get_words<T>(t + 3 * SV1a + L::FW * k);
      }
    }
  };
  auto tm_load_v2 = [&] {
    if constexpr (L::TMH) {
      uint32_t t[(5 + L::FW) * SV2];
      tm_ld<(5 + L::FW) * SV2>(ta + L::H_V2P, t);
      uint32_t gq[4 * SV2];
      if constexpr (L::TMC) tm_ld<4 * SV2>(ta + L::H_GF, gq);
      tm_wait_ld();
#pragma unroll
      for (int k = 0; k < (L::TMC ? SV2 : 0); ++k)
        tgf[k] = V4<T>{(T)__uint_as_float(gq[4 * k]), (T)__uint_as_float(gq[4 * k + 1]),
                       (T)__uint_as_float(gq[4 * k + 2]), (T)__uint_as_float(gq[4 * k + 3])};
#pragma unroll
      for (int k = 0; k < SV2; ++k) {
        v2p[k][0] = t[2 * k];
        v2p[k][1] = t[2 * k + 1];
        v2g[k][0] = t[2 * SV2 + 2 * k];
        v2g[k][1] = t[2 * SV2 + 2 * k + 1];
        v2m[k] = t[4 * SV2 + k];
        v2f[k] = get_words<T>(t + 5 * SV2 + L::FW * k);
      }
    }
  };

  // ---------------------------------------------------------------- staging
  const int64_t fs = p.K * Np;
  const T* __restrict__ q = p.q;
  const int64_t ntiles = (p.kend - p.kbeg + KE - 1) / KE;
  const int64_t stride = (int64_t)gridDim.x * NG;
  int64_t tile = (int64_t)blockIdx.x * NG + g;
  auto tile_k0 = [&](int64_t t) { return p.kbeg + t * KE; };
  auto tile_nv = [&](int64_t t) {
    const int64_t r = p.kend - tile_k0(t);
    return (int)(r < KE ? r : KE);
  };
  // producer (lanes of the logical warp GW-1, one chunk each): TMA windows of the 4 state planes
  // (+ res) and the geometry records.  Field F's window is placed so that its data starts at
  // t_q + d0 + F S (d0 = (k0 Np) mod A); a window running past the array end leaves its last
  // sub-16-byte piece to plain loads, written before the barrier arrive (release).
  constexpr int NCH = L::RESS ? 9 : 5;
  auto issue_state = [&](int64_t k0, int nv, int st) {
    T* s = stage_ptr(st);
    uint64_t* bar = stage_bar(st);
    const unsigned char* src = nullptr;
    T* dst = nullptr;
    uint32_t len = 0;
    if (lane < NCH - 1) {
      const int F = lane & 3;
      const bool isq = lane < 4;
      const int64_t g0 = k0 * Np;
      const T* base = (isq ? q : p.res) + F * fs + g0;
      const int dF = (int)(reinterpret_cast<uintptr_t>(base) & 15) / sz;   // = (F fs + g0) mod A
      src = reinterpret_cast<const unsigned char*>(base - dF);
      dst = s + (isq ? L::t_q : L::t_res) + (int)(g0 % A) + F * S - dF;
      len = (uint32_t)((dF * sz + nv * Np * sz + 15) & ~15);
      const unsigned char* end = reinterpret_cast<const unsigned char*>((isq ? q : p.res) + 4 * fs);
      if (src + len > end) {
        len -= 16;
        const T* tb = reinterpret_cast<const T*>(src + len);
        T* td = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(dst) + len);
        for (const T* x = tb; reinterpret_cast<const unsigned char*>(x) < end; ++x) td[x - tb] = *x;
      }
    } else if (lane == NCH - 1) {
      src = reinterpret_cast<const unsigned char*>(p.geo + k0 * kGeoRec);
      dst = s + L::t_geo;
      len = (uint32_t)(nv * kGeoRec * sz);
    }
    if (len) mbar_expect_tx_only(bar, len);
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
    if (len) tma_bulk_g2s(dst, src, len, bar);
  };
  // neighbour face traces of tile (k0, nv): per face-point slot, 4 fields (cp.async)
  int32_t ncode[SSa], nnbr[SSa];
  auto load_conn = [&](int64_t k0, int nv) {
#pragma unroll
    for (int k = 0; k < SS; ++k) {
      const int f = (s_ef[k] >> 8) & 3, e = s_ef[k] >> 10;
      const int64_t kk = k0 + (e < nv ? e : 0);
      ncode[k] = __ldg(p.code + kk);
      nnbr[k] = __ldg(p.nbr + kk * 4 + f);
    }
  };
  auto issue_nb = [&](int64_t k0, int nv, int st) {
    const uint32_t sn = smem_u32(stage_ptr(st) + L::t_nb);
    uint32_t* sloc = reinterpret_cast<uint32_t*>(stage_ptr(st) + L::t_loc);
    static_for<0, SS>([&](auto KK) {
      constexpr int k = decltype(KK)::value;
      slot<k, 32, NSI>(lane, [&] {
        const int m = s_ef[k] & 0xff, f = (s_ef[k] >> 8) & 3, e = s_ef[k] >> 10;
        uint32_t loc = ~0u;
        if (e < nv) {
          const int cd = (ncode[k] >> (8 * f)) & 0xff;
          const bool bnd = cd & 32;
          const T* src;
          int64_t fstride = fs;
          if (!(cd & 64)) {
            // interior: neighbour's trace; boundary: own trace (the mirror sign lives in Bs)
            const int key = bnd ? f * 6 : (cd & 3) * 6 + ((cd >> 2) & 7);
            const int64_t k2 = bnd ? k0 + e : (int64_t)nnbr[k];
            // a neighbour inside the tile (a third of the faces at KE = 3, half at KE = 6, every
            // boundary face) is read from the staged state in S1: no gather
            if (L::LOCNB && k2 >= k0 && k2 < k0 + nv) loc = ((uint32_t)(k2 - k0) << 16) | (uint32_t)key;
            src = q + k2 * Np + tr2[key * Nfp + m];
          } else {
            src = p.halo + (int64_t)nnbr[k] * Nfp + ptab[((cd >> 2) & 7) * Nfp + m];
            fstride = p.nhalo * Nfp;
          }
          if (loc != ~0u) src = nullptr;
          const uint32_t d = sn + hi16(s_of[k]) * sz;
#ifndef BBDG_EXP_NO_NB   // (experiment only: skip the neighbour-trace gather to bound its cost)
          if (src) {
#pragma unroll
            for (int F = 0; F < 4; ++F) cp_async<sz>(d + F * NB * sz, src + F * fstride);
          }
#else
          (void)d;
          (void)src;
          (void)fstride;
#endif
        }
        if (L::LOCNB && m == 0) sloc[(s_ef[k] >> 8)] = loc;   // one entry per face (ef = 4 e + f)
      });
    });
  };

  if (tile < ntiles) {
    if (wg == L::GW - 1) issue_state(tile_k0(tile), tile_nv(tile), 0);
    if constexpr (L::SURF) {
      load_conn(tile_k0(tile), tile_nv(tile));
      issue_nb(tile_k0(tile), tile_nv(tile), 0);
    }
    cp_async_commit();
    cp_async_wait_all();
  }
  group_sync<GT>(g);

  for (int it = 0; tile < ntiles; tile += stride, ++it) {
    const int st = it & 1;
    const int64_t k0 = tile_k0(tile);
    const int nv = tile_nv(tile);
    const int64_t tn = tile + stride;
    const bool has_next = tn < ntiles;
    const int64_t k0n = has_next ? tile_k0(tn) : 0;
    const int nvn = has_next ? tile_nv(tn) : 0;
    tm_load_s();
    if (has_next) {
      if (wg == L::GW - 1) {
        fence_proxy_async();
        issue_state(k0n, nvn, st ^ 1);
      }
      if constexpr (L::SURF) load_conn(k0n, nvn);
    }
    const T* stg = stage_ptr(st);
    const T* sq = stg + L::t_q + (int)((k0 * Np) % A);   // field F at sq + F S; res at sq + RQ + F S
    const T* sgeo = stg + L::t_geo;
    const T* snb = stg + L::t_nb;
    const uint32_t* sloc = reinterpret_cast<const uint32_t*>(stg + L::t_loc);
    mbar_wait(stage_bar(st), (it >> 1) & 1);

    // ------------------------------------------------------------- S1: upwind flux (solver.py:166-184)
    if constexpr (L::SURF) {
      static_for<0, SS>([&](auto KK) {
        constexpr int k = decltype(KK)::value;
        slot<k, 32, NSI>(lane, [&] {
          const int own = lo16(s_of[k]), fl = hi16(s_of[k]);
          const int f = (s_ef[k] >> 8) & 3, e = (KE == 1) ? 0 : (s_ef[k] >> 10);
          const T* gr = sgeo + e * kGeoRec;
          const V4<T> nf = *reinterpret_cast<const V4<T>*>(gr + 4 * f);
          const T tp = gr[16 + 2 * f], cu = gr[17 + 2 * f];
          T loc[4], nb[4];
          // neighbour trace: staged state (neighbour inside the tile, or own trace on a boundary)
          // or the gathered buffer
          const T* nbp = snb + fl;
          int nbs = NB;
          if constexpr (L::LOCNB) {
            const uint32_t lc = sloc[s_ef[k] >> 8];
            if (lc != ~0u) {
              nbp = sq + (int)(lc >> 16) * Np + tr2[(lc & 0xffff) * Nfp + (s_ef[k] & 0xff)];
              nbs = S;
            }
          }
#pragma unroll
          for (int F = 0; F < 4; ++F) {
            loc[F] = sq[F * S + own];
            nb[F] = nbp[F * nbs];
          }
          const T bs = nf.w, ab = fabs(bs);
          const T u = bs * nb[0] - ab * loc[0];   // |Bs| jp
          const T jun = nf.x * (nb[1] - loc[1]) + nf.y * (nb[2] - loc[2]) + nf.z * (nb[3] - loc[3]);
          T fb;
          if constexpr (L::TMC) fb = tff[k];
          else fb = ffac[s_ef[k] & 0xff];
          sflux[fl] = fb * (tp * u - ab * jun);
          sflux[NB + fl] = fb * (cu * jun - u);
        });
      });
      __syncwarp();
      if (has_next) issue_nb(k0n, nvn, st ^ 1);
      cp_async_commit();

      // ------------------------------------------------------------- S2: L0 (bernstein.py:221-229), scaled by b!
      static_for<0, SS>([&](auto KK) {
        constexpr int k = decltype(KK)::value;
        slot<k, 32, NSI>(lane, [&] {
          const int fl = hi16(s_of[k]), m = s_ef[k] & 0xff;
          const int ef = s_ef[k] >> 8;
          V4<T> c;
          if constexpr (L::TMC) c = tl0[k];
          else c = l0c[m];
          int o0, o1, o2, o3, o4, o5;
          if constexpr (L::HOIST_L0) {
            o0 = lo16(s_l0[k][0]), o1 = hi16(s_l0[k][0]), o2 = lo16(s_l0[k][1]), o3 = hi16(s_l0[k][1]);
            o4 = lo16(s_l0[k][2]), o5 = hi16(s_l0[k][2]);
          } else {
            const uint4 lp = *reinterpret_cast<const uint4*>(sm + L::o_l0p + 16 * m);
            const int fb = ef * NFS;
            o0 = fb + lo16(lp.x), o1 = fb + hi16(lp.x), o2 = fb + lo16(lp.y), o3 = fb + hi16(lp.y);
            o4 = fb + lo16(lp.z), o5 = fb + hi16(lp.z);
          }
          // lanes (j,k): 0 (0,1), 1 (0,2), 2 (1,0), 3 (1,2), 4 (2,0), 5 (2,1), grouped by k
          const T* Fp = sflux;
          const T* Fu = sflux + NB;
          const T vp = c.x * Fp[fl] + c.y * (Fp[o2] + Fp[o4]) + c.z * (Fp[o0] + Fp[o5]) + c.w * (Fp[o1] + Fp[o3]);
          const T vu = c.x * Fu[fl] + c.y * (Fu[o2] + Fu[o4]) + c.z * (Fu[o0] + Fu[o5]) + c.w * (Fu[o1] + Fu[o3]);
          reinterpret_cast<P2<T>*>(sW)[ef * Nfp + m] = P2<T>{vp, vu};   // layer 0
        });
      });
      // ------------------------------------------------------------- S3: reduction cascade (Alg. 1)
      // Levels that fit one slot keep their values in a register (item i in lane i); a level
      // whose parent level also fits one slot reads its three children with shuffles instead
      // of shared memory (its values are still stored for the gather).
      tm_load_c3();
      // Every level keeps its values in registers too (item i = lane + 32 k in prev[k]); a level
      // whose parent level spans at most BBDG_OPT_SHF_SLOTS slots reads its three children by
      // warp shuffles (one per parent slot, a SHFL costs ~1/4 of an LDS on the shared-memory pipe)
      // instead of shared memory.  The values are still stored for the lift gather.
      constexpr int PSM = L::s3_slots(1);
      T prev[PSM];
#pragma unroll
      for (int k = 0; k < PSM; ++k) prev[k] = T(0);
      static_for<1, N + 1>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int ml = N - j, nlo = tri_dim(ml), nhi = tri_dim(ml + 1);
        constexpr int PS = j >= 2 ? L::s3_slots(j - 1) : 0;
        constexpr bool SHF = j >= 2 && PS <= opt_shf_slots<N, sz>();
        const T kap = T(cascade_kappa(N, j));
        T* const Bw = sW + 8 * KE * layer_off(N, j) + 2 * wg * PPW * nlo + lane;
        const T* const Br = sW + 8 * KE * layer_off(N, j - 1) + 2 * wg * PPW * nhi + lane;
        if constexpr (SHF) {
          T cur[PSM];
          static_for<0, L::s3_slots(j)>([&](auto KK) {
            constexpr int k = decltype(KK)::value;
            constexpr int x = L::s3_base(j) + k;
            const uint32_t c = c3[x >> 1] >> (16 * (x & 1));
            const int i2 = lane + 32 * k + (int)(c & 0xff), i0 = i2 - (int)((c >> 8) & 0xff) + 2 * (ml + 2);
            const T a = warp_gather<PS>(prev, i2);
            const T b = warp_gather<PS>(prev, i2 + 2);
            const T d = warp_gather<PS>(prev, i0);
            const T val = kap * ((a + b) + d);
            if (lane + 32 * k < L::s3_items(j)) Bw[32 * k] = val;
            cur[k] = val;
          });
#pragma unroll
          for (int k = 0; k < L::s3_slots(j); ++k) prev[k] = cur[k];
        } else {
          __syncwarp();
          static_for<0, L::s3_slots(j)>([&](auto KK) {
            constexpr int k = decltype(KK)::value;
            constexpr int x = L::s3_base(j) + k;
            slot<k, 32, L::s3_items(j)>(lane, [&] {
              const uint32_t c = c3[x >> 1] >> (16 * (x & 1));
              const T* rd = Br + 32 * k + (c & 0xff);
              const T* r3 = rd - ((c >> 8) & 0xff);
              const T val = kap * ((rd[0] + rd[2]) + r3[2 * (ml + 2)]);
              Bw[32 * k] = val;
              prev[k] = val;
            });
          });
        }
      });
    }

    // ------------------------------------------------------------- V1: volume, degree N-1 half
    if constexpr (L::VOL) {
      tm_load_v1();
      static_for<0, SV1>([&](auto KK) {
        constexpr int k = decltype(KK)::value;
        slot<k, GT, KE * Npm>(ltid, [&] {
          const int e = (KE == 1) ? 0 : (int)hi16(v1w[k]);
          const T* gr = sgeo + e * kGeoRec;
          const int c0 = lo16(v1c[k][0]), c1 = hi16(v1c[k][0]), c2 = lo16(v1c[k][1]), c3i = hi16(v1c[k][1]);
          T d[4][3];
#pragma unroll
          for (int F = 0; F < 4; ++F) {
            const T* qe = sq + F * S;
            const T x0 = qe[c0], x1 = qe[c1], x2 = qe[c2], x3 = qe[c3i];
            // children b+e_0..b+e_3: Delta_m = q[b+e_{m+1}] - q[b+e_0]  (exactly 0 for constant states)
            d[F][0] = x1 - x0;
            d[F][1] = x2 - x0;
            d[F][2] = x3 - x0;
          }
          const T* G = gr + 26;   // rst_dx[m][i] = G[3m+i]
          const T sr = -gr[25] * v1f[k];   // -(1/rho)/2 / beta!
          const T sk = -gr[24] * v1f[k];   // -kappa/2 / beta!
          T wu[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) wu[c] = sr * (G[c] * d[0][0] + G[3 + c] * d[0][1] + G[6 + c] * d[0][2]);
          T div = T(0);
#pragma unroll
          for (int c = 0; c < 3; ++c) div += G[c] * d[1 + c][0] + G[3 + c] * d[1 + c][1] + G[6 + c] * d[1 + c][2];
          if constexpr (L::WAOS) {
            sw[lo16(v1w[k])] = V4<T>{sk * div, wu[0], wu[1], wu[2]};
          } else {
            T* w = swp + lo16(v1w[k]);
            w[0] = sk * div;
#pragma unroll
            for (int c = 0; c < 3; ++c) w[(1 + c) * KE * NWS] = wu[c];
          }
        });
      });
    }
    group_sync<GT>(g);

    // ------------------------------------------------------------- V2 + lift gather + epilogue
    tm_load_v2();
    T* outF = p.out + k0 * Np;
    T* resF = p.res + k0 * Np;
    static_for<0, SV2>([&](auto KK) {
      constexpr int k = decltype(KK)::value;
      slot<k, GT, KE * Np>(ltid, [&] {
        const int t = lo16(v2m[k]);
        const int e = (KE == 1) ? 0 : (int)(hi16(v2m[k]) >> 10), a = hi16(v2m[k]) & 1023;
        const T* gr = sgeo + e * kGeoRec;
        (void)gr;
        (void)a;
        T r[4], rv[4];
        if constexpr (L::RESG) {   // issued first: the loads overlap the smem work below
          if (KE == 1 || (int)(hi16(v2m[k]) >> 10) < nv) {
#pragma unroll
            for (int F = 0; F < 4; ++F) rv[F] = __ldcs(resF + F * fs + t);
          }
        }
        if constexpr (L::VOL) {
          const int p0 = lo16(v2p[k][0]), p1 = hi16(v2p[k][0]), p2 = lo16(v2p[k][1]), p3 = hi16(v2p[k][1]);
          if constexpr (L::WAOS) {
            const V4<T> w0 = sw[p0], w1 = sw[p1], w2 = sw[p2], w3 = sw[p3];
            r[0] = v2f[k] * ((w0.x + w1.x) + (w2.x + w3.x));
            r[1] = v2f[k] * ((w0.y + w1.y) + (w2.y + w3.y));
            r[2] = v2f[k] * ((w0.z + w1.z) + (w2.z + w3.z));
            r[3] = v2f[k] * ((w0.w + w1.w) + (w2.w + w3.w));
          } else {
#pragma unroll
            for (int F = 0; F < 4; ++F) {
              const T* w = swp + F * KE * NWS;
              r[F] = v2f[k] * ((w[p0] + w[p1]) + (w[p2] + w[p3]));
            }
          }
        }
        if constexpr (L::SURF) {
          const int g0 = lo16(v2g[k][0]), g1 = hi16(v2g[k][0]), g2 = lo16(v2g[k][1]), g3 = hi16(v2g[k][1]);
          V4<T> gf;
          if constexpr (L::TMC) gf = tgf[k];
          else gf = gfac[a];
          const P2<T>* W2 = reinterpret_cast<const P2<T>*>(sW);
          const P2<T> w0 = W2[g0], w1 = W2[g1], w2 = W2[g2], w3 = W2[g3];
          const T sp = gf.x * w0.x + gf.y * w1.x + gf.z * w2.x + gf.w * w3.x;
          const T u0 = gf.x * w0.y, u1 = gf.y * w1.y, u2 = gf.z * w2.y, u3 = gf.w * w3.y;
          const V4<T> n0 = *reinterpret_cast<const V4<T>*>(gr + 0);
          const V4<T> n1 = *reinterpret_cast<const V4<T>*>(gr + 4);
          const V4<T> n2 = *reinterpret_cast<const V4<T>*>(gr + 8);
          const V4<T> n3 = *reinterpret_cast<const V4<T>*>(gr + 12);
          const T kap = gr[24], irho = gr[25];
          const T s0 = kap * sp;
          const T s1 = irho * (n0.x * u0 + n1.x * u1 + n2.x * u2 + n3.x * u3);
          const T s2 = irho * (n0.y * u0 + n1.y * u1 + n2.y * u2 + n3.y * u3);
          const T s3 = irho * (n0.z * u0 + n1.z * u1 + n2.z * u2 + n3.z * u3);
          if constexpr (L::VOL) {
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
        if (KE == 1 || (int)(hi16(v2m[k]) >> 10) < nv) {
          if constexpr (OP == OP_STAGE) {
            // res = A res + dt rhs; q_out = q_in + B res   (reference solver.py:211-213)
#pragma unroll
            for (int F = 0; F < 4; ++F) {
              T x;
              if constexpr (L::RESG) x = rv[F] * p.rk_a;
              else x = sq[L::RQ + F * S + t] * p.rk_a;
              x = x + p.dt * r[F];
              const T qn = sq[F * S + t] + p.rk_b * x;
              st_stream(resF + F * fs + t, x);
              st_stream(outF + F * fs + t, qn);
            }
          } else {
#pragma unroll
            for (int F = 0; F < 4; ++F) {
              T* o = outF + F * fs + t;
              if (p.accumulate) *o = *o + r[F];
              else st_stream(o, r[F]);
            }
          }
        }
      });
    });
    cp_async_wait_all();
    group_sync<GT>(g);   // neighbour traces landed; this stage / work buffers free
  }
  if constexpr (L::TMH) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if ((tid >> 5) == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm_slot), "n"(L::tm_cols()));
  }
}

}  // namespace bbdg
