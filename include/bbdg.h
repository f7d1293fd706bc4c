/* bbdg.h -- C ABI of the B200 BB-DG hot path (libbbdg_cuda.so, sm_100a).
 *
 * Drop-in for the per-timestep RHS evaluation and LSRK4 update of the
 * reference package (Python/numpy, /root/reference/pkg/src/bbdg).  Each entry
 * point names the reference interface it replaces.  All state pointers are
 * DEVICE pointers to C-contiguous (4, K, Np) arrays of the context's dtype
 * (reference FieldState.q layout, solver.py:80-93); `stream` is a
 * cudaStream_t (NULL = legacy default stream).  No call allocates device
 * memory on the hot path and no call synchronises the device.  State pointers must be 16-byte
 * aligned (the fused kernels stage field planes with TMA bulk copies; every cudaMalloc'd or
 * torch-allocated buffer is); misaligned pointers return BBDG_ERR_ARG.  Every function
 * returns a bbdg_status; bbdg_last_error() holds a message for the calling
 * thread.  Results are deterministic (owner-computes, no atomics).
 */
#ifndef BBDG_H
#define BBDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BBDG_OK = 0,
  BBDG_ERR_ARG = 1,          /* ValueError in the reference (shape, dt <= 0, unknown mode) */
  BBDG_ERR_UNSUPPORTED = 2,  /* degree outside the compiled range, or missing tables */
  BBDG_ERR_CUDA = 3          /* CUDA runtime error */
} bbdg_status;

enum { BBDG_BASIS_BERNSTEIN = 0, BBDG_BASIS_NODAL = 1 };
enum { BBDG_F32 = 0, BBDG_F64 = 1 };
/* lift modes of BernsteinRefOps.lift_flux (bernstein.py:457-466).  FACTORIZED (the reference
 * default, L = E_L L0, bernstein.py:301-310) and OPTIMAL (Alg. 1, :313-329) both run as L0 plus
 * the one-degree reduction sweeps in shared memory (E_L is their composition; the reference's
 * own two modes differ by <= 2.4e-16).  ELL applies E_L as stored fixed-width rows (the paper's
 * non-optimal Alg. 3 surface kernel, kept for comparison).  The nodal basis runs the reference's
 * dense path (nodal.py:236-241) either as node-per-thread kernels (DENSE, paper "NPT") or as
 * block-partitioned tensor-core GEMMs with a fused chain-rule/lift epilogue (BLOCKED, paper
 * "EPT": fp64 DMMA, fp32 3xTF32); BLOCKED is nodal-only. */
enum { BBDG_LIFT_FACTORIZED = 0, BBDG_LIFT_OPTIMAL = 1, BBDG_LIFT_DENSE = 2, BBDG_LIFT_BLOCKED = 3,
       BBDG_LIFT_ELL = 4 };

typedef struct bbdg_ctx bbdg_ctx;

/* Library identity. */
int bbdg_version(void);
int bbdg_max_degree(void);
const char* bbdg_last_error(void);

/* Context for one (mesh, degree, basis, dtype): replaces the precomputation in
 * WaveSystem.__init__ (solver.py:99-123) + ops.astype (bernstein.py:416-434). */
int bbdg_ctx_create(int N, int basis, int dtype, int64_t K, bbdg_ctx** out);
void bbdg_ctx_destroy(bbdg_ctx* ctx);

/* Per-element data, float64 host arrays, cast to the context dtype like
 * WaveSystem.__init__ (solver.py:113-123):
 *   rst_dx (K,3,3) [k,m,i] = dr_m/dx_i   kappa (K)   inv_rho (K)
 *   normals (K,4,3)  face_scale (K,4) = jf/jac  tau_p, tau_u (K,4)
 * and the compact face connectivity replacing the (K,4,Nfp) gather of
 * build_trace_maps (mesh.py:158-188):
 *   nbr_elem (K,4) int32   nbr_code (K,4) int8 = f2 | perm<<2 | boundary<<5 | halo<<6 */
int bbdg_ctx_set_geometry(bbdg_ctx* ctx, const double* rst_dx, const double* kappa, const double* inv_rho,
                          const double* normals, const double* face_scale, const double* tau_p,
                          const double* tau_u, const int32_t* nbr_elem, const int8_t* nbr_code);

/* The same per-element data for an axis-aligned box of nx x ny x nz cells, 6 Kuhn tetrahedra each
 * (mesh.box_mesh / cube_mesh, reference mesh.py:95-155), computed on the device by closed-form
 * index arithmetic -- no host arrays (HBM-filling meshes; slab-local setup of partitioned runs).
 * The context holds the cell layers [cx0, cx1) (K = 6 (cx1 - cx0) ny nz, x-slab-major element
 * order); faces into layers outside the slab but inside the box are halo faces whose slots follow
 * partition.build_halo_plan's order.  xblock = 1 is that (reference) order; xblock > 1 orders the
 * cells in slabs of xblock x-layers, (y, z, x) inside a slab, so x-neighbours sit 6 elements apart
 * (cx0 and cx1 multiples of xblock).  Homogeneous materials kappa, rho.  legacy_records = 0 builds
 * only the fused record of the hot-path kernels (the ELL, dense and nodal kernels then return
 * BBDG_ERR_UNSUPPORTED).  Synchronises `stream` (setup call). */
int bbdg_ctx_set_box_mesh(bbdg_ctx* ctx, int nx, int ny, int nz, int cx0, int cx1, int xblock, const double* lo,
                          const double* hi, double kappa, double rho, int legacy_records, void* stream);

/* Lift tables (host, float64): E_L as ELL (Np, width) for the "factorized"
 * mode (bernstein.py:273-310) and the dense (Np, 4 Nfp) lift for "dense"
 * (bernstein.py:332-347, nodal.py:411-419).  Either pointer may be NULL. */
int bbdg_ctx_set_lift_tables(bbdg_ctx* ctx, const int32_t* el_cols, const double* el_vals, int width,
                             const double* dense_L);

/* Nodal derivative matrices Dr, Ds, Dt (Np, Np) row-major, float64 (nodal.py:397-399). */
int bbdg_ctx_set_nodal_ops(bbdg_ctx* ctx, const double* Dr, const double* Ds, const double* Dt);

/* Remote face traces for element-partitioned runs: device (4, nhalo, Nfp)
 * array; faces with the halo bit read slot nbr_elem of it. */
int bbdg_ctx_set_halo(bbdg_ctx* ctx, const void* halo, int64_t nhalo);

/* WaveSystem.volume_rhs (solver.py:139-158): rhs (=|+=) volume term. */
int bbdg_volume(bbdg_ctx* ctx, const void* q, void* rhs, int accumulate, void* stream);

/* WaveSystem.surface_rhs (solver.py:166-190): rhs (=|+=) surface term. */
int bbdg_surface(bbdg_ctx* ctx, const void* q, void* rhs, int lift_mode, int accumulate, void* stream);

/* WaveSystem.rhs (solver.py:192-193): rhs = volume + surface, one pass. */
int bbdg_rhs(bbdg_ctx* ctx, const void* q, void* rhs, int lift_mode, void* stream);

/* One fused LSRK stage (solver.py:208-213 around WaveSystem.rhs):
 *   res = rk_a*res + dt*rhs(q_in);  q_out = q_in + rk_b*res.
 * q_out must not alias q_in (neighbours read q_in during the stage). */
int bbdg_lsrk_stage(bbdg_ctx* ctx, const void* q_in, void* q_out, void* res, int lift_mode, double rk_a,
                    double rk_b, double dt, void* stream);

/* Element-range variants for partitioned runs: only elements [k0, k1) are
 * updated (neighbour traces are still read from the whole plane / halo), so
 * interior elements can run while the face-trace halo is in flight. */
int bbdg_lsrk_stage_range(bbdg_ctx* ctx, const void* q_in, void* q_out, void* res, int lift_mode, double rk_a,
                          double rk_b, double dt, int64_t k0, int64_t k1, void* stream);
int bbdg_rhs_range(bbdg_ctx* ctx, const void* q, void* rhs, int lift_mode, int64_t k0, int64_t k1, void* stream);

/* The stand-alone LSRK update (solver.py:211-213) over n values, in place:
 *   res = rk_a*res + dt*rhs;  q += rk_b*res. */
int bbdg_lsrk_update(int dtype, int64_t n, void* q, void* res, const void* rhs, double rk_a, double rk_b,
                     double dt, void* stream);

/* lsrk4_step (solver.py:196-214) with the reference's in-place semantics:
 * zeroes res, runs the five fused stages and leaves the result in q.  q_tmp,
 * q_tmp2 and res are caller-owned (4,K,Np) scratch.  With q_tmp2 the stages run
 * q -> q_tmp -> q_tmp2 -> q_tmp -> q_tmp2 -> q (the last stage writes q); with
 * q_tmp2 == NULL (and in bbdg_step) they alternate q <-> q_tmp and one device
 * copy returns the result to q. */
int bbdg_step(bbdg_ctx* ctx, void* q, void* q_tmp, void* res, double dt, int lift_mode, void* stream);
int bbdg_step2(bbdg_ctx* ctx, void* q, void* q_tmp, void* q_tmp2, void* res, double dt, int lift_mode,
               void* stream);

/* lsrk4_step on a host state (solver.py:196-214 called with a numpy q): H2D of
 * host_q, the five stages and the D2H of the result into host_q, pipelined over
 * element chunks bounds[0..nchunks] (bounds[0] = 0, bounds[nchunks] = K) whose
 * neighbours lie within `reach` chunks, so the copies in both directions overlap
 * the stages of other chunks.  q, q_tmp, res are (4,K,Np) device scratch; the
 * copies run on h2d_stream / d2h_stream, the kernels on `stream`, which is
 * joined with both before return (host_q is final once `stream` completes).
 * host_q should be pinned for the copies to overlap.  Results are bitwise
 * equal to bbdg_step. */
int bbdg_step_host(bbdg_ctx* ctx, void* host_q, void* q, void* q_tmp, void* res, double dt, int lift_mode,
                   const int64_t* bounds, int nchunks, int reach, void* stream, void* h2d_stream,
                   void* d2h_stream);

/* bbdg_step_host for an ordinary (pageable) host state: the chunks move through
 * context-owned pinned staging rings (allocated on first use, `slots` chunks per
 * direction), filled and drained by `threads` host threads in parallel, so the
 * host-side copies, both PCIe directions and the stages of other chunks overlap.
 * Synchronous: host_q holds the new state on return.  Bitwise equal to
 * bbdg_step.  Replaces the reference's lsrk4_step on a numpy q (solver.py:196-214). */
int bbdg_step_pageable(bbdg_ctx* ctx, void* host_q, void* q, void* q_tmp, void* res, double dt, int lift_mode,
                       const int64_t* bounds, int nchunks, int reach, int slots, int threads, void* stream,
                       void* h2d_stream, void* d2h_stream);

/* Pack the face traces of (elem, face) pairs (device int32 (n,2)) into
 * sendbuf (4, n, Nfp) in each face's own canonical order (halo send side). */
int bbdg_halo_pack(bbdg_ctx* ctx, const void* q, void* sendbuf, const int32_t* faces, int64_t n, void* stream);

/* Device-resident functionals (float64 results written to device memory `out`; `partial`
 * is caller-owned (K) float64 scratch; deterministic fixed-order reductions).
 * discrete_energy (solver.py:306-312): out = sum_k sum_F coef[F][k] q_F^T M q_F with the
 *   symmetric mass matrix M (Np, Np) and coef (4, K) = (J/kappa, J rho, J rho, J rho).
 * ErrorFunctional (solver.py:282-296): out = sqrt(sum_k jac_k sum_i w_i (E q_0 - p_exact)^2)
 *   with eval_t = E^T (Np, nq), barycentric quadrature points lam (nq, 4), element
 *   vertices (K, 4, 3) and the standing wave p_exact of exact_solution (solver.py:249-261). */
int bbdg_energy(int dtype, int64_t K, int Np, const void* q, const double* mass, const double* coef,
                double* partial, double* out, void* stream);
int bbdg_error_l2(int dtype, int64_t K, int Np, int nq, const void* q0, const double* eval_t, const double* wq,
                  const double* lam, const double* verts, const double* jac, double tau, double* partial,
                  double* out, void* stream);

/* initial_state (solver.py:264-279) on the device: q (4, K, Np) of the context dtype =
 * tmat (Np, Np) applied to the standing wave of exact_solution (solver.py:249-261) at the
 * nodal points lam (Np, 4) (barycentric) of each element (vertices (K, 4, 3)); tmat is
 * nodal_to_bernstein's matrix for the Bernstein basis and the identity for nodal. */
int bbdg_project_standing_wave(int dtype, int64_t K, int Np, const double* tmat, const double* lam,
                               const double* verts, double tau, void* q, void* stream);

/* Operator-level applies of the reference ops bundle (no mesh; degrees 1..20; device arrays,
 * C-contiguous, batch-major):
 *   bbdg_ops_grad: BernsteinRefOps.grad (bernstein.py:436-444), q (nb, Np) -> dr, ds, dt (nb, Np)
 *   bbdg_ops_lift: lift_apply_factorized / lift_apply_optimal (bernstein.py:301-329),
 *                  flux (nb, 4, Nfp) -> out (nb, Np), as L0 + one-degree reduction sweeps
 *   bbdg_dense_apply: opcount.dense_apply (opcount.py:38-43), y (nb, nrows) = x (nb, ncols) A^T
 *                  with A (nrows, ncols) row-major (dense lift, nodal grad) */
int bbdg_ops_grad(int N, int dtype, int64_t nb, const void* q, void* dr, void* ds, void* dt, void* stream);
int bbdg_ops_lift(int N, int dtype, int64_t nb, const void* flux, void* out, void* stream);
int bbdg_dense_apply(int dtype, int64_t nb, int nrows, int ncols, const void* A, const void* x, void* y,
                     void* stream);

/* Introspection used by tests and the benchmark. */
int bbdg_ctx_read_records(bbdg_ctx* ctx, void* geo, int32_t* nbr, int32_t* code);
int bbdg_tile_elems(int N, int dtype);
int64_t bbdg_kernel_smem(int N, int dtype, int op, int lift, int basis);

#ifdef __cplusplus
}
#endif
#endif /* BBDG_H */
