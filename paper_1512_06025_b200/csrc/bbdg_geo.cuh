// Per-element geometry records, packed identically on the host (bbdg_ctx_set_geometry, from the
// reference Mesh arrays) and on the device (bbdg_ctx_set_box_mesh, closed-form box meshes).
#pragma once
#include <cstdint>

#include "bbdg_opt.cuh"

namespace bbdg {

// Inputs per element, float64 (WaveSystem.__init__, reference solver.py:113-123):
//   rst_dx[9] = dr_m/dx_i (m-major), kappa, inv_rho, normals[4][3], face_scale[4] = jf/jac,
//   tau_p[4], tau_u[4], nbr[4] (neighbour element / halo slot / self), code[4] (int8 face codes)
// Outputs: the fused record gr[kGeoRec] (bbdg_opt.cuh), optionally the legacy gv[kGeoVol] and
// gs[kGeoSurf] records, the neighbour row nb[4] and the packed code word.
template <typename T>
__host__ __device__ inline void pack_element(const double* rst_dx, double kappa, double inv_rho, const double* normals,
                                             const double* face_scale, const double* tau_p, const double* tau_u,
                                             const int32_t* nbr, const int* code, T* gr, T* gv, T* gs, int32_t* nb,
                                             int32_t* cd) {
  for (int j = 0; j < kGeoRec; ++j) gr[j] = T(0);
  gr[24] = static_cast<T>(kappa);
  gr[25] = static_cast<T>(inv_rho);
  for (int j = 0; j < 9; ++j) gr[26 + j] = static_cast<T>(rst_dx[j]);
  if (gv) {
    for (int j = 0; j < kGeoVol; ++j) gv[j] = T(0);
    for (int j = 0; j < 9; ++j) gv[j] = static_cast<T>(rst_dx[j]);
    gv[9] = static_cast<T>(kappa);
    gv[10] = static_cast<T>(inv_rho);
  }
  uint32_t packed = 0;
  for (int f = 0; f < 4; ++f) {
    if (gs) {
      T* g = gs + f * 6;
      for (int i = 0; i < 3; ++i) g[i] = static_cast<T>(normals[f * 3 + i]);
      g[3] = static_cast<T>(face_scale[f]);
      g[4] = static_cast<T>(tau_p[f]);
      g[5] = static_cast<T>(tau_u[f]);
    }
    const bool bnd = (code[f] >> 5) & 1;
    // fused record: the boundary mirror (jp = -2 p-, solver.py:173) rides on the sign of Bs
    const double hs = 0.5 * face_scale[f];
    for (int i = 0; i < 3; ++i) gr[4 * f + i] = static_cast<T>(normals[f * 3 + i]);
    gr[4 * f + 3] = static_cast<T>(bnd ? -hs : hs);
    gr[16 + 2 * f] = static_cast<T>(tau_p[f]);
    gr[17 + 2 * f] = static_cast<T>(hs * tau_u[f]);
    nb[f] = nbr[f];
    packed |= static_cast<uint32_t>(code[f] & 0xff) << (8 * f);
  }
  *cd = static_cast<int32_t>(packed);
}

}  // namespace bbdg
