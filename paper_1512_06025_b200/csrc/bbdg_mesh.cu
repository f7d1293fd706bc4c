// Axis-aligned box meshes of Kuhn tetrahedra built directly into a context's device records
// (SURVEY 8f-2): the per-element geometry and compact connectivity of mesh.box_mesh /
// cube_mesh (reference mesh.py:95-155 + WaveSystem.__init__, solver.py:99-123), one thread per
// element, with no host arrays and no transient device memory -- so meshes that fill a B200's
// HBM set up in milliseconds, and each rank of a slab partition builds only its own slab.
//
// Element e of the slab [cx0, cx1) x ny x nz cells is tet t = e mod 6 of cell e / 6 in the
// (x-blocked, see cell_lin) cell order counted from layer cx0: the lattice path c, c + e_p0,
// c + e_p0 + e_p1, c + (1,1,1) for the axis permutation p = AXIS_PERMS[t] (mesh.box_mesh),
// with vertices 1 and 2 swapped for odd permutations (mesh._orient).  Face f is opposite
// vertex f (multiindex.FACE_VERTICES).  The neighbour across the face opposite path vertex
//   0: cell + e_p0, permutation (p1, p2, p0)       3: cell - e_p2, (p2, p0, p1)
//   1: same cell, (p1, p0, p2)                     2: same cell, (p0, p2, p1)
// (the Freudenthal triangulation), so connectivity, the neighbour's face and the vertex
// permutation code follow from index arithmetic.  Faces leaving the slab but not the box are
// halo faces: slots in the (receiver element, receiver face) order of partition.build_halo_plan
// (left peer first: cells (cx0, j, k), tets 3 and 5 -> 2 (j nz + k) + (t == 5); then the right
// peer: cells (cx1 - 1, j, k), tets 0 and 1 -> nleft + 2 (j nz + k) + t).
#include <vector>

#include "bbdg_geo.cuh"
#include "bbdg_internal.h"

namespace bbdg {
namespace {

__device__ const int kAxisPerms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__device__ const int kFaceVerts[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
__device__ const int kPerms3[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

struct Box {
  int nx, ny, nz;        // global cells
  int cx0, cx1;          // this slab's cell layers
  int xb;                // x-blocking of the element order (1 = the reference's x-slab-major order)
  double lo[3], step[3], hi[3];
  double kappa, inv_rho, tau_p, tau_u;
};

__device__ __forceinline__ bool odd_perm(int t) { return t == 1 || t == 2 || t == 5; }

__device__ __forceinline__ int perm_index(int a, int b) {   // AXIS_PERMS index of (a, b, 3 - a - b)
  for (int t = 0; t < 6; ++t)
    if (kAxisPerms[t][0] == a && kAxisPerms[t][1] == b) return t;
  return 0;
}

// oriented lattice vertices (cell + offsets) of tet t of cell c
__device__ void tet_vertices(const int c[3], int t, int v[4][3]) {
  int cur[3] = {c[0], c[1], c[2]};
  int path[4][3];
  for (int i = 0; i < 3; ++i) path[0][i] = cur[i];
  for (int s = 0; s < 3; ++s) {
    cur[kAxisPerms[t][s]] += 1;
    for (int i = 0; i < 3; ++i) path[s + 1][i] = cur[i];
  }
  const int ord[4] = {0, odd_perm(t) ? 2 : 1, odd_perm(t) ? 1 : 2, 3};
  for (int a = 0; a < 4; ++a)
    for (int i = 0; i < 3; ++i) v[a][i] = path[ord[a]][i];
}

__device__ __forceinline__ bool same(const int* a, const int* b) { return a[0] == b[0] && a[1] == b[1] && a[2] == b[2]; }

// Cell order: slabs of xb x-layers (the last one may be thinner), slab-major; inside a slab the cells
// run (y, z, x) with x fastest.  xb = 1 is the reference's x-slab-major cube_mesh order; xb > 1 puts
// the x-neighbours of a cell 6 elements apart (the y-neighbours 6 xb nz apart), so an HBM-filling
// mesh reads its neighbour traces from L2 instead of DRAM (only the faces between slabs are far).
__device__ __forceinline__ int64_t cell_lin(const Box& b, int cx, int cy, int cz) {
  const int s = cx / b.xb, ts = min(b.xb, b.nx - s * b.xb);
  return (int64_t)s * b.xb * b.ny * b.nz + ((int64_t)cy * b.nz + cz) * ts + (cx - s * b.xb);
}
__device__ __forceinline__ void cell_of(const Box& b, int64_t lin, int c[3]) {
  const int64_t slab = (int64_t)b.xb * b.ny * b.nz;
  const int nslab = (b.nx + b.xb - 1) / b.xb;
  int64_t s = lin / slab;
  if (s > nslab - 1) s = nslab - 1;
  const int64_t rem = lin - s * slab;
  const int ts = min(b.xb, b.nx - (int)s * b.xb);
  const int64_t yz = rem / ts;
  c[0] = (int)(s * b.xb + (rem - yz * ts));
  c[1] = (int)(yz / b.nz);
  c[2] = (int)(yz - (int64_t)c[1] * b.nz);
}

// numpy.linspace(lo, hi, n + 1)[i] = i * step + lo (last point = hi), no FMA contraction
__device__ __forceinline__ double coord(const Box& b, int axis, int i) {
  const int n = axis == 0 ? b.nx : (axis == 1 ? b.ny : b.nz);
  return i == n ? b.hi[axis] : __dadd_rn(__dmul_rn((double)i, b.step[axis]), b.lo[axis]);
}

template <typename T>
__global__ void box_mesh_kernel(Box b, int64_t K, T* __restrict__ geo, T* __restrict__ geo_vol,
                                T* __restrict__ geo_surf, int32_t* __restrict__ nbr_out, int32_t* __restrict__ code_out) {
  const int64_t plane = (int64_t)b.ny * b.nz;
  const int nleft = b.cx0 > 0 ? 2 * b.ny * b.nz : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = (int64_t)b.cx0 * plane;   // cx0 is a multiple of xb: full slabs before it
    const int t = (int)(e % 6);
    int c[3];
    cell_of(b, base + e / 6, c);
    int v[4][3];
    tet_vertices(c, t, v);
    double x[4][3];
    for (int a = 0; a < 4; ++a)
      for (int i = 0; i < 3; ++i) x[a][i] = coord(b, i, v[a][i]);
    // affine map x = v0 + (1/2) [v1-v0 | v2-v0 | v3-v0] (r+1): dxdr[x][m] (mesh._geometry)
    double A[3][3];
    for (int i = 0; i < 3; ++i)
      for (int m = 0; m < 3; ++m) A[i][m] = 0.5 * (x[m + 1][i] - x[0][i]);
    const double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                       A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    double rst_dx[9];   // inverse: rst_dx[m][i] = d r_m / d x_i
    rst_dx[0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / det;
    rst_dx[1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
    rst_dx[2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
    rst_dx[3] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / det;
    rst_dx[4] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
    rst_dx[5] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
    rst_dx[6] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / det;
    rst_dx[7] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
    rst_dx[8] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    double cen[3];
    for (int i = 0; i < 3; ++i) cen[i] = 0.25 * (x[0][i] + x[1][i] + x[2][i] + x[3][i]);
    double normals[12], fscale[4], taup[4], tauu[4];
    int32_t nb[4];
    int code[4];
    for (int f = 0; f < 4; ++f) {
      const int* fv = kFaceVerts[f];
      double u[3], w[3], a[3], fc[3];
      for (int i = 0; i < 3; ++i) {
        u[i] = x[fv[1]][i] - x[fv[0]][i];
        w[i] = x[fv[2]][i] - x[fv[0]][i];
        fc[i] = (x[fv[0]][i] + x[fv[1]][i] + x[fv[2]][i]) / 3.0 - cen[i];
      }
      a[0] = 0.5 * (u[1] * w[2] - u[2] * w[1]);
      a[1] = 0.5 * (u[2] * w[0] - u[0] * w[2]);
      a[2] = 0.5 * (u[0] * w[1] - u[1] * w[0]);
      const double area = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      double n[3] = {a[0] / area, a[1] / area, a[2] / area};
      if (n[0] * fc[0] + n[1] * fc[1] + n[2] * fc[2] <= 0.0)
        for (int i = 0; i < 3; ++i) n[i] = -n[i];
      for (int i = 0; i < 3; ++i) normals[f * 3 + i] = n[i];
      fscale[f] = (area / 2.0) / det;
      taup[f] = b.tau_p;
      tauu[f] = b.tau_u;
      // neighbour across the face opposite oriented vertex f = path vertex pv
      const int pv = odd_perm(t) && (f == 1 || f == 2) ? 3 - f : f;
      const int* p = kAxisPerms[t];
      int c2[3] = {c[0], c[1], c[2]}, t2;
      if (pv == 0) {
        c2[p[0]] += 1;
        t2 = perm_index(p[1], p[2]);
      } else if (pv == 3) {
        c2[p[2]] -= 1;
        t2 = perm_index(p[2], p[0]);
      } else if (pv == 1) {
        t2 = perm_index(p[1], p[0]);
      } else {
        t2 = perm_index(p[0], p[2]);
      }
      const bool outside = c2[0] < 0 || c2[0] >= b.nx || c2[1] < 0 || c2[1] >= b.ny || c2[2] < 0 || c2[2] >= b.nz;
      if (outside) {   // boundary: self-gather, identity permutation (mesh._connectivity)
        nb[f] = (int32_t)e;
        code[f] = f | (1 << 5);
        continue;
      }
      int v2[4][3];
      tet_vertices(c2, t2, v2);
      int f2 = 0;
      for (int a2 = 0; a2 < 4; ++a2) {
        bool shared = false;
        for (int k = 0; k < 3; ++k) shared |= same(v2[a2], v[fv[k]]);
        if (!shared) f2 = a2;
      }
      int sig[3];
      for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j)
          if (same(v2[kFaceVerts[f2][j]], v[fv[k]])) sig[k] = j;
      int s = 0;
      for (int q = 0; q < 6; ++q)
        if (kPerms3[q][0] == sig[0] && kPerms3[q][1] == sig[1] && kPerms3[q][2] == sig[2]) s = q;
      code[f] = f2 | (s << 2);
      if (c2[0] < b.cx0) {          // left peer's slab
        nb[f] = 2 * (c[1] * b.nz + c[2]) + (t == 5 ? 1 : 0);
        code[f] |= 1 << 6;
      } else if (c2[0] >= b.cx1) {  // right peer's slab
        nb[f] = nleft + 2 * (c[1] * b.nz + c[2]) + t;
        code[f] |= 1 << 6;
      } else {
        nb[f] = (int32_t)((cell_lin(b, c2[0], c2[1], c2[2]) - base) * 6 + t2);
      }
    }
    pack_element<T>(rst_dx, b.kappa, b.inv_rho, normals, fscale, taup, tauu, nb, code, geo + e * kGeoRec,
                    geo_vol ? geo_vol + e * kGeoVol : nullptr, geo_surf ? geo_surf + e * kGeoSurf : nullptr,
                    nbr_out + e * 4, code_out + e);
  }
}

template <typename T> int build_box(bbdg_ctx* c, const Box& b, bool legacy, cudaStream_t s) {
  const int64_t K = c->K;
  free_geometry(c);
  cudaError_t e = cudaSuccess;
  auto alloc = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, bytes > 0 ? bytes : 16);
  };
  alloc(&c->geo, (size_t)K * kGeoRec * sizeof(T));
  if (legacy) {
    alloc(&c->geo_vol, (size_t)K * kGeoVol * sizeof(T));
    alloc(&c->geo_surf, (size_t)K * kGeoSurf * sizeof(T));
  }
  alloc(reinterpret_cast<void**>(&c->nbr), (size_t)K * 4 * sizeof(int32_t));
  alloc(reinterpret_cast<void**>(&c->code), (size_t)K * sizeof(int32_t));
  if (e != cudaSuccess) {
    free_geometry(c);
    return set_cuda_error(e, "box mesh records");
  }
  if (K > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>((K + 255) / 256, (int64_t)sms * 16);
    box_mesh_kernel<T><<<(unsigned)grid, 256, 0, s>>>(b, K, static_cast<T*>(c->geo), static_cast<T*>(c->geo_vol),
                                                      static_cast<T*>(c->geo_surf), c->nbr, c->code);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // setup call: the records are final on return
  }
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "box mesh kernel");
}

}  // namespace
}  // namespace bbdg

using namespace bbdg;

extern "C" int bbdg_ctx_set_box_mesh(bbdg_ctx* c, int nx, int ny, int nz, int cx0, int cx1, int xblock,
                                     const double* lo, const double* hi, double kappa, double rho, int legacy_records,
                                     void* stream) {
  if (!c || !lo || !hi) return set_error(BBDG_ERR_ARG, "null argument");
  if (nx < 1 || ny < 1 || nz < 1 || cx0 < 0 || cx1 > nx || cx0 >= cx1)
    return set_error(BBDG_ERR_ARG, "bad box dimensions or slab");
  if (xblock < 1 || cx0 % xblock != 0 || (cx1 % xblock != 0 && cx1 != nx))
    return set_error(BBDG_ERR_ARG, "slab layers must be multiples of the x-blocking");
  if (c->K != 6LL * (cx1 - cx0) * ny * nz) return set_error(BBDG_ERR_ARG, "context K != 6 (cx1 - cx0) ny nz");
  if (!(kappa > 0.0) || !(rho > 0.0)) return set_error(BBDG_ERR_ARG, "kappa and rho must be positive");
  if (4LL * c->K >= (1LL << 31) || 4LL * ny * nz >= (1LL << 31)) return set_error(BBDG_ERR_ARG, "box too large for int32 ids");
  Box b{};
  b.nx = nx, b.ny = ny, b.nz = nz, b.cx0 = cx0, b.cx1 = cx1, b.xb = xblock;
  const int n[3] = {nx, ny, nz};
  for (int i = 0; i < 3; ++i) {
    if (!(hi[i] > lo[i])) return set_error(BBDG_ERR_ARG, "box must have hi > lo");
    b.lo[i] = lo[i];
    b.hi[i] = hi[i];
    b.step[i] = (hi[i] - lo[i]) / n[i];
  }
  // homogeneous materials: tau_p = 1 / mean(rho c), tau_u = mean(rho c) with the neighbour's (solver.py:113-117)
  const double rc = rho * std::sqrt(kappa / rho);
  const double mean = 0.5 * (rc + rc);
  b.kappa = kappa, b.inv_rho = 1.0 / rho, b.tau_p = 1.0 / mean, b.tau_u = mean;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return c->dtype == BBDG_F32 ? build_box<float>(c, b, legacy_records != 0, s)
                              : build_box<double>(c, b, legacy_records != 0, s);
}

// Introspection for tests: copy the context's fused records (K, kGeoRec) of the context dtype,
// neighbour rows (K, 4) and packed face codes (K) to host buffers (any may be NULL).
extern "C" int bbdg_ctx_read_records(bbdg_ctx* c, void* geo, int32_t* nbr, int32_t* code) {
  if (!c || !c->geo) return set_error(BBDG_ERR_ARG, "no geometry in the context");
  const size_t sz = c->dtype == BBDG_F32 ? 4 : 8;
  cudaError_t e = cudaSuccess;
  if (geo) e = cudaMemcpy(geo, c->geo, (size_t)c->K * kGeoRec * sz, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && nbr) e = cudaMemcpy(nbr, c->nbr, (size_t)c->K * 4 * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && code) e = cudaMemcpy(code, c->code, (size_t)c->K * sizeof(int32_t), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? BBDG_OK : set_cuda_error(e, "read records");
}
