"""Drop-in solver API (reference ``/root/reference/pkg/src/bbdg/solver.py``).

``WaveSystem``, ``lsrk4_step`` and ``integrate`` keep the reference's
signatures and semantics, but every RHS evaluation and LSRK update runs in
``libbbdg_cuda.so`` (hand-written sm_100a kernels behind the C ABI of
``include/bbdg.h``).  States may be numpy arrays (copied host<->device around
each call, as a drop-in for the reference's numpy-in/numpy-out contract) or
CUDA torch tensors (device-resident; no copies).  There is no CPU fallback:
constructing a ``WaveSystem`` without the library or a CUDA device raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mesh import Mesh, build_trace_maps
from .modal import tet_rule
from .nodal import NodalRefOps, nodal_to_bernstein

# Carpenter-Kennedy five-stage LSRK4 (reference solver.py:24-51)
RK4A = np.array([0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                 -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0])
RK4B = np.array([1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                 1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                 2277821191437.0 / 14882151754819.0])
RK4C = np.array([0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                 2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0])

_SQRT3 = np.sqrt(3.0)
LIFT_MODES = ("factorized", "optimal", "dense")


def _torch():
    import torch  # plumbing only: device buffers, streams, copies

    if not torch.cuda.is_available():
        raise _lib.BBDGError("no CUDA device: the BB-DG hot path runs only on the GPU (no CPU fallback)")
    return torch


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass(frozen=True)
class Materials:
    """Piecewise-constant bulk modulus and density (reference solver.py:56-77)."""

    kappa: np.ndarray
    rho: np.ndarray

    @classmethod
    def homogeneous(cls, K: int, kappa: float = 1.0, rho: float = 1.0):
        return cls(np.full(K, float(kappa)), np.full(K, float(rho)))

    def __post_init__(self):
        if np.any(np.asarray(self.kappa) <= 0) or np.any(np.asarray(self.rho) <= 0):
            raise ValueError("kappa and rho must be positive")

    @property
    def c(self):
        return np.sqrt(self.kappa / self.rho)

    @property
    def rho_c(self):
        return self.rho * self.c


@dataclass
class FieldState:
    """Coefficients of (p, u1, u2, u3), q shape (4, K, Np): numpy or CUDA tensor."""

    q: object
    basis: str
    time: float = 0.0

    @property
    def precision(self) -> str:
        dt = self.q.dtype
        return "single" if str(dt) in ("float32", "torch.float32") else "double"

    def copy(self) -> "FieldState":
        return FieldState(self.q.clone() if _is_tensor(self.q) else self.q.copy(), self.basis, self.time)


class WaveSystem:
    """Mesh + operators + materials bound to a device context (solver.py:96-193)."""

    def __init__(self, mesh: Mesh, ops, materials: Materials, dtype=np.float64, _plan=None,
                 legacy_records: bool | None = None):
        from .mesh_device import BoxMesh

        self._box = isinstance(mesh, BoxMesh)
        if np.ndim(materials.kappa) != 0 and len(materials.kappa) != (mesh.K_total if self._box else mesh.K):
            raise ValueError("materials sized for a different mesh")
        self.mesh = mesh
        self._plan = _plan          # partition.HaloPlan for an element-partitioned rank
        self.ops_double = ops
        self.dtype = np.dtype(dtype).type
        if self.dtype not in (np.float32, np.float64):
            raise ValueError("dtype must be float32 or float64")
        self.ops = ops.astype(self.dtype)
        self.mat = materials
        self._gather = None
        if self._box:
            # device-built box (bbdg_ctx_set_box_mesh): no per-element host arrays at all
            kap, rho = np.asarray(materials.kappa, dtype=float), np.asarray(materials.rho, dtype=float)
            if np.ptp(kap) != 0 or np.ptp(rho) != 0:
                raise ValueError("a BoxMesh takes homogeneous materials")
            self._box_mat = (float(kap.flat[0]), float(rho.flat[0]))
            self._legacy = legacy_records if legacy_records is not None else mesh.K <= (1 << 22)
            self._torch = _torch()
            self._lib = _lib.load()
            self._ctx = None
            self._ctx = self._create_context(mesh, materials)
            return
        K = mesh.K
        # per-face constants exactly as the reference forms them (solver.py:113-123)
        rc = materials.rho_c
        mean_rc = 0.5 * (rc[:, None] + rc[mesh.etoe])
        self._tau_p64 = np.ascontiguousarray(1.0 / mean_rc)
        self._tau_u64 = np.ascontiguousarray(mean_rc)
        self._fscale64 = np.ascontiguousarray(mesh.jf / mesh.jac[:, None])
        self.tau_p = self._tau_p64.astype(self.dtype)[:, :, None]
        self.tau_u = self._tau_u64.astype(self.dtype)[:, :, None]
        self.face_scale = self._fscale64.astype(self.dtype)[:, :, None]
        self.normals = mesh.normals.astype(self.dtype)
        self.rst_dx = mesh.rst_dx.astype(self.dtype)
        self.kappa = materials.kappa.astype(self.dtype)[:, None]
        self.inv_kappa = (1.0 / materials.kappa).astype(self.dtype)[:, None]
        self.inv_rho = (1.0 / materials.rho).astype(self.dtype)[:, None]
        if _plan is not None:
            sl = slice(_plan.k0, _plan.k1)
            for name in ("tau_p", "tau_u", "face_scale", "normals", "rst_dx", "kappa", "inv_kappa", "inv_rho"):
                setattr(self, name, getattr(self, name)[sl])
            self._tau_p64, self._tau_u64, self._fscale64 = (self._tau_p64[sl], self._tau_u64[sl],
                                                            self._fscale64[sl])
        self._torch = _torch()
        self._lib = _lib.load()
        self._ctx = None
        self._ctx = self._create_context(mesh, materials)

    # ---------------------------------------------------------------- context
    def _create_context(self, mesh: Mesh, materials: Materials):
        L = self._lib
        ctx = C.c_void_p()
        _lib.check(L.bbdg_ctx_create(self.ops.N, _lib.BASIS[self.basis], _lib.DTYPE[np.dtype(self.dtype).name],
                                     self.K, C.byref(ctx)), "bbdg_ctx_create")
        self._ctx = ctx   # owned from here on (released by __del__ if a later upload raises)
        if self._box:
            b = mesh
            lo, hi = (C.c_double * 3)(*b.lo), (C.c_double * 3)(*b.hi)
            _lib.check(L.bbdg_ctx_set_box_mesh(ctx, b.nx, b.ny, b.nz, b.cx0, b.cx1, b.xblock, lo, hi, self._box_mat[0],
                                               self._box_mat[1], int(self._legacy), self._stream()),
                       "bbdg_ctx_set_box_mesh")
            self._upload_operators(ctx)
            return ctx
        if self._plan is None:
            sl = slice(0, mesh.K)
            nbr, code = mesh.face_codes()
        else:
            sl = slice(self._plan.k0, self._plan.k1)
            nbr, code = self._plan.nbr, self._plan.code
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (mesh.rst_dx[sl], materials.kappa[sl], 1.0 / materials.rho[sl], mesh.normals[sl],
                 self._fscale64, self._tau_p64, self._tau_u64)]
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        code = np.ascontiguousarray(code, dtype=np.int8)
        _lib.check(L.bbdg_ctx_set_geometry(ctx, *[a.ctypes.data for a in arrs], nbr.ctypes.data, code.ctypes.data),
                   "bbdg_ctx_set_geometry")
        self._upload_operators(ctx)
        return ctx

    def _upload_operators(self, ctx):
        L = self._lib
        if self.basis == "bernstein":
            cols, vals = self.ops_double.el_ell()
            dl = np.ascontiguousarray(self.ops_double.dense_L)
            _lib.check(L.bbdg_ctx_set_lift_tables(ctx, cols.ctypes.data, vals.ctypes.data, cols.shape[1],
                                                  dl.ctypes.data), "bbdg_ctx_set_lift_tables")
        else:
            o = self.ops_double
            D = [np.ascontiguousarray(x, dtype=np.float64) for x in (o.Dr, o.Ds, o.Dt)]
            dl = np.ascontiguousarray(o.dense_L, dtype=np.float64)
            _lib.check(L.bbdg_ctx_set_nodal_ops(ctx, *[d.ctypes.data for d in D]), "bbdg_ctx_set_nodal_ops")
            _lib.check(L.bbdg_ctx_set_lift_tables(ctx, None, None, 0, dl.ctypes.data), "bbdg_ctx_set_lift_tables")

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and _lib._lib is not None:
            _lib._lib.bbdg_ctx_destroy(ctx)
            self._ctx = None

    @property
    def basis(self) -> str:
        return self.ops.basis

    @property
    def K(self) -> int:
        """Elements this system updates (the rank's slab for a partitioned system)."""
        return self.mesh.K if self._plan is None or self._box else self._plan.n_local

    @property
    def Np(self) -> int:
        return self.ops.Np

    @property
    def gather(self):
        """Reference-layout flat neighbour gather (K,4,Nfp), built on demand."""
        if self._gather is None:
            self._gather = build_trace_maps(self.mesh, self.ops.trace, self.ops.Np)
        return self._gather[0]

    @property
    def boundary(self):
        return self.mesh.boundary

    @property
    def torch_dtype(self):
        t = self._torch
        return t.float32 if self.dtype == np.float32 else t.float64

    def _stream(self):
        return self._torch.cuda.current_stream().cuda_stream

    # ---------------------------------------------------------------- marshalling
    def _check(self, state: FieldState):
        if state.basis != self.basis:
            raise ValueError(f"state basis {state.basis!r} does not match {self.basis!r}")
        if tuple(state.q.shape) != (4, self.K, self.ops.Np):
            raise ValueError("state shaped for a different system")

    def to_device(self, q):
        """Device tensor view/copy of q in the system dtype (H2D for numpy)."""
        t = self._torch
        if _is_tensor(q):
            if not q.is_cuda:
                q = q.cuda()
            if q.dtype != self.torch_dtype:
                q = q.to(self.torch_dtype)
            return q.contiguous()
        a = np.ascontiguousarray(q, dtype=self.dtype)
        return t.from_numpy(a).to("cuda")

    def empty_state(self):
        return self._torch.empty((4, self.K, self.ops.Np), dtype=self.torch_dtype, device="cuda")

    def _out(self, dq, like):
        return dq if _is_tensor(like) else dq.cpu().numpy()

    @staticmethod
    def _lift_id(lift_mode):
        if lift_mode not in _lib.LIFT:
            raise ValueError(f"unknown lift mode {lift_mode!r}")
        return _lib.LIFT[lift_mode]

    # ---------------------------------------------------------------- device entry points
    def volume_into(self, q, out, accumulate=False):
        _lib.check(self._lib.bbdg_volume(self._ctx, q.data_ptr(), out.data_ptr(), int(accumulate), self._stream()),
                   "bbdg_volume")

    def surface_into(self, q, out, lift_mode="factorized", accumulate=False):
        _lib.check(self._lib.bbdg_surface(self._ctx, q.data_ptr(), out.data_ptr(), self._lift_id(lift_mode),
                                          int(accumulate), self._stream()), "bbdg_surface")

    def rhs_into(self, q, out, lift_mode="factorized"):
        _lib.check(self._lib.bbdg_rhs(self._ctx, q.data_ptr(), out.data_ptr(), self._lift_id(lift_mode),
                                      self._stream()), "bbdg_rhs")

    def stage_into(self, q_in, q_out, res, a, b, dt, lift_mode="factorized"):
        _lib.check(self._lib.bbdg_lsrk_stage(self._ctx, q_in.data_ptr(), q_out.data_ptr(), res.data_ptr(),
                                             self._lift_id(lift_mode), float(a), float(b), float(dt),
                                             self._stream()), "bbdg_lsrk_stage")

    def stage_range_into(self, q_in, q_out, res, a, b, dt, lift_mode, k0, k1):
        _lib.check(self._lib.bbdg_lsrk_stage_range(self._ctx, q_in.data_ptr(), q_out.data_ptr(), res.data_ptr(),
                                                   self._lift_id(lift_mode), float(a), float(b), float(dt),
                                                   int(k0), int(k1), self._stream()), "bbdg_lsrk_stage_range")

    def halo_pack(self, q, faces, out):
        """bbdg_halo_pack: traces of (elem, face) pairs -> out (4, n, Nfp)."""
        if faces.shape[0] == 0:
            return
        _lib.check(self._lib.bbdg_halo_pack(self._ctx, q.data_ptr(), out.data_ptr(), faces.data_ptr(),
                                            int(faces.shape[0]), self._stream()), "bbdg_halo_pack")

    def set_halo(self, halo, nhalo):
        _lib.check(self._lib.bbdg_ctx_set_halo(self._ctx, halo.data_ptr() if nhalo else None, int(nhalo)),
                   "bbdg_ctx_set_halo")

    def step_into(self, q, q_tmp, res, dt, lift_mode="factorized", q_tmp2=None):
        """Five fused stages in place on q (bbdg_step2: with q_tmp2 the last stage writes q)."""
        _lib.check(self._lib.bbdg_step2(self._ctx, q.data_ptr(), q_tmp.data_ptr(),
                                        q_tmp2.data_ptr() if q_tmp2 is not None else None, res.data_ptr(),
                                        float(dt), self._lift_id(lift_mode), self._stream()), "bbdg_step2")

    def scratch(self, like, n=2):
        """n cached (4,K,Np) device scratch buffers shaped like `like` (reused across steps)."""
        key = (like.dtype, like.device, n)
        buf = getattr(self, "_scratch", None)
        if buf is None or buf[0] != key:
            t = self._torch
            buf = (key, [t.empty_like(like) for _ in range(n)])
            self._scratch = buf
        return buf[1]

    # ---------------------------------------------------------------- reference API
    def volume_rhs(self, state: FieldState):
        self._check(state)
        q = self.to_device(state.q)
        dq = self._torch.empty_like(q)
        self.volume_into(q, dq)
        return self._out(dq, state.q)

    def _nodal_mode(self, lift_mode):
        """The reference forces "dense" for the nodal basis (solver.py:168-169); "blocked" picks the
        block-partitioned tensor-core kernels for the same arithmetic."""
        if self.basis == "nodal":
            return "blocked" if lift_mode == "blocked" else "dense"
        if lift_mode == "blocked":
            raise ValueError("lift mode 'blocked' is nodal-only")
        return lift_mode

    def surface_rhs(self, state: FieldState, lift_mode: str = "factorized"):
        self._check(state)
        lift_mode = self._nodal_mode(lift_mode)
        self._lift_id(lift_mode)
        q = self.to_device(state.q)
        dq = self._torch.empty_like(q)
        self.surface_into(q, dq, lift_mode)
        return self._out(dq, state.q)

    def rhs(self, state: FieldState, lift_mode: str = "factorized"):
        self._check(state)
        lift_mode = self._nodal_mode(lift_mode)
        self._lift_id(lift_mode)
        q = self.to_device(state.q)
        dq = self._torch.empty_like(q)
        self.rhs_into(q, dq, lift_mode)
        return self._out(dq, state.q)


def _copy_back(dst, src_dev):
    """Write a device result into the caller's array in place (numpy or tensor)."""
    if _is_tensor(dst):
        if dst.data_ptr() != src_dev.data_ptr():
            dst.copy_(src_dev)
    elif dst.flags.c_contiguous and dst.flags.writeable and dst.dtype.name == str(src_dev.dtype).split(".")[-1]:
        import torch

        torch.from_numpy(dst).copy_(src_dev)        # D2H straight into the caller's array
    else:
        dst[...] = src_dev.cpu().numpy()


def _device_update(q_dev, res_dev, k_dev, a, b, dt):
    lib = _lib.load()
    import torch

    dt_id = 0 if q_dev.dtype == torch.float32 else 1
    _lib.check(lib.bbdg_lsrk_update(dt_id, q_dev.numel(), q_dev.data_ptr(), res_dev.data_ptr(), k_dev.data_ptr(),
                                    float(a), float(b), float(dt), torch.cuda.current_stream().cuda_stream),
               "bbdg_lsrk_update")


def host_chunk_plan(etoe, Np: int, itemsize: int, max_chunks: int = 32, min_state_bytes: int = 32 << 20,
                    chunk: int | None = None):
    """Element chunks for the host-pipelined step (``bbdg_step_host``): (bounds, reach) or None.

    Chunks are at least as long as the largest neighbour-index distance of the
    mesh (so a banded numbering such as cube_mesh's x-slabs gives reach 1) and
    at most ``max_chunks`` of them (32: measured on cube_mesh(40), fp32, the sum of the
    N=2..9 step times is 117.6 ms at 32 chunks, 119.3 at 24, 124.5 at 40, tools/e2e_chunks.py); ``reach`` is the exact largest chunk distance
    between an element and any neighbour.  None when the state is too small for
    chunking to pay, or the numbering is not banded enough to pipeline.
    """
    etoe = np.asarray(etoe)
    K = etoe.shape[0]
    if 4 * K * Np * itemsize < min_state_bytes:
        return None
    idx = np.arange(K, dtype=np.int64)[:, None]
    band = int(np.abs(etoe.astype(np.int64) - idx).max()) if K else 0
    csize = chunk if chunk is not None else max(band, -(-K // max_chunks), 1)
    nch = -(-K // csize)
    if nch < 3:
        return None
    cid = etoe.astype(np.int64) // csize
    own = idx // csize
    reach = int(np.abs(cid - own).max())
    if 4 * (reach + 1) >= nch:   # pipeline fill longer than the work: nothing overlaps
        return None
    bounds = np.minimum(np.arange(nch + 1, dtype=np.int64) * csize, K)
    return bounds, reach


def _copy_threads() -> int:
    n = os.environ.get("BBDG_COPY_THREADS")
    return max(1, int(n)) if n else max(1, min(8, (os.cpu_count() or 2) // 2))


def _host_step(system: "WaveSystem", q_host: np.ndarray, dt: float, lift: str) -> bool:
    """Pipelined H2D + five stages + D2H of a host state; False if not applicable.

    A pinned array (e.g. ``torch.empty(..., pin_memory=True).numpy()``) is copied directly by
    ``bbdg_step_host``; an ordinary pageable array of at least 4 MB goes through the context's
    pinned staging rings, filled and drained by host threads (``bbdg_step_pageable``), so that
    the host copies, both PCIe directions and the stages of other chunks overlap.
    """
    if system._plan is not None or system._box or not isinstance(q_host, np.ndarray) or not q_host.flags.c_contiguous \
            or not q_host.flags.writeable or q_host.dtype != np.dtype(system.dtype):
        return False
    torch = _torch()
    pinned = torch.from_numpy(q_host).is_pinned()
    if not pinned and q_host.nbytes < (4 << 20):
        return False   # small: the plain copy path
    if not hasattr(system, "_chunks"):
        etoe = system.mesh.etoe
        if _is_tensor(etoe):
            etoe = etoe.cpu().numpy()
        system._chunks = host_chunk_plan(etoe, system.ops.Np, np.dtype(system.dtype).itemsize)
    if system._chunks is None:
        return False
    bounds, reach = system._chunks
    if not hasattr(system, "_copy_streams"):
        system._copy_streams = (torch.cuda.Stream(), torch.cuda.Stream())
    hs, ds = system._copy_streams
    q = system.empty_state()
    tmp, r = torch.empty_like(q), torch.empty_like(q)
    cs = torch.cuda.current_stream()
    if pinned:
        _lib.check(system._lib.bbdg_step_host(system._ctx, q_host.ctypes.data, q.data_ptr(), tmp.data_ptr(),
                                              r.data_ptr(), float(dt), system._lift_id(lift), bounds.ctypes.data,
                                              len(bounds) - 1, int(reach), cs.cuda_stream, hs.cuda_stream,
                                              ds.cuda_stream), "bbdg_step_host")
        cs.synchronize()   # host_q holds the new state (reference: in place on return)
    else:
        _lib.check(system._lib.bbdg_step_pageable(system._ctx, q_host.ctypes.data, q.data_ptr(), tmp.data_ptr(),
                                                  r.data_ptr(), float(dt), system._lift_id(lift), bounds.ctypes.data,
                                                  len(bounds) - 1, int(reach), 3, _copy_threads(), cs.cuda_stream,
                                                  hs.cuda_stream, ds.cuda_stream), "bbdg_step_pageable")
    return True


def lsrk4_step(system, state: FieldState, dt: float, lift_mode: str = "factorized", res=None) -> FieldState:
    """One five-stage LSRK4 step, in place on state.q (reference solver.py:196-214).

    A ``WaveSystem`` runs the five fused stage kernels on the device.  Any
    other object with ``.rhs(state, lift_mode)`` (duck typing, as the
    reference's own tests use) gets the stand-alone CUDA update kernel.
    """
    if dt <= 0:
        raise ValueError("dt must be positive")
    torch = _torch()
    t0 = state.time
    if isinstance(system, WaveSystem):
        system._check(state)
        lift = system._nodal_mode(lift_mode)
        system._lift_id(lift)
        # numpy state, fresh res: copies in both directions overlap the stages chunk by chunk
        if res is None and _host_step(system, state.q, dt, lift):
            return FieldState(state.q, state.basis, t0 + dt)
        q = system.to_device(state.q)
        r = system.to_device(res) if res is not None else torch.empty_like(q)
        t1, t2 = system.scratch(q)
        system.step_into(q, t1, r, dt, lift, q_tmp2=t2)   # the fifth stage writes q: no final copy
        _copy_back(state.q, q)
        if res is not None:
            _copy_back(res, r)
        return FieldState(state.q, state.basis, t0 + dt)
    # duck-typed system: the system's rhs, the update on the device (no CPU arithmetic on it)
    host = not (_is_tensor(state.q) and state.q.is_cuda)
    if _is_tensor(state.q):
        q = state.q.cuda().contiguous() if host else state.q
    else:
        q = torch.from_numpy(np.ascontiguousarray(state.q)).cuda()
    r = torch.zeros_like(q)
    work = FieldState(state.q, state.basis, t0)
    for s in range(5):
        work.time = t0 + RK4C[s] * dt
        k = system.rhs(work, lift_mode)
        kd = torch.as_tensor(np.asarray(k) if not _is_tensor(k) else k).to(device=q.device, dtype=q.dtype)
        _device_update(q, r, kd.contiguous(), RK4A[s], RK4B[s], dt)
        if host:
            if _is_tensor(state.q):
                state.q.copy_(q)
            else:
                state.q[...] = q.cpu().numpy()
    if res is not None:
        _copy_back(res, r)
    return FieldState(state.q, state.basis, t0 + dt)


def integrate(system, state: FieldState, dt: float, nsteps: int, lift_mode: str = "factorized", callback=None,
              energy_guard: float | None = 10.0) -> FieldState:
    """March nsteps with the state resident on the device (reference solver.py:217-239).

    The five stages of each step ping-pong between two device buffers; the
    host sees the state only for callbacks and the energy guard (every 20
    steps), and the caller's array is updated in place at the end.
    """
    if not isinstance(system, WaveSystem):
        # any object with .rhs (reference solver.py:217-239, including its energy guard)
        res = np.zeros_like(state.q) if not _is_tensor(state.q) else state.q.new_zeros(state.q.shape)
        e0 = discrete_energy(system, state) if energy_guard else None
        if callback:
            callback(0, state)
        for step in range(1, nsteps + 1):
            state = lsrk4_step(system, state, dt, lift_mode, res)
            if callback:
                callback(step, state)
            if energy_guard and step % 20 == 0:
                e = discrete_energy(system, state)
                if e > energy_guard * max(e0, 1e-300):
                    raise RuntimeError(f"unstable run: energy grew from {e0:.3e} to {e:.3e} by step {step}")
        return state
    if dt <= 0:
        raise ValueError("dt must be positive")
    system._check(state)
    torch = _torch()
    lift = system._nodal_mode(lift_mode)
    system._lift_id(lift)
    host = not _is_tensor(state.q)
    bufs = [system.to_device(state.q), None]
    bufs[1] = torch.empty_like(bufs[0])
    res = torch.zeros_like(bufs[0])
    cur = 0
    e0 = discrete_energy(system, state) if energy_guard else None
    if callback:
        callback(0, state)
    t = state.time
    for step in range(1, nsteps + 1):
        res.zero_()
        for s in range(5):
            system.stage_into(bufs[cur], bufs[cur ^ 1], res, RK4A[s], RK4B[s], dt, lift)
            cur ^= 1
        t = t + dt
        if callback or (energy_guard and step % 20 == 0):
            view = FieldState(bufs[cur], state.basis, t)
            if callback:
                cb_state = FieldState(bufs[cur].cpu().numpy(), state.basis, t) if host else view
                callback(step, cb_state)
            if energy_guard and step % 20 == 0:
                e = discrete_energy(system, view)
                if e > energy_guard * max(e0, 1e-300):
                    _copy_back(state.q, bufs[cur])
                    raise RuntimeError(f"unstable run: energy grew from {e0:.3e} to {e:.3e} by step {step}")
    _copy_back(state.q, bufs[cur])
    return FieldState(state.q, state.basis, t)


def stable_dt(mesh: Mesh, N: int, c_max: float, cfl: float = 0.5) -> float:
    """dt = cfl h_min / (c_max N^2) (reference solver.py:242-246)."""
    if not 0.0 < cfl <= 1.0:
        raise ValueError("cfl must lie in (0, 1]")
    return cfl * mesh.h_min / (c_max * N * N)


def exact_solution(xyz, tau: float):
    """Standing wave on [-1/2,1/2]^3, rho = kappa = 1 (reference solver.py:249-261)."""
    xyz = np.asarray(xyz)
    cx, cy, cz = (np.cos(np.pi * xyz[..., i]) for i in range(3))
    sx, sy, sz = (np.sin(np.pi * xyz[..., i]) for i in range(3))
    p = cx * cy * cz * np.cos(_SQRT3 * np.pi * tau)
    amp = np.sin(_SQRT3 * np.pi * tau) / _SQRT3
    return p, np.stack([sx * cy * cz * amp, cx * sy * cz * amp, cx * cy * sz * amp])


def initial_state(mesh: Mesh, N: int, basis: str, dtype=np.float64, node_kind: str = "warp_blend",
                  tau: float = 0.0) -> FieldState:
    """Nodal interpolation of the exact solution, converted in float64 (solver.py:264-279)."""
    nops = NodalRefOps.build(N, node_kind)
    p, u = exact_solution(mesh.map_reference_points(nops.nodes), tau)
    q = np.stack([p, u[0], u[1], u[2]])
    if basis == "bernstein":
        q = nodal_to_bernstein(nops, q)
    elif basis != "nodal":
        raise ValueError(f"unknown basis {basis!r}")
    return FieldState(q.astype(dtype), basis, tau)


def initial_state_device(mesh: Mesh, N: int, basis: str, dtype=np.float64, node_kind: str = "warp_blend",
                         tau: float = 0.0, chunk: int = 1 << 22) -> FieldState:
    """initial_state (solver.py:264-279) evaluated on the device by bbdg_project_standing_wave:
    the state is born in HBM (a CUDA tensor), nothing of size K x Np is formed on the host."""
    torch = _torch()
    from .multiindex import barycentric_from_rst

    nops = NodalRefOps.build(N, node_kind)
    if basis == "bernstein":
        tm = nops.to_bernstein
    elif basis == "nodal":
        tm = np.eye(nops.Np)
    else:
        raise ValueError(f"unknown basis {basis!r}")
    f64 = dict(dtype=torch.float64, device="cuda")
    tmd = torch.as_tensor(np.array(tm, dtype=np.float64), **f64)
    lam = torch.as_tensor(np.ascontiguousarray(barycentric_from_rst(nops.nodes)), **f64)
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    K, Np = mesh.K, nops.Np
    q = torch.empty((4, K, Np), dtype=tdt, device="cuda")
    lib = _lib.load()
    tets = mesh.tets
    for k0 in range(0, K, chunk):
        k1 = min(K, k0 + chunk)
        verts = torch.as_tensor(np.ascontiguousarray(mesh.vertices[tets[k0:k1]]), **f64)
        part = torch.empty((4, k1 - k0, Np), dtype=tdt, device="cuda")
        _lib.check(lib.bbdg_project_standing_wave(0 if tdt == torch.float32 else 1, k1 - k0, Np, tmd.data_ptr(),
                                                  lam.data_ptr(), verts.data_ptr(), float(tau), part.data_ptr(),
                                                  torch.cuda.current_stream().cuda_stream),
                   "bbdg_project_standing_wave")
        q[:, k0:k1] = part
    return FieldState(q, basis, tau)


class ErrorFunctional:
    """Quadrature of (p_h - p)^2 with a degree 2N+2 rule (solver.py:282-296).

    Device states are evaluated by the bbdg_error_l2 kernel (no host copy); numpy
    states by the same float64 arithmetic on the host, as the reference does."""

    def __init__(self, mesh: Mesh, ops):
        pts, w = tet_rule(2 * ops.N + 2)
        self.w = w
        self.pts = pts
        self.mesh = mesh
        self.phys = mesh.map_reference_points(pts)
        self.E = ops.eval_matrix(pts)
        self.jac = mesh.jac
        self._dev = None

    def _device_arrays(self, device):
        if self._dev is None:
            torch = _torch()
            from .multiindex import barycentric_from_rst

            f64 = dict(dtype=torch.float64, device=device)
            self._dev = dict(
                ET=torch.as_tensor(np.ascontiguousarray(self.E.T), **f64),
                w=torch.as_tensor(np.ascontiguousarray(self.w), **f64),
                lam=torch.as_tensor(np.ascontiguousarray(barycentric_from_rst(self.pts)), **f64),
                verts=torch.as_tensor(np.ascontiguousarray(self.mesh.element_vertices()), **f64),
                jac=torch.as_tensor(np.ascontiguousarray(self.jac), **f64),
                partial=torch.empty(len(self.jac), **f64), out=torch.empty(1, **f64))
        return self._dev

    def device(self, q, tau: float) -> float:
        """Error of a device state q (4, K, Np) at time tau (one D2H of 8 bytes)."""
        torch = _torch()
        d = self._device_arrays(q.device)
        K, Np = q.shape[1], q.shape[2]
        lib = _lib.load()
        _lib.check(lib.bbdg_error_l2(0 if q.dtype == torch.float32 else 1, K, Np, len(self.w), q.data_ptr(),
                                     d["ET"].data_ptr(), d["w"].data_ptr(), d["lam"].data_ptr(),
                                     d["verts"].data_ptr(), d["jac"].data_ptr(), float(tau),
                                     d["partial"].data_ptr(), d["out"].data_ptr(),
                                     torch.cuda.current_stream().cuda_stream), "bbdg_error_l2")
        return float(d["out"].item())

    def __call__(self, state: FieldState) -> float:
        if _is_tensor(state.q) and state.q.is_cuda:
            return self.device(state.q.contiguous(), state.time)
        q0 = state.q[0]
        q0 = q0.double().cpu().numpy() if _is_tensor(q0) else np.asarray(q0, dtype=np.float64)
        ph = q0 @ self.E.T
        p, _ = exact_solution(self.phys, state.time)
        return float(np.sqrt((((ph - p) ** 2) @ self.w) @ self.jac))


def l2_error(system: WaveSystem, state: FieldState, functional: ErrorFunctional | None = None) -> float:
    if functional is None:
        functional = ErrorFunctional(system.mesh, system.ops_double)
    return functional(state)


def discrete_energy(system: WaveSystem, state: FieldState) -> float:
    """sum_k J_k [p^T M p / kappa + rho sum_i u_i^T M u_i] (solver.py:306-312).

    Device states: the bbdg_energy kernel (float64 accumulation, deterministic)."""
    M = system.ops_double.mass
    if _is_tensor(state.q) and state.q.is_cuda:
        torch = _torch()
        q = state.q.contiguous()
        d = getattr(system, "_energy_dev", None)
        if d is None or d["M"].device != q.device:
            f64 = dict(dtype=torch.float64, device=q.device)
            sl = slice(None) if system._plan is None else slice(system._plan.k0, system._plan.k1)
            if getattr(system, "_box", False):
                jac = np.full(system.K, system.mesh.cell_jac)
                kap, rho = system._box_mat
            else:
                jac = system.mesh.jac[sl]
                kap, rho = system.mat.kappa[sl], system.mat.rho[sl]
            coef = np.stack([jac / kap] + [jac * rho] * 3)
            d = dict(M=torch.as_tensor(np.array(M, dtype=np.float64), **f64),
                     coef=torch.as_tensor(np.ascontiguousarray(coef), **f64),
                     partial=torch.empty(q.shape[1], **f64), out=torch.empty(1, **f64))
            system._energy_dev = d
        lib = _lib.load()
        _lib.check(lib.bbdg_energy(0 if q.dtype == torch.float32 else 1, q.shape[1], q.shape[2], q.data_ptr(),
                                   d["M"].data_ptr(), d["coef"].data_ptr(), d["partial"].data_ptr(),
                                   d["out"].data_ptr(), torch.cuda.current_stream().cuda_stream), "bbdg_energy")
        return float(d["out"].item())
    # host arrays / CPU tensors: the reference's float64 formula on the host (solver.py:306-312)
    q = state.q.double().numpy() if _is_tensor(state.q) else np.asarray(state.q, dtype=np.float64)
    quad = np.einsum("fkn,nm,fkm->fk", q, M, q)
    return float(((quad[0] / system.mat.kappa + system.mat.rho * quad[1:].sum(axis=0)) * system.mesh.jac).sum())


def _degree_from_block(Np: int) -> int:
    N = 1
    while (N + 1) * (N + 2) * (N + 3) // 6 < Np:
        N += 1
    if (N + 1) * (N + 2) * (N + 3) // 6 != Np:
        raise ValueError(f"block length {Np} is not a tetrahedral space dimension")
    return N


def save_state(path, state: FieldState):
    """One-line text header + raw (4,K,Np) bytes (reference solver.py:324-332)."""
    q = state.q.cpu().numpy() if _is_tensor(state.q) else np.asarray(state.q)
    header = (f"bbdg-state degree={_degree_from_block(q.shape[2])} K={q.shape[1]} "
              f"basis={state.basis} precision={state.precision} time={state.time!r}\n")
    with open(path, "wb") as fh:
        fh.write(header.encode())
        fh.write(np.ascontiguousarray(q).tobytes())


def load_state(path) -> FieldState:
    with open(path, "rb") as fh:
        header = fh.readline().decode()
        raw = fh.read()
    fields = dict(tok.split("=") for tok in header.split()[1:])
    N, K = int(fields["degree"]), int(fields["K"])
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    dtype = np.float32 if fields["precision"] == "single" else np.float64
    q = np.frombuffer(raw, dtype=dtype).reshape(4, K, Np).copy()
    return FieldState(q, fields["basis"], float(fields["time"]))
