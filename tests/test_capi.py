"""The C-ABI library loads and exports every symbol include/bbdg.h declares (CPU)."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1512_06025_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "bbdg.h"


def declared_symbols():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bbdg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == decl


def test_identity_and_layout_queries():
    lib = _lib.load()
    assert lib.bbdg_version() >= 1
    assert lib.bbdg_max_degree() == 9
    for dt in (0, 1):
        for N in range(1, 10):
            ke = lib.bbdg_tile_elems(N, dt)
            Np = (N + 1) * (N + 2) * (N + 3) // 6
            assert ke >= 1
            for op, lift, basis in [(0, 1, 0), (1, 0, 0), (1, 1, 0), (1, 2, 0), (2, 0, 0), (2, 1, 0), (2, 2, 0),
                                    (3, 0, 0), (3, 1, 0), (3, 2, 0), (0, 2, 1), (1, 2, 1), (2, 2, 1), (3, 2, 1)]:
                sm = lib.bbdg_kernel_smem(N, dt, op, lift, basis)
                assert 0 < sm <= 227 * 1024, (N, dt, op, lift, basis, sm)
    assert lib.bbdg_tile_elems(10, 0) == -1


def test_error_paths_without_compute():
    lib = _lib.load()
    ctx = C.c_void_p()
    assert lib.bbdg_ctx_create(0, 0, 0, 10, C.byref(ctx)) == 2
    assert b"degree" in lib.bbdg_last_error()
    assert lib.bbdg_ctx_create(3, 7, 0, 10, C.byref(ctx)) == 1
    assert lib.bbdg_ctx_create(3, 0, 5, 10, C.byref(ctx)) == 1
    assert lib.bbdg_ctx_create(3, 0, 0, -1, C.byref(ctx)) == 1
    assert lib.bbdg_ctx_create(3, 0, 0, 48, C.byref(ctx)) == 0
    try:
        # no geometry uploaded: every compute entry point refuses
        assert lib.bbdg_volume(ctx, 1, 2, 0, None) == 2
        assert lib.bbdg_rhs(ctx, 1, 1, 0, None) == 2
        assert lib.bbdg_lsrk_update(0, 4, 1, 2, 3, 0.0, 1.0, 0.0, None) == 1    # dt <= 0
        assert lib.bbdg_lsrk_update(9, 4, 1, 2, 3, 0.0, 1.0, 1.0, None) == 1    # dtype
        assert lib.bbdg_ctx_set_halo(ctx, None, 5) == 1
    finally:
        lib.bbdg_ctx_destroy(ctx)


def test_python_layer_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1512_06025_b200 import BernsteinRefOps, Materials, WaveSystem, cube_mesh

    m = cube_mesh(1)
    with pytest.raises(_lib.BBDGError):
        WaveSystem(m, BernsteinRefOps.build(2), Materials.homogeneous(m.K))


def test_round2_entry_points_validate_without_compute():
    """Argument checks of the round-2 entry points return before any device work."""
    lib = _lib.load()
    ctx = C.c_void_p()
    assert lib.bbdg_ctx_create(3, 0, 0, 6 * 2 * 3 * 4, C.byref(ctx)) == 0
    lo, hi = (C.c_double * 3)(0, 0, 0), (C.c_double * 3)(1, 1, 1)
    try:
        assert lib.bbdg_ctx_set_box_mesh(ctx, 0, 3, 4, 0, 0, 1, lo, hi, 1.0, 1.0, 0, None) == 1      # nx < 1
        assert lib.bbdg_ctx_set_box_mesh(ctx, 2, 3, 4, 1, 1, 1, lo, hi, 1.0, 1.0, 0, None) == 1      # empty slab
        assert lib.bbdg_ctx_set_box_mesh(ctx, 3, 3, 4, 0, 3, 1, lo, hi, 1.0, 1.0, 0, None) == 1      # K mismatch
        assert lib.bbdg_ctx_set_box_mesh(ctx, 2, 3, 4, 0, 2, 1, lo, hi, -1.0, 1.0, 0, None) == 1     # kappa <= 0
        assert lib.bbdg_ctx_set_box_mesh(ctx, 2, 3, 4, 0, 2, 1, hi, lo, 1.0, 1.0, 0, None) == 1      # hi <= lo
        assert b"hi > lo" in lib.bbdg_last_error()
        assert lib.bbdg_ctx_set_box_mesh(ctx, 4, 3, 1, 1, 3, 2, lo, hi, 1.0, 1.0, 0, None) == 1   # slab not on xblock
        assert lib.bbdg_step2(ctx, 16, 32, 16, 48, 0.1, 1, None) == 2                             # no geometry
    finally:
        lib.bbdg_ctx_destroy(ctx)
    assert lib.bbdg_ops_grad(0, 0, 4, 16, 16, 16, 16, None) == 2       # degree outside 1..20
    assert lib.bbdg_ops_lift(21, 0, 4, 16, 16, None) == 2
    assert lib.bbdg_ops_grad(3, 0, 0, None, None, None, None, None) == 0   # empty batch: nothing to do
    assert lib.bbdg_dense_apply(0, 4, 0, 3, 16, 16, 16, None) == 1     # nrows < 1
    assert lib.bbdg_dense_apply(5, 4, 2, 3, 16, 16, 16, None) == 1     # dtype
