"""Operator-level drop-in API on the device (reference bernstein.py:301-329,436-466,
nodal.py:220-241, opcount.py:38-43): ops.grad / ops.lift_flux / lift_apply_factorized /
lift_apply_optimal / SparseRowOperator.apply, against the pinned oracle's tables."""

import numpy as np
import pytest

import bbdg_oracle as orc
from conftest import TOL, rel_l2
from paper_1512_06025_b200 import BernsteinRefOps, NodalRefOps
from paper_1512_06025_b200.bernstein import build_lift, derivative_ops, lift_apply_factorized, lift_apply_optimal

pytestmark = pytest.mark.gpu
DT = {"f64": np.float64, "f32": np.float32}


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_bernstein_grad_and_lift_match_oracle(N, dname):
    dtype = DT[dname]
    ops, tab = BernsteinRefOps.build(N), orc.bernstein_tables(N)
    rng = np.random.default_rng(500 + N)
    q = rng.standard_normal((37, ops.Np)).astype(dtype)
    got = ops.grad(q)
    want = tab.grad(q)
    for g, w in zip(got, want):
        assert g.dtype == dtype and g.shape == q.shape
        assert rel_l2(g, w) < TOL[dname]
    flux = rng.standard_normal((3, 5, 4, ops.Nfp)).astype(dtype)
    for mode in ("factorized", "optimal", "dense"):
        out = ops.lift_flux(flux, mode)
        assert out.shape == (3, 5, ops.Np) and out.dtype == dtype
        tol = TOL[dname] if mode != "dense" else max(TOL[dname], 1e-11)
        assert rel_l2(out, tab.lift(flux, mode, dtype)) < tol, mode
    lf = build_lift(N)
    assert rel_l2(lift_apply_factorized(lf, flux), tab.lift(flux, "factorized", dtype)) < TOL[dname]
    assert rel_l2(lift_apply_optimal(lf, flux), tab.lift(flux, "optimal", dtype)) < TOL[dname]
    with pytest.raises(ValueError):
        ops.lift_flux(flux, "bogus")
    with pytest.raises(ValueError):
        lift_apply_optimal(lf, flux[..., :-1])


def test_device_tensors_in_and_out():
    import torch

    ops = BernsteinRefOps.build(4)
    q = torch.randn((8, ops.Np), dtype=torch.float64, device="cuda")
    d = ops.grad(q)
    assert all(x.is_cuda for x in d)
    assert rel_l2(d[0].cpu().numpy(), ops.grad(q.cpu().numpy())[0]) == 0.0
    flux = torch.randn((6, 4, ops.Nfp), dtype=torch.float32, device="cuda")
    out = ops.lift_flux(flux)
    assert out.is_cuda and out.dtype == torch.float32


def test_sparse_row_operator_apply():
    ds = derivative_ops(3)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((10, 20))
    for op in ds.ops:
        assert rel_l2(op.apply(x), x @ op.toarray().T) < 1e-14
    lf = build_lift(5)
    v = rng.standard_normal((7, lf.Nfp))
    assert rel_l2(lf.L0.apply(v), v @ lf.L0.toarray().T) < 1e-14


@pytest.mark.parametrize("N", [1, 4, 9])
def test_nodal_grad_and_lift(N):
    ops = NodalRefOps.build(N)
    rng = np.random.default_rng(N)
    q = rng.standard_normal((11, ops.Np))
    for g, D in zip(ops.grad(q), (ops.Dr, ops.Ds, ops.Dt)):
        assert rel_l2(g, q @ D.T) < 1e-13
    flux = rng.standard_normal((2, 4, ops.Nfp))
    assert rel_l2(ops.lift_flux(flux), flux.reshape(2, -1) @ ops.dense_L.T) < 1e-13
    with pytest.raises(ValueError):
        ops.lift_flux(flux, "optimal")
