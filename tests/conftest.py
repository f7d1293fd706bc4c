import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libbbdg_cuda.so")
    config.addinivalue_line("markers", "slow: long-running")


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


# parity tolerances (relative L2), per the north star: 1e-12 fp64, ~1e-5 fp32
TOL = {"f64": 1e-12, "f32": 1e-5}


@pytest.fixture(scope="session")
def golden_bb():
    return dict(np.load(GOLDEN / "golden_bb.npz"))


@pytest.fixture(scope="session")
def golden_nodal():
    return dict(np.load(GOLDEN / "golden_nodal.npz"))


@pytest.fixture(scope="session")
def golden_c1():
    return dict(np.load(GOLDEN / "golden_c1.npz"))


@pytest.fixture(scope="session")
def golden_setup():
    return dict(np.load(GOLDEN / "golden_setup.npz"))
