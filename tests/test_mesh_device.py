"""The vectorised device mesh builder reproduces mesh.box_mesh."""

import numpy as np
import pytest

from paper_1512_06025_b200.mesh import box_mesh
from paper_1512_06025_b200.mesh_device import box_mesh_device

INTS = ("tets", "etoe", "etof", "face_perm")
FLOATS = ("vertices", "jac", "rst_dx", "normals", "jf", "h_elem")


def _same(a, b):
    for k in INTS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    for k in FLOATS:
        x, y = getattr(a, k), getattr(b, k)
        assert np.abs(x - y).max() <= 2e-15 * np.abs(x).max(), k   # det / inv rounding (LAPACK vs torch)


@pytest.mark.parametrize("dims", [(1, 1, 1), (3, 3, 3), (5, 2, 4), (2, 7, 3)])
def test_device_builder_matches_host_builder_cpu(dims):
    _same(box_mesh(*dims, lo=(-1, 0, 0.5), hi=(2, 1, 3)), box_mesh_device(*dims, lo=(-1, 0, 0.5), hi=(2, 1, 3),
                                                                          device="cpu"))


@pytest.mark.gpu
def test_device_builder_matches_host_builder_gpu():
    _same(box_mesh(24, 16, 20), box_mesh_device(24, 16, 20, device="cuda"))
