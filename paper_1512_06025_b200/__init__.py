"""B200-native BB-DG acoustic-wave hot path (arXiv 1512.06025).

Drop-in for the reference ``bbdg`` package's per-timestep RHS evaluation and
LSRK4 update: same Python API (mesh / operator setup, ``WaveSystem``,
``lsrk4_step``, ``integrate``, ``FieldState``), with every hot-path operation
executed by hand-written sm_100a CUDA kernels in ``libbbdg_cuda.so`` behind
the C ABI of ``include/bbdg.h``.
"""

from .bernstein import BernsteinRefOps
from .mesh import Mesh, build_trace_maps, cube_mesh, from_arrays, load_mesh_ascii, save_mesh_ascii
from .nodal import NodalRefOps, bernstein_to_nodal, nodal_to_bernstein
from .solver import (
    ErrorFunctional,
    FieldState,
    Materials,
    WaveSystem,
    discrete_energy,
    exact_solution,
    initial_state,
    initial_state_device,
    integrate,
    l2_error,
    load_state,
    lsrk4_step,
    save_state,
    stable_dt,
)

__version__ = "0.1.0"
