"""Build libbbdg_cuda.so in-tree for sm_100a (nvcc, parallel per-degree units).

    python -m paper_1512_06025_b200.build [-j JOBS] [--force]

The instantiation unit ``csrc/bbdg_kernels.cu`` is compiled once per
(dtype, degree); ``bbdg_capi.cu`` holds the C ABI.  Objects go to
``build/`` next to this file and the shared library next to the package so
it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "libbbdg_cuda.so"
INCLUDE = PKG.parent / "include"
MAX_DEGREE = 9

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-warn-spills", f"-I{CSRC}", f"-I{INCLUDE}"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(exe).exists():
        raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libbbdg_cuda.so")
    return exe


def _sources_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _units():
    units = [("bbdg_capi", CSRC / "bbdg_capi.cu", []), ("bbdg_func", CSRC / "bbdg_func.cu", []),
             ("bbdg_ops", CSRC / "bbdg_ops.cu", []), ("bbdg_mesh", CSRC / "bbdg_mesh.cu", [])]
    for tname, t in (("f32", "float"), ("f64", "double")):
        for n in range(1, MAX_DEGREE + 1):
            units.append((f"k_{tname}_{n}", CSRC / "bbdg_kernels.cu",
                          [f"-DBBDG_T={t}", f"-DBBDG_TNAME={tname}", f"-DBBDG_N={n}"]))
    return units


def build_variant(out_dir: Path, defines: list[str], dtypes=("f32",), jobs: int | None = None) -> Path:
    """Tuning build: the whole library with extra -D flags into out_dir (loaded via BBDG_LIB)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    exe = nvcc()
    units = [u for u in _units() if not u[0].startswith("k_") or u[0].split("_")[1] in dtypes]
    missing = [u for u in _units() if u not in units]

    def compile_unit(u):
        name, src, defs = u
        obj = out_dir / f"{name}.o"
        cmd = [exe, *ARCH, *FLAGS, *defs, *defines, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(jobs or os.cpu_count() or 1) as ex:
        objs = list(ex.map(compile_unit, units))
    objs += [BUILD / f"{u[0]}.o" for u in missing]   # untouched dtype units from the main build
    lib = out_dir / "libbbdg_cuda.so"
    r = subprocess.run([exe, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return lib


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> Path:
    digest = _sources_digest()
    stamp = BUILD / "digest"
    if LIB.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return LIB
    BUILD.mkdir(exist_ok=True)
    exe = nvcc()

    def compile_unit(u):
        name, src, defs = u
        obj = BUILD / f"{name}.o"
        cmd = [exe, *ARCH, *FLAGS, *defs, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip()):
            print(f"[{name}] {r.stderr.strip()}")
        return obj

    jobs = jobs or max(1, min(len(_units()), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(compile_unit, _units()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [exe, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    stamp.write_text(digest)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.jobs, a.force, a.verbose))
