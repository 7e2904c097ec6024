"""Build libmpskq.so in-tree with nvcc for sm_100a.

    python -m paper_2411_09336_b200.build [--force]

The library is written next to this file so it travels with the repository
snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmpskq.so"
SOURCES = ["runtime.cpp", "encode.cu", "sim.cu", "overlap.cu"]
HEADERS = ["internal.h", "device.cuh", "o1_site.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "mpskq.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines: tuple = ()) -> Path:
    """Compile every CUDA/C++ source into one shared library (sm_100a only).

    `out` / `defines` build a variant next to the tree for A/B and debug runs
    (e.g. ``defines=("MPSKQ_DEBUG_COUNTERS",)``); the product library is LIB."""
    target = Path(out) if out is not None else LIB
    if out is None and not defines and not force and not _stale():
        return LIB
    objs = []
    tmp = PKG / ("_obj" if not defines else "_obj_" + "_".join(d.lower() for d in defines))
    tmp.mkdir(exist_ok=True)
    for src in SOURCES:
        obj = tmp / (src + ".o")
        cmd = [_nvcc(), *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", str(ROOT / "include"), "-c",
               str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp_out = target.with_suffix(".so.tmp")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp_out), *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp_out, target)
    return target


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose=True)
    print(p)
