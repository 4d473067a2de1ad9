"""In-tree build of the sm_100a extension (``libfsa_b200.so``).

``nvcc -gencode arch=compute_100a,code=sm_100a`` straight into the package directory, so the
shared object travels with the repo snapshot to the GPU box.  No ``--use_fast_math``: the
kernels need IEEE division and unfused adds for bitwise parity with the reference
(SURVEY.md §8c).
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libfsa_b200.so"
SOURCES = [CSRC / "fsa_kernels.cu", CSRC / "fsa_head.cu"]
DEPS = SOURCES + [CSRC / "fsa_rng.cuh", PKG_DIR.parent / "include" / "fsa_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the sm_100a extension cannot be built")
    return cand


def needs_build() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > built for p in DEPS if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the CUDA extension in place; returns the library path."""
    if not force and not needs_build():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *NVCC_FLAGS, "-o", str(tmp), *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
