"""Build the in-tree CUDA library ``libradsplat_b200.so`` (sm_100a only).

    python -m paper_2403_13806_b200.build [--verbose]

The parity contract needs IEEE fp32: no FMA contraction (-fmad=false; the
kernels write every intended fusion as __fmaf_rn), IEEE division and square
root, no flush-to-zero. cudart is linked statically so the library has no
runtime dependency besides the driver (it loads on CPU-only hosts too, which
the "does it export every symbol" test relies on).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libradsplat_b200.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-shared", "-cudart", "static",
    f"-I{INCLUDE}",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "radsplat.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    extra = os.environ.get("RS_NVCC_EXTRA", "").split()  # experiments only (e.g. -DRS_EXP_...)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []),
           str(CSRC / "api.cu"), "-o", str(LIB) + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
