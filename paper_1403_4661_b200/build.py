"""Build libosph.so (sm_100a) in-tree with nvcc.

    python -m paper_1403_4661_b200.build [--force]

The library travels with the repository snapshot to the GPU box; nothing is
JIT-compiled at run time.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
SOURCES = ["plan.cu", "tables.cu", "ringdft.cu", "synth.cu", "factor.cu", "sweep.cu", "sweep_large.cu", "factor_bf.cu", "pivots.cu", "window.cu", "sweep_gemm.cu", "shard.cu", "spin.cu"]
OUT = HERE / "libosph.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", str(HERE.parent / "include"),
]


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "osph.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [NVCC, *FLAGS, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
