"""Build libosph.so (sm_100a) in-tree with nvcc.

    python -m paper_1403_4661_b200.build [--force]

The library travels with the repository snapshot to the GPU box; nothing is
JIT-compiled at run time.

Every .cu file is compiled to an object on its own (in parallel; only the
files whose sources changed are recompiled) and the objects are linked.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
SOURCES = ["plan.cu", "tables.cu", "ringdft.cu", "synth.cu", "factor.cu", "sweep.cu", "sweep_large.cu", "factor_bf.cu", "pivots.cu", "window.cu", "sweep_gemm.cu", "sweep_block.cu", "shard.cu", "spin.cu"]
OUT = HERE / "libosph.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
OBJ = CSRC / "build"  # git-ignored, gpurun-ignored (only libosph.so travels)
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I", str(HERE.parent / "include"),
    *os.environ.get("OSPH_NVCC_FLAGS", "").split(),  # e.g. -DOSPH_SWEEP_PROF (debug builds)
]


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "osph.h"]


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(d.stat().st_mtime > t for d in [CSRC / s for s in SOURCES] + _headers())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    OBJ.mkdir(exist_ok=True)
    hdr_t = max(h.stat().st_mtime for h in _headers())
    jobs = []
    for s in SOURCES:
        src, obj = CSRC / s, OBJ / (Path(s).stem + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_t):
            jobs.append([NVCC, *FLAGS, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    tmp = OUT.with_suffix(".so.tmp")
    run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
         *[str(OBJ / (Path(s).stem + ".o")) for s in SOURCES]])
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
