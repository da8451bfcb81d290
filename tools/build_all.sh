#!/bin/bash
# Build libosph.so and the profiling variants; exit non-zero on any compile error.
set -e
cd /root/repo
python -c "from paper_1403_4661_b200 import build; build.build()"
S=paper_1403_4661_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include -lcusolver -Xlinker -rpath=/usr/local/cuda/lib64"
SRC="$S/plan.cu $S/tables.cu $S/ringdft.cu $S/synth.cu $S/factor.cu $S/factor_np.cu $S/sweep.cu $S/sweep_large.cu $S/factor_bf.cu $S/pivots.cu $S/window.cu $S/sweep_gemm.cu"
nvcc $F -DOSPH_SWEEP_PROF -o tools/libosph_prof.so $SRC
nvcc $F -DOSPH_FACTOR_PROF -o tools/libosph_fprof.so $SRC
