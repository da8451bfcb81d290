#!/bin/bash
# Spin-weighted transforms on the GPU: parity tests, the scalar GPU suite, and
# the reference arm re-measured after the BLAS thread cap.
set -x
mkdir -p gpurun_out/spin
timeout 1200 python -m pytest tests/test_gpu_spin.py -q -m gpu -x > gpurun_out/spin/spin_tests.log 2>&1
tail -15 gpurun_out/spin/spin_tests.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/spin/gpu_tests.log 2>&1
tail -3 gpurun_out/spin/gpu_tests.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/spin/bench_reference.json 2> gpurun_out/spin/bench_reference.err
tail -c 600 gpurun_out/spin/bench_reference.json
nproc
