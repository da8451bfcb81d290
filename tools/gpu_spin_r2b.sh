#!/bin/bash
set -x
mkdir -p gpurun_out/spin
timeout 1200 python -m pytest tests/test_gpu_spin.py -q -m gpu > gpurun_out/spin/spin_tests.log 2>&1
grep -E "^E  .*(Error|assert)" gpurun_out/spin/spin_tests.log | head -30
tail -15 gpurun_out/spin/spin_tests.log
