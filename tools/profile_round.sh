#!/bin/bash
# Round profiling on one B200: bench line, ncu launch list of one bench step,
# full ncu captures of the two dominant kernels (sweep, static-pivot factor).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 1 -c 1 \
  -o gpurun_out/sweep_full -f python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_sweep.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_factor_np -s 0 -c 1 \
  -o gpurun_out/factornp_full -f python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_factor.log 2>&1
ls -la gpurun_out
