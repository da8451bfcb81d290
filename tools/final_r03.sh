#!/bin/bash
# End-of-round evidence on one B200 (second half of round 2): GPU tests + smoke, bench lines of
# configs 1-5 and the reference arm, then the ncu launch lists and captures (tools/profile_r03.sh).
set -x
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final/gpu_tests.log 2>&1
tail -3 gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
tail -2 gpurun_out/final/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final/bench_config2.json 2> gpurun_out/final/bench_config2.err
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 > gpurun_out/final/bench_config1.json 2> gpurun_out/final/bench_config1.err
timeout 1200 python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/final/bench_config3.json 2> gpurun_out/final/bench_config3.err
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/final/bench_config4.json 2> gpurun_out/final/bench_config4.err
timeout 2400 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/final/bench_config5.json 2> gpurun_out/final/bench_config5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
for f in gpurun_out/final/bench_*.json; do echo "$f: $(tail -c 300 $f)"; done
bash tools/profile_r03.sh > gpurun_out/final/prof.log 2>&1
ls gpurun_out/*.ncu-rep
