set -x
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
cat gpurun_out/r2e_bench.json
timeout 900 python -m pytest tests/test_gpu_pivots_sweeps.py -q -m gpu -k "sweep or config3" > gpurun_out/r2e_sw.log 2>&1
tail -3 gpurun_out/r2e_sw.log
bash tools/sanitize.sh > gpurun_out/r2e_san.log 2>&1
cat gpurun_out/sanitize_summary.txt
