# End-of-round evidence on one B200: bench lines (configs 1-5), launch list of the default bench,
# ncu --set full captures of the dominant kernels.  Summaries: tools/ncu_summary.py -> profiles/.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 1 -c 1 -o gpurun_out/sweep_full -f python tools/fwd_once.py 256 64 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_gemm -s 200 -c 1 -o gpurun_out/sweepgemm_full -f python tools/fwd_once.py 512 128 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bf_update -s 40 -c 1 -o gpurun_out/bfu2048_full -f python tools/fwd_once.py 2048 1 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ring_inverse_bluestein -s 0 -c 1 -o gpurun_out/ringinv_full -f python tools/fwd_once.py 256 64 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
