# Round-1 (session d) evidence on one B200: bench lines of configs 1-5, the launch list of the default
# bench (config 2), ncu full captures of the sweep (L=256) and of the wide update (L=2048).
mkdir -p gpurun_out/r01d
for c in 2 1 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/r01d/bench_config$c.json 2> gpurun_out/r01d/bench_config$c.err
  tail -1 gpurun_out/r01d/bench_config$c.json | cut -c1-200
done
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/r01d/bench_config5.json 2> gpurun_out/r01d/bench_config5.err
tail -1 gpurun_out/r01d/bench_config5.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r01d/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r01d/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 1 -c 1 -o gpurun_out/r01d/sweep_full -f python tools/fwd_once.py 256 64 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bf_update_w -s 40 -c 1 -o gpurun_out/r01d/bfuw2048_full -f python tools/fwd_once.py 2048 1 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bf_update_w -s 4 -c 1 -o gpurun_out/r01d/bfuw256_full -f python tools/fwd_once.py 256 64 2 > /dev/null 2>&1
ls -la gpurun_out/r01d
