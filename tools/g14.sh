mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_bf --csv --log-file gpurun_out/bf_launches.csv python tools/fwd_once.py 2048 1 2 > gpurun_out/ncu_bf.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bf_update -s 40 -c 1 -o gpurun_out/bf_update_full -f python tools/fwd_once.py 2048 1 2 > gpurun_out/ncu_bfu.log 2>&1
ls -la gpurun_out | head -30
