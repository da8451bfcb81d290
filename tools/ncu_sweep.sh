timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -s 1 -c 1 -o gpurun_out/sweep_r01b -f python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_sweep.log 2>&1
tail -3 gpurun_out/ncu_sweep.log
