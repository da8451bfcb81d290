timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_factor_np -s 0 -c 1 -o gpurun_out/factornp_r01c -f python tools/fwd_once.py 256 1 2 > gpurun_out/ncu_factor.log 2>&1
tail -2 gpurun_out/ncu_factor.log
