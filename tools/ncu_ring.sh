timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ring_inverse_bluestein -s 1 -c 1 -o gpurun_out/ringinv_full -f python tools/fwd_once.py 256 64 1 > gpurun_out/ncu_ri.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_synth_dmma -s 1 -c 1 -o gpurun_out/synth_full -f python tools/fwd_once.py 256 64 1 > gpurun_out/ncu_sy.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ring_forward_bluestein -s 1 -c 1 -o gpurun_out/ringfwd_full -f python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_rf.log 2>&1
ls gpurun_out/*.ncu-rep
