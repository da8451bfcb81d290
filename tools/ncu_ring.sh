timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ring_inverse_bluestein -s 0 -c 1 -o gpurun_out/ringinv2 -f python tools/dbg_ring.py 256 > gpurun_out/ncu_ri.log 2>&1
