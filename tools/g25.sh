mkdir -p gpurun_out
OSPH_BF_NMIN=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bf_diag -s 4 -c 1 -o gpurun_out/bf_diag_full -f python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_diag.log 2>&1
tail -2 gpurun_out/ncu_diag.log
