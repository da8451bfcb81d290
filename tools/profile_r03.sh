#!/bin/bash
# Round-2 (second half) evidence on one B200, after the timed runs: ncu launch lists of
# configs 2 and 3 (one factor chain per call: OSPH_FACTOR_SPLIT=0) and --set full captures
# (+ the fp64 DMMA pipe counters) of the new kernels.  Summaries: tools/launch_summary.py,
# tools/ncu_summary.py -> profiles/.
mkdir -p gpurun_out
M="--metrics sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
OSPH_FACTOR_SPLIT=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_r03_c2.csv python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_l2.log 2>&1
OSPH_FACTOR_SPLIT=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_r03_c3.csv python tools/fwd_once.py 512 128 1 > gpurun_out/ncu_l3.log 2>&1
cap() {  # name regex skip L B N
  timeout 900 ncu --set full $M --import-source on --clock-control none --kernel-name-base demangled -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/$1 -f python tools/fwd_once.py $4 $5 $6 > gpurun_out/ncu_$1.log 2>&1
}
cap sbsolve_r03 'k_sb_gemm<\(int\)0' 7 256 64 1
cap sbcorr_r03 'k_sb_gemm<\(int\)1' 3 256 64 1
cap sbchain_r03 'k_sb_chain<\(int\)16' 3 256 64 1
cap ringinv_r03 'k_ring_inverse_reg' 0 256 64 1
cap ringfwd_r03 'k_ring_forward_reg' 0 256 64 1
cap synth_r03 'k_synth_dmma' 0 256 64 1
cap sbsolve512_r03 'k_sb_gemm<\(int\)0' 15 512 128 1
ls -la gpurun_out/*.ncu-rep
