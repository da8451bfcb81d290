#!/bin/bash
# Round-2 evidence on one B200 (after the timed runs): ncu launch lists and
# --set full captures (+ the fp64 DMMA pipe counters) of the dominant kernels.
# Summaries: python tools/launch_summary.py / tools/ncu_summary.py -> profiles/.
mkdir -p gpurun_out
M="--metrics sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_r02_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_l2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_r02_c4.csv python tools/fwd_once.py 2048 1 2 > gpurun_out/ncu_l4.log 2>&1
cap() {  # name regex skip L B N
  timeout 900 ncu --set full $M --import-source on --clock-control none --kernel-name-base demangled -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/$1 -f python tools/fwd_once.py $4 $5 $6 > gpurun_out/ncu_$1.log 2>&1
}
cap sweep_r02 'k_sweep<\(int\)8>' 1 256 64 2
cap synth_r02 'k_synth_dmma' 0 256 64 1
cap ringinv_r02 'k_ring_inverse_bluestein\(' 0 256 64 1
cap ringfwd_r02 'k_ring_forward_bluestein\(' 1 256 64 2
cap bfu256_r02 'k_bf_update<\(bool\)1>' 2 256 64 2
cap bfpair2048_r02 'k_bf_update_w<\(bool\)1>' 4 2048 1 1
cap sweepgemm_r02 'k_sweep_gemm<\(int\)0' 300 512 128 1
ls -la gpurun_out/*.ncu-rep
