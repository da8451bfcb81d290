mkdir -p gpurun_out
OSPH_BF_NMIN=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bf256_launches.csv python tools/fwd_once.py 256 64 2 > gpurun_out/ncu_bf256.log 2>&1
tail -2 gpurun_out/ncu_bf256.log
