#!/bin/bash
# ncu --set full capture of one kernel: tools/cap_kernel.sh NAME REGEX SKIP L B N [env...]
name=$1; regex=$2; skip=$3; L=$4; B=$5; N=$6
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none --kernel-name-base demangled \
  -k regex:$regex -s $skip -c 1 -o gpurun_out/$name -f python tools/fwd_once.py $L $B $N > gpurun_out/ncu_$name.log 2>&1
ls -la gpurun_out/$name.ncu-rep
