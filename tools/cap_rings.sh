cap() {  # name regex skip L B N
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/$1 -f python tools/fwd_once.py $4 $5 $6 > gpurun_out/ncu_$1.log 2>&1
}
cap ringinv_r03 'k_ring_inverse_reg' 0 256 64 1
cap ringfwd_r03 'k_ring_forward_reg' 0 256 64 1
ls -la gpurun_out/*.ncu-rep
