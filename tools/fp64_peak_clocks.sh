#!/bin/bash
# fp64 peak probe (tools/probe/fp64_peak.cu, prebuilt) with SM clocks and throttle
# reasons sampled by nvidia-smi while it runs -> gpurun_out/fp64_peak_r02.txt
mkdir -p gpurun_out
out=gpurun_out/fp64_peak_r02.txt
( for i in $(seq 1 60); do nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw --format=csv,noheader; sleep 0.2; done ) > gpurun_out/fp64_clk.csv &
CLK=$!
echo "fp64 peak probe (tools/probe/fp64_peak.cu), B200 sm_100a, $(date -u +%FT%TZ)" > $out
./tools/probe/fp64_peak >> $out 2>&1
kill $CLK 2>/dev/null; wait $CLK 2>/dev/null
echo "clocks during the run (nvidia-smi every 0.2 s: sm MHz, max MHz, hw_slowdown, sw_thermal, sw_power_cap, W):" >> $out
sort gpurun_out/fp64_clk.csv | uniq -c | sort -rn | head -8 >> $out
cat $out
