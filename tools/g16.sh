mkdir -p gpurun_out
OSPH_SWEEP_LARGE=1 timeout 600 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu > gpurun_out/bench3L.json 2> gpurun_out/bench3L.err; tail -1 gpurun_out/bench3L.json | cut -c1-1200
timeout 1800 python -m paper_1403_4661_b200.gridopt 4096 gpurun_out/grid-L4096-uniform-condmin.txt --progress 512 > gpurun_out/gridopt4096.txt 2>&1
tail -3 gpurun_out/gridopt4096.txt
