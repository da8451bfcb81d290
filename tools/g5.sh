mkdir -p gpurun_out
timeout 900 python -m paper_1403_4661_b200.gridopt 2048 gpurun_out/grid-L2048-uniform-condmin.txt --progress 256 > gpurun_out/gridopt2048.txt 2>&1
tail -2 gpurun_out/gridopt2048.txt
timeout 1800 python -m paper_1403_4661_b200.gridopt 4096 gpurun_out/grid-L4096-uniform-condmin.txt --progress 256 > gpurun_out/gridopt4096.txt 2>&1
tail -2 gpurun_out/gridopt4096.txt
