set -x
bash tools/profile_r02.sh > gpurun_out/r2i_prof.log 2>&1
tail -12 gpurun_out/r2i_prof.log
python -m paper_1403_4661_b200.gridopt 1024 gpurun_out/grid-L1024-uniform-condmin.txt --progress 256 > gpurun_out/r2i_grid1024.log 2>&1
timeout 1800 python tools/gridopt_validate.py 1024 gpurun_out/grid-L1024-uniform-condmin.txt > gpurun_out/gridopt_validate_1024.txt 2>&1
timeout 2400 python tools/gridopt_validate.py 2048 > gpurun_out/gridopt_validate_2048.txt 2>&1
timeout 900 python tools/gridopt_validate.py 256 > gpurun_out/gridopt_validate_256.txt 2>&1
cat gpurun_out/gridopt_validate_*.txt
