#!/bin/bash
# tools/probe/run.sh NAME: compile tools/probe/NAME.cu for sm_100a and run it on the GPU box
set -e
cd /root/repo/tools/probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -o "$1" "$1.cu"
cd /root/repo
/usr/local/graft/bin/gpurun --timeout 300 -- "./tools/probe/$1" > /dev/null 2>&1 || true
python3 -c "import json; d=json.load(open('/root/repo/gpurun_out/.last_call.json')); print(d.get('stdout_tail','')[-1500:])"
