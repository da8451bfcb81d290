mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -1 gpurun_out/bench3.json | cut -c1-150
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json | cut -c1-150
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -1 gpurun_out/bench5.json | cut -c1-150
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -1 gpurun_out/bench2.json | cut -c1-150
