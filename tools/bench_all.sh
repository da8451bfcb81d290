# bench lines of configs 1-5 (with the CPU baseline legs) into gpurun_out/$1/
mkdir -p gpurun_out/$1
for c in 2 1 3 4; do timeout 900 python bench.py --config $c > gpurun_out/$1/bench_config$c.json 2> gpurun_out/$1/bench_config$c.err; done
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/$1/bench_config5.json 2> gpurun_out/$1/bench_config5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$1/bench_reference.json 2> gpurun_out/$1/bench_reference.err
