run() { timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$1" > /tmp/pp.txt 2>&1; echo "$(tail -1 /tmp/pp.txt) :: $1 :: $2"; }
run "real or L512 or large_L or windowed" default
OSPH_SWEEP_LARGE=1 run "real or L512 or large_L or windowed" sweep_large
run "real or L512 or large_L or windowed" default-again
run "(real or L512) and not batched" default-nobatched
