run() { timeout 900 python -m pytest tests -q -m gpu -k "$1" > /tmp/pp.txt 2>&1; echo "$(tail -1 /tmp/pp.txt) :: $1"; }
run "not L2048_roundtrip and not real and not L512"
run "not L2048_roundtrip and (L2048 or L4096 or real or L512 or large_L or windowed)"
run "not L2048_roundtrip and (L2048 or L4096 or batch or static or torch or large_L)"
