# breadth-first factorisation variants: round-trip error, determinism and factor time
for pv in 1 0; do
  for L in 256 512 1024 2048; do OSPH_BF_PERSISTENT=$pv timeout 300 python tools/determinism.py $L 1 2 2>&1 | tail -1 | sed "s/^/persistent=$pv /"; done
done
