for cfg in "2 4 6" "2 8 6" "2 8 4" "1 4 6" "1 8 4" "4 8 6" "4 4 4"; do
  set -- $cfg
  echo "MINB2 G=$1 T=$2 S=$3"; OSPH_DEBUG=1 OSPH_LIB=tools/libosph_minb2.so OSPH_SWEEP_G=$1 OSPH_SWEEP_T=$2 OSPH_SWEEP_S=$3 timeout 60 python tools/fwd_once.py 256 64 3 2>&1 | tail -2
done
