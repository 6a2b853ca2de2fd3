for k in 64 128 256; do
  echo "== k=$k"; WS=1 K=$k NRANKS=8 SLC_LIB=build/variants/libslc_phase.so timeout 600 python tools/phase_timing.py llama2-7b 2>&1 | tail -11
done
