timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "compress or geometry" 2>&1 | tail -2
for k in 64 256; do
  echo "== k=$k"; WS=1 K=$k NRANKS=8 SLC_LIB=build/variants/libslc_phase.so timeout 600 python tools/phase_timing.py llama2-7b 2>&1 | tail -11
done
rm build/variants/libslc_phase.so
bash scripts/gpu_sweepvar.sh
