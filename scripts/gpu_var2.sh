mkdir -p gpurun_out
for so in build/variants/*.so; do
  n=$(basename $so .so)
  for spec in "llama3.2-1b:" "llama3-8b:--shard-of 4" "covenant-72b:--shard-of 8"; do
    wl=${spec%%:*}; ex=${spec#*:}
    SLC_LIB=$so timeout 600 python bench.py --workload $wl $ex --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v_${n}_$wl.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/v_${n}_$wl.log').read().strip().splitlines()[-1]); k=d['kernels']; print('$n $wl', round(d['ms_per_step'],3), round(k['compress_ms'],3), round(k['fused_update_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/v_${n}_$wl.log
  done
done
