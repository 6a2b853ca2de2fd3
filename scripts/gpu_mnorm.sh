mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "median or sqnorm or crafted or misaligned" 2>&1 | tail -15 > gpurun_out/mn_pytest.log
tail -3 gpurun_out/mn_pytest.log
for spec in "llama3.2-1b:" "llama3-8b:--shard-of 4"; do
  wl=${spec%%:*}; ex=${spec#*:}
  for mn in "" "--median-norm"; do
    timeout 600 python bench.py --workload $wl $ex $mn --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mn_$wl.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/mn_$wl.log').read().strip().splitlines()[-1]); k=d['kernels']; print('$wl $mn', round(d['ms_per_step'],3), round(k['compress_ms'],3), round(k['fused_update_ms'],3))" || tail -5 gpurun_out/mn_$wl.log
  done
done
