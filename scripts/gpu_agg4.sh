# parity of the aggregate kernels + update timing at R=8 (1B) and R=20 (8B shard of 4) + ncu of the R=20 update
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -rf 2>&1 | tail -15 > gpurun_out/agg_pytest.log
tail -3 gpurun_out/agg_pytest.log
for spec in "llama3.2-1b:" "llama3-8b:--shard-of 4"; do
  wl=${spec%%:*}; ex=${spec#*:}
  timeout 600 python bench.py --workload $wl $ex --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/a4_$wl.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/a4_$wl.log').read().strip().splitlines()[-1]); k=d['kernels']; print('$wl', round(d['ms_per_step'],3), round(k['compress_ms'],3), round(k['fused_update_ms'],3), 'upd GB/s', round(k['update_bytes_per_launch']/k['fused_update_ms']/1e6))"
done
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe" -s 2 -c 1 -o gpurun_out/prof_r20b python bench.py --workload llama3-8b --shard-of 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r20b.log 2>&1
echo ncu rc=$?
