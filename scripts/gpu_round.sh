# full evidence pass: GPU tests, smoke, default bench, 72B shard (f32/bf16), launch list + ncu of the default step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf 2>&1 | tail -5 > gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log | cut -c1-200
for dt in f32 bf16; do
  timeout 900 python bench.py --workload covenant-72b --shard-of 8 --dtype $dt --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b72_$dt.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b72_$dt.log').read().strip().splitlines()[-1]); print('72b/8 $dt', d['ms_per_step'], d['kernels'], d['hbm_frac_of_peak'], d['clocks'])"
done
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"compress_ws|agg_pipe" -s 9 -c 2 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
