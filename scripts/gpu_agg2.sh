# aggregate kernel A/B: parity tests of every aggregate kernel, then bench with each
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -rf 2>&1 | tail -30 > gpurun_out/agg_pytest.log
for k in pipe simple; do
  if [ $k = simple ]; then export SLC_AGG_KERNEL=simple; else unset SLC_AGG_KERNEL; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/agg_bench_$k.log 2>&1
  tail -n 1 gpurun_out/agg_bench_$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['ms_per_step'], d['kernels'])"
done
unset SLC_AGG_KERNEL
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype bf16 > gpurun_out/agg_bench_bf16.log 2>&1
tail -n 1 gpurun_out/agg_bench_bf16.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe" -s 2 -c 1 -o gpurun_out/prof_aggpipe python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aggpipe.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/agg_pytest.log
