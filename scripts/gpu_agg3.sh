# parity of the aggregate kernels, then variant sweep (compress / update / step ms)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -rf 2>&1 | tail -15 > gpurun_out/agg_pytest.log
tail -2 gpurun_out/agg_pytest.log
WORKLOADS="${WORKLOADS:-llama3.2-1b}" bash scripts/gpu_variants.sh
SLC_AGG_KERNEL=simple timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/agg_simple.log 2>&1
echo "simple $(tail -n 1 gpurun_out/agg_simple.log | cut -c1-0)$(python -c "import json; d=json.loads(open('gpurun_out/agg_simple.log').read().strip().splitlines()[-1]); print(d['kernels'])")"
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe" -s 2 -c 1 -o gpurun_out/prof_aggpipe python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_aggpipe.log 2>&1
echo ncu rc=$?
