mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for R in 8 20; do
  timeout 600 python bench.py --workload llama3.2-1b --R $R --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/agg_R$R.log 2>&1
  echo "R=$R $(python -c "import json; d=json.loads(open('gpurun_out/agg_R$R.log').read().strip().splitlines()[-1]); print(d['kernels'], d['ms_per_step'])" 2>&1 | tail -1)"
done
