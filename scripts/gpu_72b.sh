# the target config (BASELINE configs[3]): one GPU's shard of the 8-way Covenant-72B job, R = 20
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv
for dt in f32 bf16; do
  timeout 900 python bench.py --workload covenant-72b --shard-of 8 --shard-rank 0 --dtype $dt --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b72_$dt.log 2>&1
  echo "72b/8 $dt rc=$? $(tail -n 1 gpurun_out/b72_$dt.log | cut -c1-200)"
  python -c "import json; d=json.loads(open('gpurun_out/b72_$dt.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernels'], d['hbm_frac_of_peak'])"
done
timeout 900 python bench.py --workload llama3-8b --shard-of 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b8b_2.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b8b_2.log').read().strip().splitlines()[-1]); print('8b/2', d['ms_per_step'], d['kernels'], d['hbm_frac_of_peak'])"
