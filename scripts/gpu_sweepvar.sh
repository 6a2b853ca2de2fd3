mkdir -p gpurun_out
for so in build/variants/*.so; do
  n=$(basename $so .so)
  for spec in "64 128" "64 256" "64 32" "32 16"; do
    set -- $spec
    SLC_LIB=$so timeout 600 python bench.py --workload llama2-7b --shard-of 8 --block $1 --k $2 --R 20 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sv.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/sv.log').read().strip().splitlines()[-1]); k=d['kernels']; print('$n B=$1 k=$2', round(d['ms_per_step'],3), round(k['compress_ms'],3), round(k['fused_update_ms'],3))" || tail -3 gpurun_out/sv.log
  done
done
