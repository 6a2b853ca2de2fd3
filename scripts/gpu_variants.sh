# time compress/update of each libslc variant in build/variants (bench.py, short run)
mkdir -p gpurun_out
for wl in ${WORKLOADS:-llama3.2-1b}; do
for so in build/variants/*.so; do
  n=$(basename $so .so)
  SLC_LIB=$so timeout 600 python bench.py --workload $wl ${EXTRA} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_${n}_$wl.log 2>&1
  echo "$wl $n $(python -c "import json,sys; d=json.loads(open('gpurun_out/var_${n}_$wl.log').read().strip().splitlines()[-1]); print(d['kernels']['compress_ms'], d['kernels']['fused_update_ms'], d['ms_per_step'])" 2>&1 | tail -1)"
done
done
