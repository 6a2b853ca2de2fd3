#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
OUT=gpurun_out/rsweep.txt; : > $OUT
for R in 2 4 8 16 20 32 64; do
  timeout 600 python bench.py --workload llama2-7b --shard-of 8 --R $R --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rs.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rs.log').read().strip().splitlines()[-1]); k=d['kernels']
print(f'C=  4096 k=  64 R={$R:3d}  step {d[\"ms_per_step\"]:7.3f} ms  compress {k[\"compress_ms\"]:7.3f}  update {k[\"fused_update_ms\"]:7.3f}  step_frac {d[\"step_roofline\"][\"frac_of_measured_peak\"]:.3f}  sm_mhz {d[\"clocks\"][\"sm_mhz\"]}')" >> $OUT
done
for R in 20 64; do for dt in bf16; do
  timeout 600 python bench.py --workload llama2-7b --shard-of 8 --R $R --dtype $dt --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rs.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/rs.log').read().strip().splitlines()[-1]); k=d['kernels']
print(f'C=  4096 k=  64 R={$R:3d} $dt step {d[\"ms_per_step\"]:7.3f} ms  compress {k[\"compress_ms\"]:7.3f}  update {k[\"fused_update_ms\"]:7.3f}  step_frac {d[\"step_roofline\"][\"frac_of_measured_peak\"]:.3f}  sm_mhz {d[\"clocks\"][\"sm_mhz\"]}')" >> $OUT
done; done
cat $OUT
