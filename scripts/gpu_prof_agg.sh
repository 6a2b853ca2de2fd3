#!/bin/bash
# ncu --set full of the fused update at R=20 (8B shard of 4), fp32 and bf16
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pa_build.log 2>&1
for dt in f32 bf16; do
CMD="python bench.py --workload llama3-8b --shard-of 4 --dtype $dt --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/pa_$dt.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe" -s 3 -c 1 -o gpurun_out/pa_$dt $CMD > gpurun_out/pa_ncu_$dt.log 2>&1
done
echo done
