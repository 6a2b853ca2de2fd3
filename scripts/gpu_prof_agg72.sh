#!/bin/bash
# ncu --set full of the fused update (agg_pipe) on the 72B shard of 8, R=20
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --workload covenant-72b --shard-of 8 --dtype ${DT:-f32} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe" -s 1 -c 1 -o gpurun_out/prof_agg72_${DT:-f32} $CMD > gpurun_out/pagg_ncu.log 2>&1
tail -2 gpurun_out/pagg_ncu.log
