#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pb_build.log 2>&1
CMD="python bench.py --workload llama3-8b --shard-of 4 --dtype ${DT:-f32} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --agg-kernel batch"
ncu --set full --clock-control none --import-source on -k regex:"agg_batch" -s 3 -c 1 -o gpurun_out/pb_${DT:-f32} $CMD > gpurun_out/pb_ncu.log 2>&1
echo done
