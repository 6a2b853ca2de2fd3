#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --dtype bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"compress_ws" -s 10 -c 1 -o gpurun_out/prof_bf16 $CMD > gpurun_out/pbf16.log 2>&1
tail -1 gpurun_out/pbf16.log
