#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --workload llama2-7b --shard-of 8 --block ${BLK:-64} --k ${KK:-256} --R 20 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"compress_fallback" -s 2 -c 1 -o gpurun_out/prof_fbk $CMD > gpurun_out/pfbk.log 2>&1
tail -1 gpurun_out/pfbk.log
SLC_LIB=build/variants/libslc_pt.so python tools/bench_paths.py --workload llama2-7b --shard-of 8 --block ${BLK:-64} --k ${KK:-256} --R 20 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -A1 "paths over"
