#!/bin/bash
# ncu of the fused update of a tuning variant: V=<variant> DT=<f32|bf16>
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
L=build/variants/libslc_${V}.so; [ "${V:-default}" = default ] && L=paper_2603_08163_b200/libslc.so
CMD="python bench.py --workload llama3-8b --shard-of 4 --dtype ${DT:-f32} --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --agg-kernel ${K:-batch}"
SLC_LIB=$L ncu --set full --clock-control none --import-source on -k regex:"agg_" -s 3 -c 1 -o gpurun_out/pv_${V:-default}_${DT:-f32} $CMD > gpurun_out/pv_ncu.log 2>&1
tail -2 gpurun_out/pv_ncu.log
