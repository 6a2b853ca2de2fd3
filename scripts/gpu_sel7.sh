#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
for v in default hbr2; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "== $v"; SLC_LIB=$L SPECS="64:256 32:64 64:128" bash scripts/gpu_sweep2.sh
done
VARIANTS="default" ROUNDS=1 bash scripts/gpu_cmpv.sh
SLC_LIB=build/variants/libslc_pt.so python tools/bench_paths.py --workload llama2-7b --shard-of 8 --k 256 --R 20 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -A1 "paths over"
