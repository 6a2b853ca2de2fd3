#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SLC_LIB=build/variants/libslc_sm64.so timeout 900 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py -m gpu -q -x -k "select or compress or geometry" 2>&1 | tail -1
VARIANTS="default sm64 sm80" ROUNDS=1 bash scripts/gpu_cmpv.sh
for v in default sm64; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "== $v"; SLC_LIB=$L SPECS="64:128 64:256 32:16 32:64" bash scripts/gpu_sweep2.sh
done
