#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default fb6 fb8; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "== $v"; SLC_LIB=$L SPECS="64:256 32:64" bash scripts/gpu_sweep2.sh
done
VARIANTS="default fb6 fb8" ROUNDS=1 bash scripts/gpu_cmpv.sh
