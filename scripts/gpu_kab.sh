#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for v in v5c4 default; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "== $v"; SLC_LIB=$L SPECS="64:128 64:256 32:64 64:64" bash scripts/gpu_sweep2.sh | sed 's/density.*step/ step/'
done; done
