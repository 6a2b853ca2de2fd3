#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for a in "" "--special-period 32" "--special-period 8" "--dtype bf16 --cold-ef"; do
  echo "[$a] $(SLC_LIB=build/variants/libslc_pt.so python tools/bench_paths.py $B $a 2>&1 | grep -A1 "paths over")"
done
