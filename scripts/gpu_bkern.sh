#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for a in ${CFGS:-"--special-period 32" "--dtype bf16 --cold-ef"}; do
  echo "[$a]"; SEQ=compress python tools/bench_kernels.py $B $a 2>&1 | grep -i "compress\|in order"
done
