#!/bin/bash
# compress ms per variant (VARIANTS="head default ..."), configs interleaved, two rounds
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['kernels']['compress_ms'],3))"; }
for round in $(seq ${ROUNDS:-2}); do
for cfg in "" "--special-period 32" "--dtype bf16" "--dtype bf16 --cold-ef"; do
  line="[$cfg]"
  for v in ${VARIANTS:-head default}; do
    L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
    line="$line $v $(SLC_LIB=$L $B $cfg 2>&1 | show)"
  done
  echo "$line"
done
done
