#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do for v in ${VARIANTS:-head default}; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "$v special 8: $(SLC_LIB=$L $B --special-period 8 | tail -1 | python -c "import sys,json; print(json.load(sys.stdin)['kernels']['compress_ms'])")  bf16 cold: $(SLC_LIB=$L $B --dtype bf16 --cold-ef | tail -1 | python -c "import sys,json; print(json.load(sys.stdin)['kernels']['compress_ms'])")"
done; done
