#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'compress', round(d['kernels']['compress_ms'],3))"; }
for v in r1 default; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  for sp in 0 32; do echo "$v special $sp $(SLC_LIB=$L $B --special-period $sp 2>&1 | show)"; done
  echo "$v bf16 cold $(SLC_LIB=$L $B --dtype bf16 --cold-ef 2>&1 | show)"
done
