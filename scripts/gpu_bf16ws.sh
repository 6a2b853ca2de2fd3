#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['kernels']['compress_ms'],3), round(d['roofline']['frac'],3))"; }
for v in ${VARIANTS:-default s5 s6 s5d4 s4d4}; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "$v bf16: $(SLC_LIB=$L $B --dtype bf16 | show)  f32: $(SLC_LIB=$L $B | show)  bf16-72b: $(SLC_LIB=$L $B --dtype bf16 --workload covenant-72b --shard-of 8 --steps 3 | show)"
done
