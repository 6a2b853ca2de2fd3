#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --workload llama2-7b --shard-of 8"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); k=d['kernels']; print('upd', round(k['fused_update_ms'],3))"; }
for v in default fm64 fm1; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "$v R2: $(SLC_LIB=$L $B --R 2 | show) R4: $(SLC_LIB=$L $B --R 4 | show) R8: $(SLC_LIB=$L $B --R 8 | show) C1024k4: $(SLC_LIB=$L $B --R 20 --block 32 --k 4 | show) C1024k16: $(SLC_LIB=$L $B --R 20 --block 32 --k 16 | show) k16: $(SLC_LIB=$L $B --R 20 --k 16 | show) 1b: $(SLC_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | show)"
done
