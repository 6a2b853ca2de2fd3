#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --workload llama3-8b --shard-of 4"
for v in default; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  for dt in f32 bf16; do
    echo "== $v $dt $(SLC_LIB=$L $B --dtype $dt --agg-kernel batch 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['kernels']['fused_update_ms'],3))")"
  done
done
for R in 16 32; do
  echo "== R$R batch $($B --agg-kernel batch --R $R 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['kernels']['fused_update_ms'],3))") pipe $($B --agg-kernel pipe --R $R 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['kernels']['fused_update_ms'],3))")"
done
