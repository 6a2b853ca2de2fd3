#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_pins.py tests/test_gpu_guard.py tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --workload covenant-72b --shard-of 8 --median-norm"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); k=d['kernels']; print(round(d['ms_per_step'],3), 'upd', round(k['fused_update_ms'],3))"; }
for r in 1 2; do for v in head default; do
  L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so
  echo "$v 72b mn f32: $(SLC_LIB=$L $B | show) bf16: $(SLC_LIB=$L $B --dtype bf16 | show) | 1b mn: $(SLC_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --median-norm | show)"
done; done
