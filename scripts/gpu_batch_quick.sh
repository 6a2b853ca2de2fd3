#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bq_build.log 2>&1 || { tail -20 gpurun_out/bq_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py -m gpu -q -x -k "batch or canonical or inv_r or quantizer" 2>&1 | tail -2
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for k in ${KS:-batch}; do for dt in f32 bf16; do
  echo "== 8b/4 $k $dt $($B --workload llama3-8b --shard-of 4 --dtype $dt --agg-kernel $k 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['kernels']['fused_update_ms'],3))")"
done; done
