#!/bin/bash
# batched decode kernel: parity tests, then bench vs the pipelined kernel
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1 || { tail -20 gpurun_out/b_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_scale.py -m gpu -q -x -k "not covenant" > gpurun_out/b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/b_tests.log
tail -5 gpurun_out/b_tests.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
: > gpurun_out/b_bench.log
for k in batch pipe; do
  for dt in f32 bf16; do
    echo "== 8b/4 $k $dt" >> gpurun_out/b_bench.log
    $B --workload llama3-8b --shard-of 4 --dtype $dt --agg-kernel $k 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels'])" >> gpurun_out/b_bench.log 2>&1
  done
  echo "== 1b $k" >> gpurun_out/b_bench.log
  $B --agg-kernel $k 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels'])" >> gpurun_out/b_bench.log 2>&1
done
cat gpurun_out/b_bench.log
