#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/build_variants.py checked=SLC_CHECKED > gpurun_out/g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_guard.py -m gpu -q 2>&1 | tail -2
SLC_LIB=build/variants/libslc_checked.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-e2e --cpu-seconds 6 > gpurun_out/g_bench.log 2>&1; tail -1 gpurun_out/g_bench.log | cut -c1-400
tail -1 gpurun_out/g_bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['kernels'], d['roofline']['frac'], d.get('step_roofline'), {k:v for k,v in d['cpu_baseline'].items() if k!='affinity'})"
