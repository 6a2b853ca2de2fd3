#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_scale.py -m gpu -q -x 2>&1 | tail -3
VARIANTS="${VARIANTS:-default}" ROUNDS=1 bash scripts/gpu_cmpv.sh; B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"; echo "special 8: $($B --special-period 8 | tail -1 | python -c "import sys,json; print(json.load(sys.stdin)['kernels']['compress_ms'])")"
for sp in 32 8; do echo "fb split $sp"; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:compress_fallback --csv python bench.py --steps 1 --warmup 3 --special-period $sp --no-cpu-baseline --no-e2e 2>/dev/null | grep fallback | tail -2 | awk -F'","' '{print $NF}'; done
bash scripts/gpu_phase_sp.sh 2>&1 | grep -E "==|kernel|selection|key_select"
