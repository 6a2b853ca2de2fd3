#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
VARIANTS="${VARIANTS:-default}" ROUNDS=1 bash scripts/gpu_cmpv.sh
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"; echo "special 8: $($B --special-period 8 | tail -1 | python -c "import sys,json; print(json.load(sys.stdin)['kernels']['compress_ms'])")"
bash scripts/gpu_bpaths.sh 2>&1 | grep -v "^\[\]"
CFGS="--special-period 32" bash scripts/gpu_bkern.sh
