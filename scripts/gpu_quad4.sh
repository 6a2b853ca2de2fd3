#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_scale.py tests/test_gpu_pins.py -m gpu -q -x 2>&1 | tail -2
SPECS="64:64 64:128 64:256 32:4 32:16 32:32 32:64 128:64 128:256" bash scripts/gpu_sweep2.sh
VARIANTS="default" ROUNDS=1 bash scripts/gpu_cmpv.sh
