#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_select_paths.py -m gpu -q 2>&1 | grep -E "Error|assert |passed|failed|FAILED" | head -12
SLC_LIB=build/variants/libslc_checked.so timeout 600 python -m pytest tests/test_gpu_select_paths.py -m gpu -q -x 2>&1 | grep -E "SLC_CHECK|Error|passed|failed" | head -8
