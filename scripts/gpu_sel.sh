#!/bin/bash
# selection paths: crafted parity + compress parity, then timings and path counts
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_select_paths.py -m gpu -q -x 2>&1 | tail -15
bash scripts/gpu_compress.sh
bash scripts/gpu_phase_sp.sh 2>&1 | grep -E "==|kernel|selection|cycles per call|key_select|R rank"
