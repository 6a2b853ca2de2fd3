#!/bin/bash
# round-2 parity tests on one GPU (new files) + the full GPU suite
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_pins.py tests/test_gpu_scale.py -m gpu -q -x --durations=15 > gpurun_out/t_new.log 2>&1
echo "new rc=$?" >> gpurun_out/t_new.log
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_gpu_scale.py --deselect tests/test_gpu_pins.py > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
