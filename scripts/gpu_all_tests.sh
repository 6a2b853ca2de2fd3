#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/at_build.log 2>&1 || { tail -20 gpurun_out/at_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/at_tests.log 2>&1
echo "rc=$?" >> gpurun_out/at_tests.log
tail -16 gpurun_out/at_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
