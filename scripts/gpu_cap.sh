#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in cap192 cap256; do SLC_LIB=build/variants/libslc_$v.so timeout 600 python -m pytest tests/test_gpu_select_paths.py tests/test_gpu_parity.py -m gpu -q -x -k "select or compress" 2>&1 | tail -1; done
VARIANTS="default cap192 cap256" ROUNDS=1 bash scripts/gpu_cmpv.sh
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in default cap192 cap256; do L=build/variants/libslc_$v.so; [ $v = default ] && L=paper_2603_08163_b200/libslc.so; echo "$v special 8: $(SLC_LIB=$L $B --special-period 8 | tail -1 | python -c "import sys,json; print(json.load(sys.stdin)['kernels']['compress_ms'])")"; done
