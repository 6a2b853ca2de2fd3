#!/bin/bash
# compress: parity (special chunks exercise tie_select) + timings clean / degenerate / bf16 cold EF
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pins.py tests/test_gpu_scale.py -m gpu -q -x -k "compress or quantizer or cold or wide or sharding or geometry" 2>&1 | tail -2
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
show() { tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'compress', round(d['kernels']['compress_ms'],3), 'frac', round(d['roofline']['frac'],3))"; }
echo "1b clean $($B 2>&1 | show)"
for sp in 32 8; do echo "1b special $sp $($B --special-period $sp 2>&1 | show)"; done
echo "1b bf16 $($B --dtype bf16 2>&1 | show)"
echo "1b bf16 cold $($B --dtype bf16 --cold-ef 2>&1 | show)"
echo "1b f32 cold $($B --cold-ef 2>&1 | show)"
