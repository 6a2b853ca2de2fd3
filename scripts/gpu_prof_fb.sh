#!/bin/bash
# ncu --set full of the compress fallback kernel (special-period 32) and of the main kernel
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 3 --special-period ${SP:-32} --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"compress_fallback" -s ${SKIP:-3} -c 1 -o gpurun_out/prof_fb_sp${SP:-32} $CMD > gpurun_out/pfb_ncu.log 2>&1
tail -2 gpurun_out/pfb_ncu.log
