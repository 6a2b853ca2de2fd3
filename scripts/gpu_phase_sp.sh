#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for sp in 0 32; do echo "== special $sp"; SPECIAL=$sp WS=1 SLC_LIB=build/variants/libslc_pt.so python tools/phase_timing.py llama3.2-1b; done
echo "== bf16 cold"; COLD=1 DTYPE=bf16 WS=1 SLC_LIB=build/variants/libslc_pt.so python tools/phase_timing.py llama3.2-1b
