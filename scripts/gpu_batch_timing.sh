#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python tools/build_variants.py bt=SLC_BATCH_TIMING > gpurun_out/bt_build.log 2>&1 || { tail gpurun_out/bt_build.log; exit 1; }
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/bt_build.log 2>&1
SLC_LIB=build/variants/libslc_bt.so python tools/batch_timing.py llama3-8b 4 20 f32
SLC_LIB=build/variants/libslc_bt.so python tools/batch_timing.py llama3-8b 4 20 bf16
