#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spec in 64:128 64:256 32:64 32:16; do set -- ${spec//:/ }
  echo "C=$(( $1 * $1 )) k=$2: $(SLC_LIB=build/variants/libslc_pt.so python tools/bench_paths.py --workload llama2-7b --shard-of 8 --block $1 --k $2 --R 20 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -A1 'paths over' | tr '\n' ' ')"
  BLOCK=$1 K=$2 NRANKS=8 WS=1 SLC_LIB=build/variants/libslc_pt.so python tools/phase_timing.py llama2-7b 2>&1 | grep -v Warn | head -12
done
