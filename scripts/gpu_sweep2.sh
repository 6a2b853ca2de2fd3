#!/bin/bash
# config-5 sweep (llama2-7b shard of 8): compress ms and roofline fraction per (C, k), R=20
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
OUT=gpurun_out/sweep2.txt
: > $OUT
run() {  # block k R [extra]
  timeout 600 python bench.py --workload llama2-7b --shard-of 8 --block $1 --k $2 --R $3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $4 > gpurun_out/sw.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); k=d['kernels']
C=$1*$1; print(f'C={C:6d} k={$2:4d} R={$3:3d} density={$2/C*100:5.2f}% $4 step {d[\"ms_per_step\"]:7.3f} ms  compress {k[\"compress_ms\"]:7.3f} (frac {d[\"roofline\"][\"frac\"]:.3f})  update {k[\"fused_update_ms\"]:7.3f}  sm_mhz {d[\"clocks\"][\"sm_mhz\"]}')" >> $OUT 2>&1 || { echo "C=$1 k=$2 R=$3 FAILED" >> $OUT; tail -3 gpurun_out/sw.log >> $OUT; }
}
for spec in ${SPECS:-64:64 64:16 64:32 64:128 64:256 32:4 32:16 32:64 128:64 128:256}; do set -- ${spec//:/ }; run $1 $2 20 "$3"; done
cat $OUT
