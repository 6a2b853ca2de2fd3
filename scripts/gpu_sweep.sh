# BASELINE configs[4]: chunk-size / k / peer-count sweep on one GPU's shard of Llama-2-7B over 8 GPUs
mkdir -p gpurun_out
OUT=gpurun_out/sweep.txt
echo "# llama2-7b shard 0 of 8 (842M params/GPU), fp32, bench.py --steps 5 --warmup 3; C k R density -> ms/step compress update  step-HBM-frac(measured peak)" > $OUT
run() {  # block k R
  timeout 600 python bench.py --workload llama2-7b --shard-of 8 --block $1 --k $2 --R $3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); k=d['kernels']
C=$1*$1; print(f'C={C:6d} k={$2:4d} R={$3:3d} density={$2/C*100:5.2f}%  step {d[\"ms_per_step\"]:7.3f} ms  compress {k[\"compress_ms\"]:7.3f}  update {k[\"fused_update_ms\"]:7.3f}  hbm_frac {d[\"hbm_frac_of_peak\"]:.3f}  sm_mhz {d[\"clocks\"][\"sm_mhz\"]}')" >> $OUT 2>&1 || { echo "C=$1 k=$2 R=$3 FAILED" >> $OUT; tail -3 gpurun_out/sw.log >> $OUT; }
}
for R in 2 4 8 16 20 32 64; do run 64 64 $R; done
for k in 16 32 128 256; do run 64 $k 20; done
run 32 16 20
run 128 256 20
cat $OUT
