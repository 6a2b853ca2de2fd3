# 72B shard of 8: readings A/B, fp32/bf16, median-norm, R sweep
mkdir -p gpurun_out
OUT=gpurun_out/sweep72.txt
echo "# one GPU's shard of the 8-GPU Covenant-72B job (9.09 B params), bench.py --steps 5 --warmup 3" > $OUT
run() {
  timeout 900 python bench.py --shard-of 8 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/s72.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/s72.log').read().strip().splitlines()[-1]); k=d['kernels']
print(f'{\" \".join(sys.argv[1:]):50s} step {d[\"ms_per_step\"]:7.2f} ms  compress {k[\"compress_ms\"]:6.2f}  update {k[\"fused_update_ms\"]:6.2f}  hbm_frac {d[\"hbm_frac_of_peak\"]:.3f}  of8TB {d[\"hbm_gbs\"]/8000:.3f}  sm_mhz {d[\"clocks\"][\"sm_mhz\"]} {d[\"clocks\"][\"reasons\"]}')" "$@" >> $OUT 2>&1 || { echo "$@ FAILED" >> $OUT; tail -3 gpurun_out/s72.log >> $OUT; }
}
run --workload covenant-72b
run --workload covenant-72b-b
run --workload covenant-72b --dtype bf16
run --workload covenant-72b-b --dtype bf16
run --workload covenant-72b --median-norm
for R in 2 8 32 64; do run --workload covenant-72b --R $R; done
cat $OUT
