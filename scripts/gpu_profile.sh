# profile the bench step: launch list (all kernels) + full set of one compress and one fused update launch
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress_kernel|aggregate_kernel" -s 9 -c 2 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/prof_plain.log gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
