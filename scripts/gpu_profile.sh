# profile the default bench step: launch list (all kernels) + ncu --set full of one compress and one
# fused update launch (after 7 peer compresses + 1 warm-up step); each ncu only after the plain run exits 0
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_EXTRA}"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress|aggregate" -s ${SKIP:-9} -c 2 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
tail -n 1 gpurun_out/prof_plain.log | cut -c1-400
