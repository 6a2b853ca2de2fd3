mkdir -p gpurun_out
CMD="python bench.py --workload covenant-72b --shard-of 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/p72_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches72.csv $CMD > gpurun_out/ncu72_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress_ws|agg_pipe" -s 21 -c 2 -o gpurun_out/prof72 $CMD > gpurun_out/ncu72.log 2>&1
echo rc=$?
tail -n 1 gpurun_out/p72_plain.log | cut -c1-200
