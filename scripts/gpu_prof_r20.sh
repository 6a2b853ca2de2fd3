mkdir -p gpurun_out
CMD="python bench.py --workload llama3-8b --shard-of 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r20_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"agg_pipe|compress_ws" -s 20 -c 2 -o gpurun_out/prof_r20 $CMD > gpurun_out/ncu_r20.log 2>&1
echo rc=$?
tail -n 1 gpurun_out/r20_plain.log | cut -c1-300
