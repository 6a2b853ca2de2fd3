mkdir -p gpurun_out
CMD="python bench.py --workload llama2-7b --shard-of 8 --k 256 --R 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/k256_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"compress_ws" -s 3 -c 1 -o gpurun_out/prof_k256 $CMD > gpurun_out/ncu_k256.log 2>&1
echo rc=$?
