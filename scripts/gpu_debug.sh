mkdir -p gpurun_out
timeout 600 python bench.py --workload tiny --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/dbg_plain.log 2>&1; echo "plain rc=$?"
tail -2 gpurun_out/dbg_plain.log | cut -c1-300
