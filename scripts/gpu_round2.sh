#!/bin/bash
# round-2 evidence pass: GPU tests, smoke, bench lines (default, reference arm, 72B shard f32/bf16/median-norm),
# compress robustness, config-5 sweep, row f4 at R=20/64, launch list + ncu --set full of the default step
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; tail -n 1 $O/bench.log > $O/bench.json; cut -c1-300 $O/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; tail -n 1 $O/bench_ref.log > $O/bench_ref.json; cut -c1-200 $O/bench_ref.json
B72="python bench.py --workload covenant-72b --shard-of 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for a in "--dtype f32" "--dtype bf16" "--dtype f32 --median-norm" "--dtype bf16 --median-norm" "--dtype f32 --shard-rank 7"; do
  timeout 900 $B72 $a > $O/b72.log 2>&1; echo "$a $(tail -n 1 $O/b72.log)" >> $O/b72_lines.txt
done
B1="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for a in "" "--special-period 32" "--special-period 8" "--dtype bf16" "--dtype bf16 --cold-ef" "--cold-ef" "--dtype bf16 --special-period 32"; do
  timeout 600 $B1 $a > $O/b1.log 2>&1; echo "[$a] $(tail -n 1 $O/b1.log)" >> $O/robust_lines.txt
done
bash scripts/gpu_sweep2.sh > /dev/null 2>&1; cp gpurun_out/sweep2.txt $O/sweep.txt
for R in 20 64; do
  timeout 1200 $B72 --dtype f32 --R $R --index-code --steps 3 > $O/bidx.log 2>&1; echo "R=$R $(tail -n 1 $O/bidx.log)" >> $O/index_code_lines.txt
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"compress_ws|compress_fallback|agg_pipe" -s 24 -c 3 -o $O/prof_step $CMD > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls $O
