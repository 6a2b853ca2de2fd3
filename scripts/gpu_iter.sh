# one build->measure iteration: GPU tests, smoke, bench, then an ncu capture of the step's two kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_EXTRA}"
if [ "$PROFILE" = "1" ]; then
  $CMD > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"compress|aggregate" -s ${SKIP:-9} -c 2 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1
fi
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; tail -n 1 gpurun_out/bench.log | cut -c1-1500
