set -x
mkdir -p gpurun_out
nvidia-smi -L
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log
