#!/bin/bash
# NCCL multi-GPU parity (tests/test_gpu_multi.py) + the a8/a9 collectives at bench sizes
cd "$GRAFT_REPO_ROOT" || exit 1
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/m_tests_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/m_tests_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 10 --warmup 3 --no-e2e > gpurun_out/m_bench_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/m_bench_n$N.log
