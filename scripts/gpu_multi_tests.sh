#!/bin/bash
# NCCL / NVLink multi-GPU parity (tests/test_gpu_multi.py) + the step and collectives at bench sizes
cd "$GRAFT_REPO_ROOT" || exit 1
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/m_tests_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/m_tests_n$N.log
tail -5 gpurun_out/m_tests_n$N.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for gth in p2p nccl; do
  timeout 900 $TR bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --gather $gth > gpurun_out/m_bench_${gth}_n$N.log 2>&1
  echo "== $gth rc=$?"; tail -1 gpurun_out/m_bench_${gth}_n$N.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['kernels']['compress_ms'], d['kernels']['fused_update_ms'], d['collectives'])"
done
