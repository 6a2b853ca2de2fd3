# multi-GPU bench (one process per GPU, NCCL)
mkdir -p gpurun_out
N=${N:-2}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 10 --warmup 3 ${EXTRA} > gpurun_out/bench_n$N.log 2>&1; echo "rc=$?"
tail -n 1 gpurun_out/bench_n$N.log | cut -c1-2500
grep -iE "error|Traceback" gpurun_out/bench_n$N.log | head -5
