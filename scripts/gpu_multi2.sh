# N-GPU bench (default workload llama3-8b R=20), plain and median-norm, plus the 72B job shard check
mkdir -p gpurun_out
N=${N:-2}
nvidia-smi -L
for mn in "" "--median-norm"; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 10 --warmup 3 $mn > gpurun_out/bench_n${N}$mn.log 2>&1; echo "rc=$?"
  tail -n 1 gpurun_out/bench_n${N}$mn.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mn', d['value'], d['ms_per_step'], d['kernels'], d.get('collectives'), d['clocks'], d.get('e2e'))" || tail -20 gpurun_out/bench_n${N}$mn.log
done
