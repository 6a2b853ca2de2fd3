#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544"
out=gpurun_out/coll_n$N.log; : > $out
nvidia-smi topo -m >> $out 2>&1
for sz in 28.4 257.5; do
  $TR tools/coll_bench.py --slot-mb $sz >> $out 2>&1
  NCCL_MIN_NCHANNELS=32 $TR tools/coll_bench.py --slot-mb $sz >> $out 2>&1
  NCCL_MIN_NCHANNELS=64 NCCL_P2P_NET_CHUNKSIZE=524288 $TR tools/coll_bench.py --slot-mb $sz >> $out 2>&1
  NCCL_NVLS_ENABLE=0 $TR tools/coll_bench.py --slot-mb $sz >> $out 2>&1
  NCCL_PROTO=Simple NCCL_ALGO=Ring $TR tools/coll_bench.py --slot-mb $sz >> $out 2>&1
done
NCCL_DEBUG=INFO $TR tools/coll_bench.py --slot-mb 257.5 > gpurun_out/coll_debug_n$N.log 2>&1
