"""Collective micro-benchmark for rows a8 / a9 at the bench's message sizes.

  torchrun --nproc-per-node N tools/coll_bench.py [--slot-mb 257.5] [--peers 20]

Times (CUDA events, max over ranks): all_gather_into_tensor of one padded
shard payload per rank (a8), the staged all_to_all_single exchange (a9), and
a copy-engine peer-to-peer variant of both (cudaMemcpyPeerAsync through torch
.copy_ between devices' IPC-shared buffers is not available across processes,
so only NCCL paths are measured here).  Prints one JSON line from rank 0."""
import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slot-mb", type=float, default=257.5)
    ap.add_argument("--peers", type=int, default=20)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    slot = int(args.slot_mb * 1e6) // 16 * 16
    out = {"world": world, "slot_bytes": slot, "peers": args.peers,
           "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        a.record(s)
        for _ in range(args.reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    mine = torch.full((slot,), rank, dtype=torch.uint8, device=dev)
    msg = torch.empty(world * slot, dtype=torch.uint8, device=dev)
    ms = timed(lambda: dist.all_gather_into_tensor(msg, mine))
    out["allgather_ms"] = ms
    out["allgather_busbw_gbs"] = slot * (world - 1) / (ms * 1e-3) / 1e9
    n_own = [len(range(g, args.peers, world)) for g in range(world)]
    send = torch.ones(world * n_own[rank] * slot, dtype=torch.uint8, device=dev)
    recv = torch.empty(args.peers * slot, dtype=torch.uint8, device=dev)
    ms = timed(lambda: dist.all_to_all_single(recv, send, output_split_sizes=[n * slot for n in n_own],
                                              input_split_sizes=[n_own[rank] * slot] * world))
    out["alltoall_ms"] = ms
    out["alltoall_gbs_per_rank"] = args.peers * slot * (world - 1) / world / (ms * 1e-3) / 1e9
    # one big all-gather of every owned message at once (exchange as all-gather of [n_own, slot] parts)
    del send, recv
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
