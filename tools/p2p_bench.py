"""NVLink peer-memory copy bandwidth with torch symmetric memory (rows a8 / a9):
   torchrun --nproc-per-node N tools/p2p_bench.py [--mb 257.5]
pull of one `mb` slice from every other rank: (a) copy engines (tensor.copy_ of
the peer view, one stream per peer), (b) one slc_peer_copy kernel (all SMs)."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08163_b200 import slc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=257.5)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    slot = int(args.mb * 1e6) // 16 * 16
    buf = symm.empty(slot, dtype=torch.uint8, device=dev)
    buf.fill_(rank)
    h = symm.rendezvous(buf, dist.group.WORLD.group_name)
    out = torch.empty(world * slot, dtype=torch.uint8, device=dev)
    plan = slc.Plan([("w", (4096,))], device=local)
    peers = [g for g in range(world) if g != rank]
    views = [h.get_buffer(g, (slot,), torch.uint8) for g in peers]
    streams = [torch.cuda.Stream() for _ in peers]
    s0 = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def ce():
        for v, st, g in zip(views, streams, peers):
            st.wait_stream(s0)
            with torch.cuda.stream(st):
                out[g * slot:(g + 1) * slot].copy_(v)
        for st in streams:
            s0.wait_stream(st)

    pairs = [(int(h.buffer_ptrs[g]), out.data_ptr() + g * slot, slot) for g in peers]

    def sm():
        plan.peer_copy(pairs, stream=s0)

    # exchange-like: 20 segments of slot/2 bytes, alternating local and remote sources
    seg = slot // 2 // 16 * 16
    ex_pairs = []
    for r in range(20):
        owner = r % world
        src = (int(h.buffer_ptrs[owner]) if owner != rank else buf.data_ptr()) + (r // world % 2) * seg
        ex_pairs.append((src, out.data_ptr() + (r % world) * slot + (r // world % 2) * seg, seg))

    def smx():
        plan.peer_copy(ex_pairs, stream=s0)

    res = {"world": world, "slot_bytes": slot}
    for name, fn in (("copy_engine", ce), ("sm_kernel", sm), ("sm_exchange20", smx)):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        a.record(s0)
        for _ in range(args.reps):
            fn()
        b.record(s0)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        res[name + "_ms"] = ms
        nbytes = slot * (world - 1) if name != "sm_exchange20" else 20 * seg
        res[name + "_gbs_per_rank"] = nbytes / (ms * 1e-3) / 1e9
        ok = all(bool((out[g * slot:g * slot + 1024] == g).all()) for g in peers)
        res[name + "_ok"] = ok
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
