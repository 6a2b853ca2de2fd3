"""Multi-process host logic of the N > 1 path on CPU (gloo, world_size 2 and 3):
the payload all-gather (a8) assembles the peer message in global chunk order,
and the simulated-peer exchange (a9) hands each rank its slice of every peer's
message.  Record bytes are stand-ins (each shard's payload filled with a
pattern derived from its global chunk ids); the kernels are not involved."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from slcgen import layouts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pattern(first_chunk, n_chunks, rb, peer):
    ids = np.repeat(np.arange(first_chunk, first_chunk + n_chunks, dtype=np.int64), rb)
    pos = np.tile(np.arange(rb, dtype=np.int64), n_chunks)
    return torch.from_numpy(((ids * 131 + pos * 7 + peer * 29) % 251).astype(np.uint8))


def _worker(rank, world, port, layout_name, n_peers, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__
        __graft_entry__.build()
        from paper_2603_08163_b200 import slc
        from paper_2603_08163_b200.dist import PayloadGather, PeerExchange
        layout = layouts.LAYOUTS[layout_name]
        plan = slc.Plan(layout, rank=rank, nranks=world, device=-1)
        cpu = torch.device("cpu")
        gather = PayloadGather(plan, device=cpu)
        rb = plan.record_bytes
        # a8: own payload -> message
        rec = gather.alloc_records(cpu)
        rec[:plan.payload_bytes] = _pattern(plan.info.first_chunk, plan.n_chunks, rb, 0)
        gather.start(rec)
        gather.wait()
        msg = gather.contiguous_message()
        expect = _pattern(0, plan.info.total_chunks, rb, 0)
        ok_gather = torch.equal(msg, expect)
        # a9: peer r's padded message on rank r % world
        ex = PeerExchange(gather, n_peers)
        owned = []
        for r in range(rank, n_peers, world):
            m = torch.zeros(world * gather.slot, dtype=torch.uint8)
            for g in range(world):
                pg = slc.Plan(layout, rank=g, nranks=world, device=-1)
                m[g * gather.slot:g * gather.slot + pg.payload_bytes] = _pattern(pg.info.first_chunk, pg.n_chunks,
                                                                                 rb, r)
            owned.append(m)
        slices = ex.run(owned)
        ok_ex = all(torch.equal(slices[r], _pattern(plan.info.first_chunk, plan.n_chunks, rb, r))
                    for r in range(n_peers))
        q.put((rank, ok_gather, ok_ex))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout_name,n_peers", [(2, "ragged", 5), (3, "llama3.2-1b", 4)])
def test_gather_and_exchange_gloo(world, layout_name, n_peers):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout_name, n_peers, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(g and e for _, g, e in res), res
