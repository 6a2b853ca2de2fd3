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
        slices = ex.run(owned)           # staged all-to-all
        ok_ex = all(torch.equal(slices[r], _pattern(plan.info.first_chunk, plan.n_chunks, rb, r))
                    for r in range(n_peers))
        slices = ex.run_p2p(owned)       # grouped send/recv
        ok_ex &= all(torch.equal(slices[r], _pattern(plan.info.first_chunk, plan.n_chunks, rb, r))
                     for r in range(n_peers))
        q.put((rank, ok_gather, ok_ex))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout_name,n_peers", [(2, "ragged", 5), (3, "llama3.2-1b", 4), (3, "ragged", 2)])
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


def _median_worker(rank, world, port, q):
    """Each rank holds the exact squared norms of its shard of R crafted payloads
    as 32-bit limbs (host stand-in for slc_payload_sqnorm); MedianNorm's int64
    all-reduce must reproduce the whole payloads' exact sums on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__
        __graft_entry__.build()
        from fractions import Fraction

        import oracle
        from helpers import craft_records, shard_chunk_lengths
        from paper_2603_08163_b200 import slc
        from paper_2603_08163_b200.dist import MedianNorm
        layout = layouts.LAYOUTS["ragged"]
        full = slc.Plan(layout, device=-1)
        rng = np.random.default_rng(5)
        R = 4
        recs = [craft_records(full, rng, 0, 30) for _ in range(R)]  # same on every rank (seeded)
        RW = full.record_bytes // 4
        lens = shard_chunk_lengths(full)

        def sq_units(rec, c0, c1):
            t = Fraction(0)
            for c in range(c0, c1):
                _, dq = oracle.decode_chunk(rec[c * RW:(c + 1) * RW], lens[c])
                t += sum(Fraction(float(x)) ** 2 for x in dq)
            return int(t * (1 << 48))

        p = slc.Plan(layout, rank=rank, nranks=world, device=-1)
        c0, c1 = p.info.first_chunk, p.info.first_chunk + p.n_chunks
        mine = [sq_units(r, c0, c1) for r in recs]
        limbs = torch.tensor([[(v >> (32 * i)) & 0xFFFFFFFF for i in range(4)] for v in mine], dtype=torch.int64)
        mn = MedianNorm.__new__(MedianNorm)
        mn.group, mn.world = None, world
        mn.reduce_limbs(limbs)
        got = [sum(int(x) << (32 * i) for i, x in enumerate(row)) for row in limbs.tolist()]
        want = [sq_units(r, 0, full.n_chunks) for r in recs]
        q.put((rank, got == want))
    finally:
        dist.destroy_process_group()


def test_median_norm_limb_allreduce_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_median_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
