"""One-process-per-GPU harness: the two exchange steps of the path that cross
GPUs, done with NCCL through torch.distributed (BASELINE.json north_star: "NCCL
over NVLink is used only to all-gather each GPU's compressed shard payload
into the peer message, and to exchange simulated peers' payloads").

* a8, PayloadGather — the FSDP shards of one peer each compress their own chunk
  range; the peer message (what the paper uploads to R2,
  P:139-145) is the concatenation of the shard payloads in rank order, i.e. in
  global chunk order.  Shard payload sizes differ by a few chunks, so every
  rank's records buffer is padded to the largest shard payload and one
  ncclAllGather moves them; rank g's part sits at byte g*slot of the gathered
  buffer.  The gather runs on NCCL's stream and overlaps the fused
  aggregate/update kernel, which only needs the rank's own slices.
* a9, PeerExchange — stand-in for the R2 download: peer r's full
  message sits on rank r % n "as if downloaded", staged so that what each
  destination needs is contiguous; one all-to-all hands every rank its slice
  of every message.  Reported separately.

No dense tensor ever crosses NVLink.  Works with the gloo backend on CPU
tensors too (tests/test_dist_cpu.py).
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist

from . import slc


def shard_payloads(layout, geom, nranks: int, dtype: str = "f32") -> List[int]:
    """Payload bytes of every rank's shard (host-only plans, no device work)."""
    return [slc.Plan(layout, geom=geom, rank=r, nranks=nranks, dtype=dtype, device=-1).payload_bytes
            for r in range(nranks)]


class PayloadGather:
    """a8: all-gather of the shard payloads into the peer message."""

    def __init__(self, plan: slc.Plan, group=None, device=None):
        self.plan = plan
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.sizes = shard_payloads(plan.layout, plan.geom, self.world, plan.dtype)
        self.slot = max(self.sizes)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.message = torch.zeros(self.world * self.slot, dtype=torch.uint8, device=dev)
        self._work = None

    def alloc_records(self, device=None) -> torch.Tensor:
        """Own records buffer, padded to the gather slot."""
        dev = device if device is not None else self.message.device
        return torch.zeros(self.slot, dtype=torch.uint8, device=dev)

    def start(self, records: torch.Tensor):
        assert records.numel() == self.slot, "records must come from alloc_records()"
        self._work = dist.all_gather_into_tensor(self.message, records, group=self.group, async_op=True)

    def wait(self):
        if self._work is not None:
            self._work.wait()
            self._work = None

    def contiguous_message(self) -> torch.Tensor:
        """The peer message in global chunk order without the padding."""
        return torch.cat([self.message[g * self.slot:g * self.slot + self.sizes[g]] for g in range(self.world)])

    def slice_of(self, message: torch.Tensor, g: int) -> torch.Tensor:
        return message[g * self.slot:g * self.slot + self.sizes[g]]


class PeerMessage:
    """a8 over NVLink peer memory, folded into the compress kernel: the peer
    message (world * slot bytes, rank g's records at g * slot) lives in
    symmetric memory on every rank, and slc_compress_multi stores each record
    both into the rank's own slot and, through the NVLink peer mappings, into
    the same slot of every other rank's message — no separate collective.  A
    device-side barrier (symmetric-memory signal pads) then tells every rank
    that all shards have landed (`wait`).  The own slot doubles as the rank's
    records buffer for the fused update."""

    def __init__(self, plan: slc.Plan, group=None):
        import torch.distributed._symmetric_memory as symm
        self.plan = plan
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.sizes = shard_payloads(plan.layout, plan.geom, self.world, plan.dtype)
        self.slot = (max(self.sizes) + 15) // 16 * 16
        dev = torch.device("cuda", torch.cuda.current_device())
        self.message = symm.empty(self.world * self.slot, dtype=torch.uint8, device=dev)
        self.message.zero_()
        self.handle = symm.rendezvous(self.message, self.group.group_name)
        base = [int(self.handle.buffer_ptrs[g]) for g in range(self.world)]
        own = self.rank * self.slot
        # own slot first (the binding size-checks it), then the same slot of every other rank's message
        self.records = self.message[own:own + self.slot]
        self._outs = [self.records] + [base[g] + own for g in range(self.world) if g != self.rank]

    def compress(self, theta, theta_local, ef, beta: float = 0.95, stream=None):
        self.plan.compress_multi(theta, theta_local, ef, self._outs, beta=beta, stream=stream)

    def wait(self, stream=None):
        """Every rank's records are in every message (device-side barrier on `stream`)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.handle.barrier(channel=0)

    def slice_of(self, g: int) -> torch.Tensor:
        return self.message[g * self.slot:g * self.slot + self.sizes[g]]

    def contiguous_message(self) -> torch.Tensor:
        return torch.cat([self.slice_of(g) for g in range(self.world)])


class PeerExchange:
    """a9: peer r's (padded) message lives on rank r % n; every rank receives
    its own slice of every message.

    The owned messages are staged (as the download would write them) in a
    [dst rank][owned peer][slot] buffer, so that the part every destination
    needs is one contiguous range, and ONE ncclAllToAll-style call
    (all_to_all_single with per-rank split sizes) moves every (peer, dst)
    slice at once; it lands in a [src rank][owned peer of src][slot] buffer.
    `run_p2p` is the earlier grouped send/recv version (one op per (peer,
    dst) pair), kept for comparison in bench.py's collectives report."""

    def __init__(self, gather: PayloadGather, n_peers: int):
        self.g = gather
        self.n_peers = n_peers
        world, rank, slot = gather.world, gather.rank, gather.slot
        dev = gather.message.device
        self.n_own = [len(range(g, n_peers, world)) for g in range(world)]
        self.send = torch.zeros(world * self.n_own[rank] * slot, dtype=torch.uint8, device=dev)
        self.recv = torch.zeros(n_peers * slot, dtype=torch.uint8, device=dev)
        self._roff = [sum(self.n_own[:g]) * slot for g in range(world)]
        self.slices = None  # run_p2p's receive buffers, allocated on first use

    def owner(self, r: int) -> int:
        return r % self.g.world

    def stage(self, i: int, message: torch.Tensor):
        """Place owned peer i's full padded message (peer r = rank + i*world) in the send buffer."""
        world, slot, no = self.g.world, self.g.slot, self.n_own[self.g.rank]
        self.send.view(world, no, slot)[:, i, :].copy_(message.view(world, slot))

    def exchange(self):
        """The one collective: every rank gets its slice of every peer's message."""
        world, rank, slot = self.g.world, self.g.rank, self.g.slot
        dist.all_to_all_single(self.recv, self.send, output_split_sizes=[n * slot for n in self.n_own],
                               input_split_sizes=[self.n_own[rank] * slot] * world, group=self.g.group)

    def slice(self, r: int) -> torch.Tensor:
        """Peer r's slice for this rank (a view into the receive buffer)."""
        src, i = r % self.g.world, r // self.g.world
        o = self._roff[src] + i * self.g.slot
        return self.recv[o:o + self.g.sizes[self.g.rank]]

    def run(self, owned_messages: Sequence[torch.Tensor]):
        """owned_messages[i] = full padded message of peer r = rank + i*world."""
        for i, m in enumerate(owned_messages):
            self.stage(i, m)
        self.exchange()
        return [self.slice(r) for r in range(self.n_peers)]

    def run_p2p(self, owned_messages: Sequence[torch.Tensor]):
        """Grouped send/recv, one op per (peer, destination) slice."""
        world, rank, slot = self.g.world, self.g.rank, self.g.slot
        if self.slices is None:
            self.slices = [torch.zeros(slot, dtype=torch.uint8, device=self.recv.device) for _ in range(self.n_peers)]
        ops = []
        for r in range(self.n_peers):
            o = self.owner(r)
            if o == rank:
                msg = owned_messages[r // world]
                for dst in range(world):
                    part = msg[dst * slot:(dst + 1) * slot]
                    if dst == rank:
                        self.slices[r].copy_(part)
                    else:
                        ops.append(dist.P2POp(dist.isend, part, dst, group=self.g.group))
            else:
                ops.append(dist.P2POp(dist.irecv, self.slices[r], o, group=self.g.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return [s[:self.g.sizes[rank]] for s in self.slices]


class PeerExchangeP2P:
    """a9 over NVLink peer memory: the owners' staged messages live in symmetric
    memory; after a device barrier every rank PULLS its slice of every peer's
    message straight from the owner with one slc_peer_copy kernel (all SMs, all
    links at once), then a second barrier lets the owners re-stage."""

    def __init__(self, plan: slc.Plan, sizes, slot: int, n_peers: int, group=None):
        import torch.distributed._symmetric_memory as symm
        self.plan = plan
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.sizes, self.slot, self.n_peers = list(sizes), slot, n_peers
        self.n_own_max = (n_peers + self.world - 1) // self.world
        dev = torch.device("cuda", torch.cuda.current_device())
        self.store = symm.empty(max(1, self.n_own_max) * self.world * slot, dtype=torch.uint8, device=dev)
        self.handle = symm.rendezvous(self.store, self.group.group_name)
        self.base = [int(self.handle.buffer_ptrs[g]) for g in range(self.world)]
        self.recv = torch.zeros(n_peers * slot, dtype=torch.uint8, device=dev)
        mine = self.sizes[self.rank]
        msg = self.world * slot
        self.pairs = [(self.base[r % self.world] + (r // self.world) * msg + self.rank * slot,
                       self.recv.data_ptr() + r * slot, mine) for r in range(n_peers)]

    def stage(self, i: int, message: torch.Tensor):
        """Owned peer i's full padded message (peer r = rank + i*world), as the download would write it."""
        msg = self.world * self.slot
        self.store[i * msg:(i + 1) * msg].copy_(message[:msg])

    def exchange(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.handle.barrier(channel=0)   # every owner has staged its messages
            self.plan.peer_copy(self.pairs, stream=s)
            self.handle.barrier(channel=1)   # every pull has finished reading

    def slice(self, r: int) -> torch.Tensor:
        return self.recv[r * self.slot:r * self.slot + self.sizes[self.rank]]

    def run(self, owned_messages: Sequence[torch.Tensor]):
        for i, m in enumerate(owned_messages):
            self.stage(i, m)
        self.exchange()
        return [self.slice(r) for r in range(self.n_peers)]


class MedianNorm:
    """Median-norm weights (reading R#20) for the R peers of one round,
    identical on every rank: each rank computes the exact squared norms of its
    shard of every peer's payload (slc_payload_sqnorm: four un-carried 32-bit
    limbs per peer), one int64 all-reduce (SUM) adds the limbs exactly — the
    only extra collective, 32*R bytes — and slc_median_norm_weights turns them
    into weights on the device.  No host synchronisation."""

    def __init__(self, plan: slc.Plan, n_peers: int, group=None, device=None):
        self.plan = plan
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.limbs = torch.zeros((n_peers, 4), dtype=torch.int64, device=dev)
        self.weights = torch.ones(n_peers, dtype=torch.float32, device=dev)
        self.norms = torch.zeros(n_peers, dtype=torch.float64, device=dev)

    def reduce_limbs(self, limbs: torch.Tensor) -> torch.Tensor:
        """Exact cross-rank sum of the un-carried limbs (each < 2^63 for any realistic job)."""
        if self.world > 1:
            dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=self.group)
        return limbs

    def __call__(self, records: Sequence[torch.Tensor], hdrs=None, stream=None) -> torch.Tensor:
        # the all-reduce is ordered on torch's current stream: run the whole
        # sequence (sqnorm kernel -> all-reduce -> weights kernel) on `stream`
        # made current, so each step sees the previous one's result
        s = stream if stream is not None else torch.cuda.current_stream(self.limbs.device)
        with torch.cuda.stream(s):
            self.plan.payload_sqnorm(records, self.limbs, hdrs=hdrs, stream=s)
            self.reduce_limbs(self.limbs)
            self.plan.median_norm_weights(self.limbs, self.weights, self.norms, stream=s)
        return self.weights
