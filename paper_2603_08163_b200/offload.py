"""NEXT row f3: host-offloaded error-feedback buffer.

PAPER.md P:118-132 (§3) and the Fig. 1 caption: the EF buffer is
sharded like the inner-optimizer state, kept in host memory while the H inner
steps run, swapped into GPU memory for the compression of the outer step and
swapped out again, the swap-out overlapped with communication.  Here:

* `host`  — the shard's e_r in pinned host memory (fp32, [shard_elems]); the
  copy that persists between outer steps.
* `dev`   — the device swap buffer that slc_compress updates in place.  It is
  only live between swap_in() and the end of swap_out(); `release=True` hands
  it back to the caching allocator after every swap-out (the memory the paper
  frees for the inner state), at the price of a re-allocation per step.
* swap_in(stream): H2D on a dedicated copy stream; `stream` waits on it.
* swap_out(stream): the copy stream waits for the compress already enqueued
  on `stream`, then D2H — it runs while `stream` goes on with the payload
  all-gather and the fused decode/aggregate/outer update (which never read e).
* wait(stream): `stream` waits for the swap-out (before the next swap_in or a
  host read of `host`).
* compress_pipelined(...): the shard cut into `n_pieces` runs of whole chunk
  rows (each a contiguous element range): piece j's swap-in (H2D stream),
  compress (slc_compress_range on `stream`) and swap-out (D2H stream) form a
  three-stage pipeline, so the full-duplex host link carries the swap-in of
  piece j+1 and the swap-out of piece j-1 at once and the step approaches
  max(H2D, D2H) instead of their sum.

The copies are plain cudaMemcpyAsync over the host link (torch copy_ with
non_blocking on pinned memory); every arithmetic step of the path still runs in
libslc.so.  The bound of the two swaps is host-link bandwidth (4 B/param each
way), the second roofline of DESIGN.md's f3 section.
"""
from __future__ import annotations

import torch

from . import slc


class EFOffload:
    def __init__(self, plan: slc.Plan, device=None, release: bool = False, n_pieces: int = 16):
        if not torch.cuda.is_available():
            raise RuntimeError("EFOffload needs a CUDA device (the EF swap targets GPU memory)")
        self.plan = plan
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = plan.shard_elems
        self.host = torch.zeros(n, dtype=torch.float32, pin_memory=True)
        self.release = release
        self.dev = None if release else torch.empty(n, dtype=torch.float32, device=self.device)
        self.copy_stream = torch.cuda.Stream(self.device)
        self._in_done = torch.cuda.Event()
        self._compressed = torch.cuda.Event()
        self._out_done = torch.cuda.Event()
        self._out_done.record(self.copy_stream)
        self.d2h_stream = torch.cuda.Stream(self.device)
        self.pieces = shard_pieces(plan, n_pieces)
        self._ev_in = [torch.cuda.Event() for _ in self.pieces]
        self._ev_c = [torch.cuda.Event() for _ in self.pieces]

    @property
    def bytes_per_swap(self) -> int:
        return self.host.numel() * 4

    def swap_in(self, stream=None) -> torch.Tensor:
        """Host -> device copy of e_r (after the inner steps); returns the device buffer."""
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cs = self.copy_stream
        cs.wait_event(self._out_done)
        with torch.cuda.stream(cs):
            if self.dev is None:
                self.dev = torch.empty(self.host.numel(), dtype=torch.float32, device=self.device)
            self.dev.copy_(self.host, non_blocking=True)
            self._in_done.record(cs)
        stream.wait_event(self._in_done)
        self.dev.record_stream(stream)
        return self.dev

    def swap_out(self, stream=None) -> None:
        """Device -> host copy of e_r^(t+1), ordered after the compress on `stream`, overlapping what
        `stream` does next ("swapped out ... overlapped with communication")."""
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cs = self.copy_stream
        self._compressed.record(stream)
        cs.wait_event(self._compressed)
        with torch.cuda.stream(cs):
            self.host.copy_(self.dev, non_blocking=True)
            self._out_done.record(cs)
        if self.release:
            self.dev.record_stream(cs)
            self.dev = None

    def wait(self, stream=None) -> None:
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        stream.wait_event(self._out_done)

    def compress(self, theta, theta_local, records, beta: float = 0.95, stream=None) -> None:
        """One outer step's compression with the EF swapped in and out around slc_compress."""
        ef = self.swap_in(stream)
        self.plan.compress(theta, theta_local, ef, records, beta=beta, stream=stream)
        self.swap_out(stream)

    def compress_pipelined(self, theta, theta_local, records, beta: float = 0.95, stream=None) -> None:
        """Swap-in / compress / swap-out of the pieces as a three-stage pipeline (see module doc)."""
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h2d, d2h = self.copy_stream, self.d2h_stream
        h2d.wait_event(self._out_done)
        with torch.cuda.stream(h2d):
            if self.dev is None:
                self.dev = torch.empty(self.host.numel(), dtype=torch.float32, device=self.device)
            for (_, _, e0, e1), ev in zip(self.pieces, self._ev_in):
                self.dev[e0:e1].copy_(self.host[e0:e1], non_blocking=True)
                ev.record(h2d)
        self.dev.record_stream(stream)
        for (c0, nc, e0, e1), ev_in, ev_c in zip(self.pieces, self._ev_in, self._ev_c):
            stream.wait_event(ev_in)
            self.plan.compress_range(c0, nc, theta, theta_local, self.dev, records, beta=beta, stream=stream)
            ev_c.record(stream)
            d2h.wait_event(ev_c)
            with torch.cuda.stream(d2h):
                self.host[e0:e1].copy_(self.dev[e0:e1], non_blocking=True)
        self._out_done.record(d2h)
        if self.release:
            self.dev.record_stream(d2h)
            self.dev = None


def shard_pieces(plan: slc.Plan, n_pieces: int = 16):
    """Cut the shard's chunk sequence into about n_pieces runs of whole chunk rows (a 64-row block row of a
    blocked slice, one chunk of a flat one), so that every run is a contiguous element range of the shard
    buffers.  Returns [(chunk_begin, n_chunks, elem_begin, elem_end)] covering every chunk once, in order."""
    B = plan.geom.block
    C = B * B
    target = max(1, -(-plan.shard_elems // max(1, n_pieces)))
    pieces, c = [], 0
    cur = None  # [c0, nc, e0, e1]
    for s in plan.segments:
        if s.blocked:
            nbc = -(-s.cols // B)
            units = [(nbc, s.shard_offset + i * B * s.cols, s.shard_offset + min((i + 1) * B, s.rows) * s.cols)
                     for i in range(-(-s.rows // B))]
        else:
            units = [(1, s.shard_offset + j * C, s.shard_offset + min((j + 1) * C, s.n_elems))
                     for j in range(-(-s.n_elems // C))]
        for nc, e0, e1 in units:
            if cur is None:
                cur = [c, 0, e0, e1]
            cur[1] += nc
            cur[3] = e1
            c += nc
            if cur[3] - cur[2] >= target:
                pieces.append(tuple(cur))
                cur = None
    if cur is not None:
        pieces.append(tuple(cur))
    assert c == plan.n_chunks, (c, plan.n_chunks)
    return pieces
