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

The copies are plain cudaMemcpyAsync over the host link (torch copy_ with
non_blocking on pinned memory); every arithmetic step of the path still runs in
libslc.so.  The bound of the two swaps is host-link bandwidth (4 B/param each
way), the second roofline of DESIGN.md's f3 section.
"""
from __future__ import annotations

import torch

from . import slc


class EFOffload:
    def __init__(self, plan: slc.Plan, device=None, release: bool = False):
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
