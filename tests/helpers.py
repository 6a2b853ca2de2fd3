"""Test helpers: build a shard's device inputs with slcgen and the oracle's
reference for the same inputs.  (Test infrastructure: may use oracle/.)"""
from __future__ import annotations

import numpy as np

import oracle
import slcgen


def tensor_offsets(layout):
    offs, o = [], 0
    for _, shape in layout:
        offs.append(o)
        o += int(np.prod(shape))
    return offs


def seg_shape(seg):
    return (seg.rows, seg.cols) if seg.blocked else (seg.n_elems,)


def fill_shard(plan, layout, buf, what, seed, peer, **kw):
    offs = tensor_offsets(layout)
    for s in plan.segments:
        slcgen.fill_cuda(buf[s.shard_offset:s.shard_offset + s.n_elems], what, seed, peer,
                         offs[s.tensor] + s.tensor_begin, **kw)


def host_segment(layout, seg, what, seed, peer, dtype="f32", **kw):
    offs = tensor_offsets(layout)
    return slcgen.generate(what, seed, peer, offs[seg.tensor] + seg.tensor_begin, seg.n_elems, dtype=dtype, **kw)


def make_device_inputs(plan, layout, seed, peer, dtype="f32", special_period=0, warm_ef=False, theta=None):
    import torch
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n = plan.shard_elems
    dev = torch.device("cuda", plan.device)
    if theta is None:
        theta = torch.zeros(n, dtype=tdt, device=dev)
        fill_shard(plan, layout, theta, slcgen.WHAT_THETA, seed, peer, special_period=special_period)
    tl = torch.zeros(n, dtype=tdt, device=dev)
    ef = torch.zeros(n, dtype=torch.float32, device=dev)
    fill_shard(plan, layout, tl, slcgen.WHAT_THETA_LOCAL, seed, peer, special_period=special_period)
    fill_shard(plan, layout, ef, slcgen.WHAT_EF, seed, peer, special_period=special_period, warm_ef=warm_ef)
    return theta, tl, ef


def oracle_compress_shard(plan, layout, seed, peer, dtype="f32", special_period=0, warm_ef=False, beta=0.95,
                          g=None):
    """Oracle records (uint32, shard chunk order) and per-segment EF for the shard."""
    g = g or oracle.geom(plan.geom.block, plan.geom.k, plan.geom.index_bits)
    recs, efs, thetas = [], [], []
    for s in plan.segments:
        a = host_segment(layout, s, slcgen.WHAT_THETA, seed, peer, dtype, special_period=special_period)
        l = host_segment(layout, s, slcgen.WHAT_THETA_LOCAL, seed, peer, dtype, special_period=special_period)
        e = host_segment(layout, s, slcgen.WHAT_EF, seed, peer, special_period=special_period, warm_ef=warm_ef)
        r, en = oracle.compress_tensor(seg_shape(s), a, l, e, beta, g=g)
        recs.append(r.reshape(-1))
        efs.append(en)
        thetas.append(a)
    return np.concatenate(recs) if recs else np.zeros(0, np.uint32), efs, thetas


def oracle_update_shard(plan, thetas, peer_recs, alpha, peer_ids=None, weights=None, g=None, only_delta=False):
    """Per-segment oracle theta after the outer step (or Delta if only_delta)."""
    g = g or oracle.geom(plan.geom.block, plan.geom.k, plan.geom.index_bits)
    RW = oracle.record_words(g)
    out, off = [], 0
    for s, th in zip(plan.segments, thetas):
        nrec = s.n_chunks * RW
        per = [pr[off:off + nrec] for pr in peer_recs]
        off += nrec
        if only_delta:
            out.append(oracle.aggregate_tensor(seg_shape(s), per, peer_ids=peer_ids, weights=weights, g=g))
        else:
            out.append(oracle.aggregate_update_tensor(seg_shape(s), th, per, alpha, peer_ids=peer_ids,
                                                      weights=weights, g=g))
    return out


def seg_view(buf, s):
    return buf[s.shard_offset:s.shard_offset + s.n_elems]


def bits(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    return x.view(np.uint16 if x.dtype.itemsize == 2 else np.uint32)
