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


def shard_chunk_lengths(plan, g=None):
    """Positions per chunk of the shard, in shard chunk order."""
    g = g or oracle.geom(plan.geom.block, plan.geom.k, plan.geom.index_bits)
    C = plan.geom.chunk
    out = []
    for s in plan.segments:
        shape = seg_shape(s)
        nc = oracle.tensor_chunks(shape, g)
        if oracle.is_blocked(shape, g):
            out += [C] * nc
        else:
            n = int(np.prod(shape))
            out += [min(C, n - c * C) for c in range(nc)]
    return out


def pack_record(pos, codes, s_lo_bits, s_hi_bits, k, ib):
    """One record in the R#6 layout: slot j's index at stream
    bits [ib*j, ib*j+ib), code bits 2j (sign) / 2j+1 (bucket) of the code
    stream, last word s_lo | s_hi << 16; unused slots zero."""
    iw = (k * ib + 31) // 32
    cw = (2 * k + 31) // 32
    words = np.zeros(iw + cw + 1, np.uint64)
    for j, p in enumerate(pos):
        b = ib * j
        words[b // 32] |= np.uint64((int(p) << (b % 32)) & 0xFFFFFFFF)
        if b % 32 + ib > 32:
            words[b // 32 + 1] |= np.uint64(int(p) >> (32 - b % 32))
        words[iw + (2 * j) // 32] |= np.uint64(int(codes[j]) << ((2 * j) % 32))
    words[-1] = np.uint64(int(s_lo_bits) | (int(s_hi_bits) << 16))
    return words.astype(np.uint32)


def craft_records(plan, rng, exp_lo, exp_hi, zero_frac=0.05):
    """A random but well-formed payload for the shard: per chunk k_eff distinct
    ascending positions, random 2-bit codes and two fp16 scales whose exponent
    fields are uniform in [exp_lo, exp_hi] (0 = subnormal), some zero."""
    g = oracle.geom(plan.geom.block, plan.geom.k, plan.geom.index_bits)
    k, ib = plan.geom.k, plan.geom.index_bits
    out = []
    for n in shard_chunk_lengths(plan, g):
        ke = oracle.effective_k(n, g)
        pos = np.sort(rng.choice(n, ke, replace=False))
        codes = rng.integers(0, 4, ke)
        sc = []
        for _ in range(2):
            if rng.random() < zero_frac:
                sc.append(0)
            else:
                sc.append((int(rng.integers(exp_lo, exp_hi + 1)) << 10) | int(rng.integers(0, 1024)))
        out.append(pack_record(pos, codes, sc[0], sc[1], k, ib))
    return np.concatenate(out) if out else np.zeros(0, np.uint32)


def record_from_values(pos_vals, n, k_eff, k=64, ib=12):
    """A record (R#6 layout) whose decoded entries are exactly {position: value}
    (at most two distinct nonzero magnitudes; a single magnitude goes to the
    high bucket with S_lo = 0), padded to k_eff entries with zero-valued low
    entries at the lowest unused positions."""
    items = sorted(pos_vals.items())
    mags = sorted({abs(float(v)) for _, v in items if v != 0})
    assert len(mags) <= 2 and len(items) <= k_eff
    if len(mags) == 2:
        lo, hi = mags
    else:
        lo, hi = 0.0, (mags[0] if mags else 0.0)
    pos, codes = [], []
    for p, v in items:
        pos.append(p)
        codes.append((1 if v < 0 else 0) | (2 if (abs(float(v)) == hi and hi != lo) else 0))
    used = set(pos)
    for p in range(n):
        if len(pos) == k_eff:
            break
        if p not in used:
            pos.append(p)
            codes.append(0)
    order = np.argsort(pos)
    return pack_record(np.array(pos)[order], np.array(codes)[order], np.float16(lo).view(np.uint16),
                       np.float16(hi).view(np.uint16), k, ib)
