"""Compress parity on crafted chunks that drive every selection path of the
warp selector (warp_select.cuh): the candidate rank path, key_select (more
than CAP candidates, at most XCAP: a tied level crossing the top k), tie_select
(the k-th key is the smallest candidate key: whole-chunk constants, fewer than
k nonzeros), and the radix fallback (a large tied level above distinct
values).  Top-k with ties going to the lower position (R#3, R#4) makes the
records unique, so they must equal the oracle's bit for bit, as must e.

Inputs: theta = 0, theta_local = -d, e = 0, so b = d exactly (P:68-75 with a
cold EF); d per 64x64 block (or 4096-run of a 1-D tensor) follows one of the
patterns below, on top of distinct "normal" magnitudes in [2^-12, 2^-10)."""
import numpy as np
import pytest

import oracle
from helpers import bits, seg_shape, seg_view

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")
LAYOUT = [("w", (640, 576)), ("ragged", (100, 200)), ("v", (4096 * 9 + 17,))]
N_PATTERNS = 10


def _pattern(rng, shape, kind):
    """d for one 2-D block (rows, cols) or 1-D run (n,) of pattern `kind`."""
    n = int(np.prod(shape))
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0).astype(np.float32)
    d = (rng.uniform(2.0 ** -12, 2.0 ** -10, n).astype(np.float32) * sgn).reshape(shape)
    flat = d.reshape(-1)
    two_d = len(shape) == 2
    rows = (lambda r0, r1: (slice(r0, r1), slice(None))) if two_d else (lambda r0, r1: slice(64 * r0, 64 * r1))
    if kind == 1:    # two rows at one value above everything: 128 tied, top 64 by position (key_select)
        d[rows(5, 7)] = np.float32(2.0 ** -9)
    elif kind == 2:  # two rows at a value inside the normal range
        d[rows(10, 12)] = np.float32(-(2.0 ** -11))
    elif kind == 3:  # 40 distinct large + one row tied below them: K* = the tie, 24 of 64 taken
        d[rows(20, 21)] = np.float32(2.0 ** -9)
        idx = rng.choice(n, 40, replace=False)
        idx = idx[(idx // 64) != 20] if two_d else idx[(idx // 64) != 20]
        flat[idx] = rng.uniform(2.0 ** -8, 2.0 ** -7, idx.size).astype(np.float32) * sgn[idx]
    elif kind == 4:  # eight rows tied on top: 512 candidates (> XCAP), tie_select / radix
        d[rows(8, 16)] = np.float32(2.0 ** -9) * np.sign(d[rows(8, 16)])
    elif kind == 5:  # three tie levels over four rows
        lv = rng.integers(1, 4, size=d[rows(30, 34)].shape).astype(np.float32)
        d[rows(30, 34)] = lv * np.float32(2.0 ** -9) * np.sign(d[rows(30, 34)])
    elif kind == 6:  # whole chunk one magnitude, random signs (tie_select, A = 0)
        flat[:] = np.float32(2.0 ** -10) * sgn
    elif kind == 7:  # fewer than k nonzeros, the rest signed zeros
        keep = rng.choice(n, 10, replace=False)
        z = np.where(rng.random(n) < 0.5, np.float32(-0.0), np.float32(0.0))
        z[keep] = flat[keep]
        flat[:] = z
    elif kind == 8:  # a tied level crossing k among 2 rows + a spike
        d[rows(40, 42)] = np.float32(2.0 ** -10)
        flat[rng.integers(n)] = np.float32(2.0 ** -4)
    elif kind == 9:  # two partial rows of one value (63 + 65 ties)
        fl = d.reshape(-1)
        fl[64 * 3:64 * 3 + 63] = np.float32(2.0 ** -9)
        fl[64 * 50 + 1:64 * 50 + 66] = np.float32(2.0 ** -9)
    return d


def _crafted(seed, shape, dtype):
    rng = np.random.default_rng(seed)
    if len(shape) == 2:
        d = np.zeros(shape, np.float32)
        R, C = shape
        for bi, r0 in enumerate(range(0, R, 64)):
            for bj, c0 in enumerate(range(0, C, 64)):
                blk = (min(64, R - r0), min(64, C - c0))
                kind = (bi * 7 + bj) % N_PATTERNS
                d[r0:r0 + blk[0], c0:c0 + blk[1]] = _pattern(rng, blk, kind) if min(blk) >= 64 else \
                    _pattern(rng, (64, 64), kind)[:blk[0], :blk[1]]
    else:
        n = shape[0]
        d = np.zeros(n, np.float32)
        for ci, c0 in enumerate(range(0, n, 4096)):
            m = min(4096, n - c0)
            d[c0:c0 + m] = _pattern(rng, (4096,), ci % N_PATTERNS)[:m]
    if dtype == "bf16":  # theta_local = -d must be exact in bf16: keep 8 significant bits
        d = (d.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    return d.reshape(-1)


def _to_dev(x, dtype):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype == "bf16":
        return t.view(torch.int16).to(DEV).view(torch.bfloat16)
    return t.to(DEV)


@pytest.mark.parametrize("dtype,block,k", [("f32", 64, 64), ("bf16", 64, 64), ("f32", 64, 256), ("f32", 32, 64),
                                           ("bf16", 64, 128)])
def test_crafted_selection_paths(dtype, block, k):
    plan = slc.Plan(LAYOUT, geom=slc.geometry(block=block, k=k), dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    theta = torch.zeros(plan.shard_elems, dtype=tdt, device=DEV)
    tl = torch.zeros(plan.shard_elems, dtype=tdt, device=DEV)
    ef = torch.zeros(plan.shard_elems, dtype=torch.float32, device=DEV)
    host = []
    for s in plan.segments:
        d = _crafted(100 + s.tensor, seg_shape(s), dtype)
        neg = (-d).astype(np.float32)
        if dtype == "bf16":
            a = np.zeros(d.size, np.uint16)
            l = (neg.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
        else:
            a = np.zeros(d.size, np.float32)
            l = neg
        seg_view(tl, s).copy_(_to_dev(l, dtype))
        host.append((a, l))
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    plan.compress(theta, tl, ef, rec)
    assert plan.get_status() == slc.OK
    got = rec.cpu().numpy().view(np.uint32)
    g = oracle.geom(block=block, k=k)
    RW = oracle.record_words(g)
    off = 0
    for s, (a, l) in zip(plan.segments, host):
        shape = seg_shape(s)
        ref, en = oracle.compress_tensor(shape, a, l, np.zeros(a.size, np.float32), 0.95, g=g)
        nrec = ref.size
        mism = np.nonzero(got[off:off + nrec] != ref.reshape(-1))[0]
        assert mism.size == 0, f"{s.tensor}: {mism.size} record words differ; first chunks {np.unique(mism // RW)[:8]}"
        off += nrec
        e_dev = seg_view(ef, s).cpu().numpy()
        assert np.array_equal(bits(e_dev), bits(en)), f"{s.tensor}: EF differs"
