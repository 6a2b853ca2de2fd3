"""CPU tests of the C-ABI library: it loads, exports every symbol include/slc.h
declares, and its host-side logic (geometry checks, FSDP-style partition,
record size, digest) is right.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from slcgen import layouts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def slc():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_08163_b200 import slc as m
    return m


def test_exports_every_declared_symbol(slc):
    hdr = open(os.path.join(ROOT, "include", "slc.h")).read()
    declared = set(re.findall(r"\b(slc_[a-z_]+)\s*\(", hdr))
    assert {"slc_compress", "slc_decode_aggregate", "slc_outer_update", "slc_plan_create"} <= declared
    lib = ctypes.CDLL(slc.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(slc.EXPORTED) == declared


def test_record_bytes_and_geometry_checks(slc):
    assert slc.record_bytes(slc.geometry()) == 116
    for block, k in [(32, 16), (64, 16), (64, 128), (64, 256), (128, 256)]:
        g = slc.geometry(block, k)
        assert slc.record_bytes(g) == 4 * oracle.record_words(oracle.geom(block, k))
    bad = slc.Geometry(64, 4000, 64, 12)
    assert slc.record_bytes(bad) == -1
    with pytest.raises(slc.SlcError) as ei:
        slc.Plan([("w", (64, 64))], geom=slc.geometry(16, 8), device=-1)
    assert ei.value.status == slc.UNSUPPORTED
    with pytest.raises(slc.SlcError) as ei:
        slc.Plan([("w", (64, 64))], rank=2, nranks=2, device=-1)
    assert ei.value.status == slc.INVALID_ARGUMENT


@pytest.mark.parametrize("name", ["ragged", "llama3.2-1b", "llama3-8b", "covenant-72b", "1m-2d"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_partition(slc, name, nranks):
    layout = layouts.LAYOUTS[name]
    total = layouts.total_params(layout)
    tchunks = [oracle.tensor_chunks(s) for _, s in layout]
    tstart = np.concatenate([[0], np.cumsum(tchunks)])
    first = 0
    elems = []
    for r in range(nranks):
        p = slc.Plan(layout, rank=r, nranks=nranks, device=-1)
        assert p.info.total_elems == total and p.info.total_chunks == sum(tchunks)
        assert p.info.first_chunk == first
        first += p.n_chunks
        assert p.payload_bytes == p.n_chunks * 116
        n = 0
        prev_end = 0
        for s in p.segments:
            shape = layout[s.tensor][1]
            assert s.shard_offset % 64 == 0 and s.shard_offset >= prev_end
            prev_end = s.shard_offset + s.n_elems
            assert s.blocked == oracle.is_blocked(shape)
            # slice starts on a chunk (flat) or block-row (blocked) boundary and matches oracle chunk ids
            if s.blocked:
                assert s.tensor_begin % (64 * shape[1]) == 0 and s.rows % 64 == 0 and s.cols == shape[1]
                c0 = s.tensor_begin // (64 * shape[1]) * (shape[1] // 64)
            else:
                assert s.tensor_begin % 4096 == 0
                c0 = s.tensor_begin // 4096
            assert s.first_chunk == tstart[s.tensor] + c0
            n += s.n_elems
        assert p.shard_elems == prev_end
        elems.append(n)
    assert first == sum(tchunks) and sum(elems) == total
    if nranks > 1 and name != "ragged":
        # balanced to within one unit (a 64-row band of the widest tensor)
        assert max(elems) - min(elems) <= 2 * 64 * max(s[-1] for _, s in layout if len(s) == 2)


def test_digest(slc):
    g = slc.geometry()
    a = slc.layout_digest(g, [("w", (64, 64))])
    assert a == slc.layout_digest(g, [("x", (64, 64))]) and len(a) == 32
    assert a != slc.layout_digest(g, [("w", (64, 128))])
    assert a != slc.layout_digest(slc.geometry(64, 32), [("w", (64, 64))])


def test_ef_offload_needs_cuda():
    """Row f3's swap targets GPU memory: without a device it fails loudly (no host-side fallback)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2603_08163_b200 import slc
    from paper_2603_08163_b200.offload import EFOffload
    from slcgen import layouts
    plan = slc.Plan(layouts.LAYOUTS["ragged"], device=-1)
    with pytest.raises(RuntimeError, match="CUDA"):
        EFOffload(plan)


@pytest.mark.parametrize("name", ["ragged", "1m-2d", "1m-1d", "llama-tiny"])
@pytest.mark.parametrize("nranks", [1, 3])
@pytest.mark.parametrize("n_pieces", [1, 2, 7, 1000])
def test_shard_pieces_cover_shard(name, nranks, n_pieces):
    """Row f3's swap pieces: in chunk order, every chunk exactly once, disjoint increasing element ranges, and
    every segment's elements inside the pieces (so the piecewise swap moves all of e)."""
    from paper_2603_08163_b200 import slc
    from paper_2603_08163_b200.offload import shard_pieces
    for r in range(nranks):
        plan = slc.Plan(layouts.LAYOUTS[name], rank=r, nranks=nranks, device=-1)
        pcs = shard_pieces(plan, n_pieces)
        c = 0
        for c0, nc, e0, e1 in pcs:
            assert c0 == c and nc > 0 and e1 > e0
            c += nc
        assert c == plan.n_chunks
        assert all(a[3] <= b[2] for a, b in zip(pcs, pcs[1:]))
        covered = np.zeros(plan.shard_elems, bool)
        for _, _, e0, e1 in pcs:
            covered[e0:e1] = True
        for s in plan.segments:
            assert covered[s.shard_offset:s.shard_offset + s.n_elems].all()
        # each piece's chunk count equals the chunks its element range holds
        for c0, nc, e0, e1 in pcs:
            B = plan.geom.block
            n = 0
            for s in plan.segments:
                lo, hi = max(e0, s.shard_offset), min(e1, s.shard_offset + s.n_elems)
                if hi <= lo:
                    continue
                if s.blocked:
                    assert (lo - s.shard_offset) % (B * s.cols) == 0
                    n += -(-((hi - lo) // s.cols) // B) * -(-s.cols // B)
                else:
                    n += -(-(hi - lo) // (B * B))
            assert n == nc
