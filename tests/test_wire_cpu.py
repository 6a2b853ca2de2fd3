"""NEXT row f2 — SLC1 wire format, CPU side: the
oracle's plain bit-string codec pinned by SPEC's worked examples and
invariants, its mapping from the device record layout (R#6) checked against
the C oracle's decoder, and the host parts of the C ABI (65-byte header,
per-shard body layout) checked against the oracle."""
import numpy as np
import pytest

import oracle
from oracle import wire
from helpers import pack_record, shard_chunk_lengths
from slcgen import layouts


def test_pack_indices_spec_examples():
    assert wire.pack_indices([0, 4095]) == bytes([0x00, 0x0F, 0xFF])
    assert wire.pack_indices([]) == b""
    rng = np.random.default_rng(0)
    for _ in range(50):
        x = sorted(rng.choice(4096, int(rng.integers(0, 65)), replace=False).tolist())
        assert wire.unpack_indices(wire.pack_indices(x), len(x)) == x
    with pytest.raises(ValueError):
        wire.pack_indices([4096])


def test_empty_delta_is_65_header_bytes():
    assert len(wire.serialize(0, b"p", b"d" * 32, [])) == 65 == wire.HEADER_BYTES


def test_record_chunk_mapping_matches_oracle_decoder():
    """record_to_chunk's (index, sign*2 + bucket, scales) reproduce the C
    oracle's decoded values, and chunk_to_record inverts it."""
    g = oracle.geom()
    rng = np.random.default_rng(3)
    for _ in range(100):
        n = int(rng.choice([4096, 777]))
        ke = oracle.effective_k(n, g)
        pos = np.sort(rng.choice(n, ke, replace=False))
        codes = rng.integers(0, 4, ke)  # record convention: bit0 sign, bit1 bucket
        lo, hi = sorted(int(x) for x in rng.integers(0, 0x7BFF, 2))
        rec = pack_record(pos, codes, lo, hi, 64, 12)
        idx, sym, l2, h2 = wire.record_to_chunk(rec, ke)
        assert idx == pos.tolist() and (l2, h2) == (lo, hi)
        _, dq = oracle.decode_chunk(rec, n, g)
        S = [np.uint16(lo).view(np.float16).astype(np.float32), np.uint16(hi).view(np.float16).astype(np.float32)]
        want = np.array([-S[s & 1] if s >> 1 else S[s & 1] for s in sym], np.float32)
        assert np.array_equal(dq.view(np.uint32), want.view(np.uint32))
        assert wire.chunk_to_record(idx, sym, l2, h2) == [int(w) for w in rec]


def test_serialize_roundtrip_on_oracle_compress_output():
    g = oracle.geom()
    rng = np.random.default_rng(4)
    shape = (128, 192)
    a = rng.normal(0, 0.02, shape).astype(np.float32)
    l = (a - rng.normal(0, 1e-3, shape)).astype(np.float32)
    recs, _ = oracle.compress_tensor(shape, a, l, np.zeros(a.size, np.float32), 0.95, g=g)
    chunks = [wire.record_to_chunk(r, 64) for r in recs]
    buf = wire.serialize(7, b"peer", b"\x11" * 32, chunks)
    assert len(buf) == 65 + len(chunks) * wire.chunk_wire_bytes(64)
    br, pid, dig, back = wire.deserialize(buf, [4096] * len(chunks), [64] * len(chunks))
    assert br == 7 and dig == b"\x11" * 32 and back == chunks
    for r, c in zip(recs, back):
        assert wire.chunk_to_record(*c) == [int(w) for w in r]


def test_deserialize_errors():
    chunks = [([1, 5, 9] + list(range(10, 71)), [0] * 64, 0x1000, 0x2000)]
    ok = wire.serialize(1, b"x", b"y" * 32, chunks)
    wire.deserialize(ok, [4096], [64])
    with pytest.raises(wire.FormatError):
        wire.deserialize(b"SLC2" + ok[4:], [4096], [64])          # magic
    with pytest.raises(wire.FormatError):
        wire.deserialize(ok[:4] + b"\x02" + ok[5:], [4096], [64])  # version
    with pytest.raises(wire.FormatError):
        wire.deserialize(ok[:-1], [4096], [64])                    # truncated
    with pytest.raises(wire.FormatError):
        wire.deserialize(ok + b"\0", [4096], [64])                 # trailing
    bad_order = [([5, 1] + list(range(10, 72)), [0] * 64, 0x1000, 0x2000)]
    with pytest.raises(wire.InvalidData):
        wire.deserialize(wire.serialize(1, b"x", b"y" * 32, bad_order), [4096], [64])
    bad_scale = [(chunks[0][0], [0] * 64, 0x2000, 0x1000)]           # lo > hi
    with pytest.raises(wire.InvalidData):
        wire.deserialize(wire.serialize(1, b"x", b"y" * 32, bad_scale), [4096], [64])
    with pytest.raises(wire.InvalidData):
        wire.deserialize(ok, [4096], [63])                         # count != k_eff


def test_c_abi_header_and_body_layout():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_08163_b200 import slc
    layout = layouts.LAYOUTS["ragged"]
    full = slc.Plan(layout, device=-1)
    hdr = slc.make_header(full, b"peer-0001", base_round=42)
    h = slc.wire_header_write(hdr, full.info.total_chunks)
    assert h == wire.serialize(42, b"peer-0001", full.digest, [])[:61] + \
        full.info.total_chunks.to_bytes(4, "big")
    back, n = slc.wire_header_read(h)
    assert n == full.info.total_chunks and back.base_round == 42 and bytes(back.peer_id)[:9] == b"peer-0001"
    for bad in (h[:64], b"XLC1" + h[4:], h[:4] + b"\x07" + h[5:]):
        with pytest.raises(slc.SlcError) as e:
            slc.wire_header_read(bad)
        assert e.value.status == slc.FORMAT_ERROR
    # body layout: shards tile the body contiguously; sizes follow S:143 per chunk
    g = oracle.geom()
    total = sum(wire.chunk_wire_bytes(oracle.effective_k(n, g)) for n in shard_chunk_lengths(full))
    assert full.wire_layout() == (total, 0)
    for nranks in (2, 3, 5):
        off = 0
        for r in range(nranks):
            p = slc.Plan(layout, rank=r, nranks=nranks, device=-1)
            b, o = p.wire_layout()
            assert o == off
            assert b == sum(wire.chunk_wire_bytes(oracle.effective_k(n, g)) for n in shard_chunk_lengths(p))
            off += b
        assert off == total
