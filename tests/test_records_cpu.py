"""The test-side record packer (helpers.pack_record, used to craft payloads
with chosen scale ranges for the GPU decode tests) agrees with the oracle's
decoder (R#6 layout), and crafted payloads aggregate through the oracle."""
import numpy as np

import oracle
from helpers import pack_record


def test_pack_record_roundtrip_through_oracle_decode():
    g = oracle.geom()
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.choice([4096, 2048, 100, 1]))
        ke = oracle.effective_k(n, g)
        pos = np.sort(rng.choice(n, ke, replace=False))
        codes = rng.integers(0, 4, ke)
        lo = (int(rng.integers(0, 31)) << 10) | int(rng.integers(0, 1024))
        hi = (int(rng.integers(0, 31)) << 10) | int(rng.integers(0, 1024))
        rec = pack_record(pos, codes, lo, hi, 64, 12)
        assert rec.size == oracle.record_words(g)
        p2, dq = oracle.decode_chunk(rec, n, g)[:2]
        S = [np.uint16(lo).view(np.float16).astype(np.float32), np.uint16(hi).view(np.float16).astype(np.float32)]
        want = np.array([-S[(c >> 1) & 1] if c & 1 else S[(c >> 1) & 1] for c in codes], np.float32)
        assert np.array_equal(p2[:ke], pos)
        assert np.array_equal(dq[:ke].view(np.uint32), want.view(np.uint32))
