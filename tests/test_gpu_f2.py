"""Row f2 fast checks through the C ABI vs the CPU oracle
(oracle/fast_checks.py, reading R#29), on crafted payloads of a sharded layout:
a good peer, a stale one, a non-finite one (Inf scale in a used bucket), one
with an Inf scale in an unused bucket (finite), a 100x-norm one and a missing
one; the norm check uses the exact payload norms (slc_payload_sqnorm limbs)."""
import numpy as np
import pytest

import oracle
from helpers import craft_records, shard_chunk_lengths
from oracle import fast_checks as fc
from slcgen import layouts

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")


def _set_scale(rec_words, RW, which, bits, chunk=0):
    w = rec_words.copy()
    row = w.reshape(-1, RW)[chunk]
    if which == "hi":
        row[-1] = (row[-1] & 0xFFFF) | (bits << 16)
    else:
        row[-1] = (row[-1] & 0xFFFF0000) | bits
    return w


@pytest.mark.parametrize("name", ["ragged", "1m-2d"])
def test_fast_checks_parity(name):
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout)
    RW = plan.record_bytes // 4
    rng = np.random.default_rng(7)
    base = [craft_records(plan, rng, 8, 14, zero_frac=0.0) for _ in range(6)]
    # peer 2: +Inf in the high bucket of chunk 0, with at least one high code there
    row = base[2].reshape(-1, RW)[0]
    row[24] |= 2  # slot 0's bucket bit
    base[2] = _set_scale(base[2], RW, "hi", 0x7C00)
    # peer 3: NaN in the low bucket of a chunk where every code is high -> unused
    row = base[3].reshape(-1, RW)[1]
    row[24:28] |= np.uint32(0xAAAAAAAA)
    base[3] = _set_scale(base[3], RW, "lo", 0x7E00, chunk=1)
    # peer 4: scales x 2^10 -> norm ~1000x the others
    w4 = base[4].reshape(-1, RW)
    lo, hi = w4[:, -1] & 0x3FF, (w4[:, -1] >> 16) & 0x3FF
    w4[:, -1] = (lo | (24 << 10)) | ((hi | (24 << 10)) << 16)
    recs = [torch.from_numpy(b.view(np.uint8).copy()).to(DEV) for b in base]
    recs_in = list(recs)
    recs_in[5] = None  # peer 5: nothing arrived
    hdrs = [slc.make_header(plan, bytes([r + 1]) * 16, base_round=9) for r in range(6)]
    hdrs[1].base_round = 8  # stale
    sq = torch.zeros((6, 4), dtype=torch.int64, device=DEV)
    plan.payload_sqnorm(recs, sq)
    plan.get_status()  # the Inf scales latch INVALID_DATA in sqnorm; cleared here
    lens = shard_chunk_lengths(plan)
    chunks = [[(b[c * RW:(c + 1) * RW], n) for c, n in enumerate(lens)] for b in base]
    good_norms = [oracle.payload_norm(chunks[r]) for r in (0, 1)]
    history = [good_norms[0], good_norms[1], good_norms[0] * 1.5]
    flags = torch.full((6,), -1, dtype=torch.int32, device=DEV)
    plan.fast_checks(recs_in, flags, current_round=9, hdrs=hdrs, sqnorm=sq, norm_history=history)
    got = flags.cpu().numpy().tolist()
    want = [fc.fast_checks(None if r == 5 else chunks[r], 9, history, base_round=hdrs[r].base_round,
                           digest=bytes(hdrs[r].layout_digest), expected_digest=plan.digest) for r in range(6)]
    assert want == [0, fc.SYNC, fc.FINITE, 0, fc.NORM, fc.LIVENESS]
    assert got == want
    # no history: no norm check; no headers: no sync check
    plan.fast_checks(recs_in, flags, current_round=9, sqnorm=sq)
    assert flags.cpu().numpy().tolist() == [0, 0, fc.FINITE, 0, 0, fc.LIVENESS]
