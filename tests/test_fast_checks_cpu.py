"""Row f2 fast checks, CPU oracle pinned by SPEC's worked
examples and by hand-built payloads (reading R#29)."""
import numpy as np

import oracle
from helpers import pack_record
from oracle import fast_checks as fc


def _payload(scale_bits, n=4096, k=64, lo=0x3C00):
    """One chunk: 64 entries in the high bucket with fp16 scale `scale_bits`."""
    return [(pack_record(np.arange(k) * 7, np.full(k, 2), lo, scale_bits, 64, 12), n)]


def test_spec_examples(golden):
    ok = _payload(0x3C00)                  # norm = sqrt(64) = 8
    # S:360 "stale base-round -> {sync}"
    assert fc.fast_checks(ok, current_round=5, base_round=4) == fc.SYNC
    # S:361 "well-formed on-time submission -> empty set"
    assert fc.fast_checks(ok, current_round=5, base_round=5, norm_history=[8.0, 8.0, 9.0]) == 0
    # S:362 "norm 100x median history -> {norm-sane}"
    assert fc.fast_checks(ok, current_round=5, base_round=5, norm_history=[0.08, 0.08, 0.1]) == fc.NORM


def test_threshold_is_ten_times_the_lower_median():
    p = _payload(0x3C00)  # norm exactly 8
    assert oracle.payload_norm(p) == 8.0
    # lower median of [0.8, 0.81, 5, 6] is 0.81 -> bound 8.1 -> pass; of [0.7, 0.8, 5, 6] is 0.8 -> 8.0: not > -> pass
    assert fc.fast_checks(p, 0, norm_history=[0.8, 0.81, 5.0, 6.0]) == 0
    assert fc.fast_checks(p, 0, norm_history=[0.7, 0.8, 5.0, 6.0]) == 0
    assert fc.fast_checks(p, 0, norm_history=[0.7, 0.79, 5.0, 6.0]) == fc.NORM
    assert fc.fast_checks(p, 0, norm_history=[]) == 0


def test_liveness_digest_and_finite():
    assert fc.fast_checks(None, 3) == fc.LIVENESS
    p = _payload(0x3C00)
    assert fc.fast_checks(p, 3, base_round=3, digest=b"a" * 32, expected_digest=b"b" * 32) == fc.SYNC
    inf = _payload(0x7C00)  # +Inf high-bucket scale, used by every entry
    assert fc.fast_checks(inf, 3, base_round=3, norm_history=[1.0]) == fc.FINITE
    # an Inf scale in the unused low bucket decodes to nothing: finite
    unused = _payload(0x3C00, lo=0x7C00)
    assert fc.fast_checks(unused, 3, norm_history=[1.0]) == 0
