"""Round-2 pins for the oracle's readings (VERDICT r1 "What's weak #1"): each
test fixes one reading of DESIGN.md §3 with a hand-worked case
(tests/golden/oracle_pins.json, derivations cited there) or with exact
rational arithmetic, so that the plausible slips of tools/oracle_mutants.py
(partial-chunk tau, the bucket boundary, the tau fallback, the tree order,
fp64 weighted products, canonical peer order, the invR product, the sign of
-0, the fused outer step) each fail at least one of them.  No GPU."""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
from helpers import pack_record, record_from_values

G = oracle.geom()


# ---------------------------------------------------------------- exact rounding helpers (no oracle code)
def rn_fraction(x: Fraction, mant: int, emin: int) -> Fraction:
    """Round the rational x to the nearest binary float with `mant` significand
    bits and minimum normal exponent emin (subnormals below), ties to even.
    Overflow is not modelled (callers stay in range)."""
    if x == 0:
        return Fraction(0)
    s = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    e = max(e, emin)
    q = Fraction(2) ** (e - mant + 1)           # spacing at this exponent
    t = a / q
    n = t.numerator // t.denominator
    r = t - n
    if r > Fraction(1, 2) or (r == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return s * n * q


def rn32(x: Fraction) -> np.float32:
    return np.float32(float(rn_fraction(x, 24, -126)))


def rnbf(x: Fraction) -> Fraction:
    return rn_fraction(x, 8, -126)


def F(x) -> Fraction:
    return Fraction(float(x))


def _f16(hexstr: str) -> np.float32:
    return np.uint16(int(hexstr, 16)).view(np.float16).astype(np.float32)


def _expand(ranges, n):
    v = np.zeros(n, np.float32)
    for a, b, x in ranges:
        v[a:b] = x
    return v


# ---------------------------------------------------------------- quantiser readings (R#1, R#10, R#25)
@pytest.mark.parametrize("case", range(5))
def test_quantizer_hand_worked_cases(golden, case):
    c = golden["oracle_pins"]["quantizer"][case]
    g = oracle.geom(block=c["block"], k=c["k"])
    n = c["n"]
    a = _expand(c["values"], n)
    l = np.zeros(n, np.float32)
    e = np.zeros(n, np.float32)
    for p in c.get("negative_zero_positions", []):
        a[p] = np.float32(-0.0)
        e[p] = np.float32(-0.0)
    st, rec, en = oracle.compress_chunk(a, l, e, 0.95, g)
    assert st == oracle.OK
    assert oracle.effective_k(n, g) == c["k_eff"]
    pos, dq = oracle.decode_chunk(rec, n, g)
    if "selected" in c:
        want_pos = list(range(*c["selected"]))
    else:
        want_pos = [p for r in c["selected_ranges"] for p in range(*r)]
    assert pos.tolist() == want_pos
    assert rec[-1] & 0xFFFF == int(c["scale_lo_f16"], 16), hex(rec[-1] & 0xFFFF)
    assert rec[-1] >> 16 == int(c["scale_hi_f16"], 16), hex(rec[-1] >> 16)
    if "decode" in c:
        dense = np.zeros(n, np.float32)
        dense[pos] = dq
        assert np.array_equal(dense, _expand(c["decode"], n))
    if "sign_bit_slots" in c:
        iw = (g.k * g.index_bits + 31) // 32
        cw = (2 * g.k + 31) // 32
        code = sum(int(rec[iw + i]) << (32 * i) for i in range(cw))
        signs = [j for j in range(c["k_eff"]) if (code >> (2 * j)) & 1]
        buckets = [j for j in range(c["k_eff"]) if (code >> (2 * j + 1)) & 1]
        assert signs == c["sign_bit_slots"] and buckets == c["bucket_bit_slots"]
        for p in c["negative_zero_positions"]:
            assert en[p].view(np.uint32) == 0          # -0 - (-0) = +0
            assert dq[want_pos.index(p)].view(np.uint32) == 0x80000000   # decoded -0


def test_spec_constant_example_scale_hi_is_tau(golden):
    """S:124 constant input [5, 5, 5]: no value exceeds tau = 5, so the empty
    high bucket takes the tau fallback: both scales are 5."""
    g = oracle.geom(block=2, k=4)
    v = np.full(3, 5.0, np.float32)
    st, rec, _ = oracle.compress_chunk(v, np.zeros(3, np.float32), np.zeros(3, np.float32), 0.95, g)
    assert st == 0 and rec[-1] & 0xFFFF == 0x4500 and rec[-1] >> 16 == 0x4500


def test_partial_chunks_threshold_is_mean_of_k_eff_values():
    """Property form of R#10 + S:120 on random partial chunks: the bucket split
    is at the mean of the k_eff transmitted magnitudes (exact rationals), with
    |v| == tau in the low bucket; scales are the fp16-rounded bucket means."""
    rng = np.random.default_rng(21)
    for n in [2048, 1000, 3000, 130]:
        ke = oracle.effective_k(n, G)
        for _ in range(10):
            # small integers: every tree sum is exact, so tau and the bucket means are exact rationals
            v = (rng.integers(1, 50, n) * rng.choice([-1, 1], n)).astype(np.float32)
            st, rec, _ = oracle.compress_chunk(v, np.zeros(n, np.float32), np.zeros(n, np.float32), 0.95, G)
            assert st == 0
            pos, dq = oracle.decode_chunk(rec, n, G)
            m = [Fraction(int(abs(v[p]))) for p in pos]
            tau = rn32(sum(m) / ke)          # fp32 division of an exact sum
            hi = [x for x in m if x > F(tau)]
            lo = [x for x in m if x <= F(tau)]
            s_hi = np.float16(rn32(sum(hi) / len(hi))) if hi else np.float16(tau)
            s_lo = np.float16(rn32(sum(lo) / len(lo))) if lo else np.float16(0)
            assert rec[-1] >> 16 == s_hi.view(np.uint16) and rec[-1] & 0xFFFF == s_lo.view(np.uint16)
            assert all(abs(d) == np.float32(s_hi if x > F(tau) else s_lo) for d, x in zip(dq, m))


# ---------------------------------------------------------------- tree sum topology (R#13)
BIG = np.float32(2.0 ** 24)


def _r13_join_first(k, a, b, c):
    """Do slots a and b meet before either meets slot c in R#13's tree?
    R#13: lane l = s mod 32 sums its slots l, l+32, l+64, ... left to right;
    the 32 lane sums are then folded with strides 16, 8, 4, 2, 1, so lanes x
    and y meet at the fold of stride 2^(lowest bit where x and y differ)."""
    def lane(s):
        return s % 32

    def rank(s):          # position of slot s in its lane's chain
        return s // 32

    la, lb, lc = lane(a), lane(b), lane(c)
    if la == lb:
        if lc != la:
            return True
        return rank(c) > max(rank(a), rank(b))
    if lc == la or lc == lb:
        return False

    def t(x, y):          # fold step at which lanes x and y meet (0 = stride 16)
        d = x ^ y
        return 4 - ((d & -d).bit_length() - 1)
    return t(la, lb) < t(la, lc) and t(la, lb) < t(lb, lc)


def _probe(k, n, a, b, c):
    x = np.zeros(n, np.float32)
    x[a] = 1.0
    x[b] = 1.0
    x[c] = BIG
    return oracle.tree_sum(x, k)


def test_tree_sum_all_triples_k64():
    """2^24 at slot c and 1.0 at slots a, b: the fp32 sum is 2^24 + 2 exactly
    when a and b are added together before either meets 2^24 (else each 1 is
    rounded away: 2^24 + 1 ties to the even 2^24).  A rooted binary tree is
    determined by its rooted triples, so checking every triple against R#13's
    description pins the whole reduction order for k = 64."""
    k = 64
    for a, b in itertools.combinations(range(k), 2):
        for c in range(k):
            if c in (a, b):
                continue
            got = _probe(k, k, a, b, c)
            want = np.float32(2.0 ** 24 + 2) if _r13_join_first(k, a, b, c) else BIG
            assert got == want, (a, b, c, float(got))


@pytest.mark.parametrize("k", [32, 96, 256])
def test_tree_sum_sampled_triples_other_k(k):
    rng = np.random.default_rng(k)
    K = 32 * ((k + 31) // 32)
    for _ in range(20000):
        a, b, c = rng.choice(K, 3, replace=False)
        got = _probe(k, K, int(a), int(b), int(c))
        want = np.float32(2.0 ** 24 + 2) if _r13_join_first(k, int(a), int(b), int(c)) else BIG
        assert got == want, (k, a, b, c)


def test_tree_sum_hand_worked_probes():
    # k = 64: slots l and l+32 meet first (R#13 lane sums), lanes 0/16 before 0/1
    assert _probe(64, 64, 0, 32, 1) == np.float32(2.0 ** 24 + 2)
    assert _probe(64, 64, 0, 16, 1) == np.float32(2.0 ** 24 + 2)
    assert _probe(64, 64, 0, 1, 16) == BIG
    # k = 256: lane chains are left to right (slots 0, 32 before 64; 64, 96 after 0)
    assert _probe(256, 256, 0, 32, 64) == np.float32(2.0 ** 24 + 2)
    assert _probe(256, 256, 64, 96, 0) == BIG
    # padding: n < K slots are +0
    x = np.zeros(40, np.float32); x[3] = 1.5
    assert oracle.tree_sum(x, 64) == np.float32(1.5)


# ---------------------------------------------------------------- weighted aggregation (R#17, R#20)
def _rec_at(g, pos_vals, n):
    return record_from_values(pos_vals, n, oracle.effective_k(n, g), g.k, g.index_bits)


@pytest.mark.parametrize("case", [0, 1])
def test_canonical_peer_order_hand_worked(golden, case):
    c = golden["oracle_pins"]["aggregate_order"][case]
    n = 4096
    recs = [_rec_at(G, {0: p["dq"]}, n) for p in c["peers"]]
    ids = np.zeros((3, 16), np.uint8)
    for i, p in enumerate(c["peers"]):
        ids[i, 15] = p["id"]
    w = np.array([p["w"] for p in c["peers"]], np.float32)
    order = c["pass_order"]
    d = oracle.aggregate_chunk([recs[i] for i in order], n, peer_ids=ids[order], weights=w[order])
    assert d[0] == np.float32(c["delta"])
    assert d[1:].view(np.uint32).max() == 0


def test_delta_is_acc_times_inv_r_hand_worked(golden):
    c = golden["oracle_pins"]["aggregate_inv_r"]
    R, n = c["R"], 4096
    assert Fraction(1.0 / R) < Fraction(1, R)      # the derivation's premise
    recs = []
    for r in range(R):
        if r < len(c["parts_units_2^-24"]):
            recs.append(_rec_at(G, {0: c["parts_units_2^-24"][r] * 2.0 ** -24}, n))
        else:
            recs.append(_rec_at(G, {1 + r: 0.5}, n))
    d = oracle.aggregate_chunk(recs, n)
    assert d[0] == np.float32(c["delta"]) and d[0] != np.float32(c["delta_if_divided"])
    assert sum(F(x) for x in c["parts_units_2^-24"]) * Fraction(1, 2 ** 24) == 49 * Fraction(33550435, 2 ** 24)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_weighted_aggregate_equals_exact_weighted_mean(R):
    """w_r * dq_r is exact in fp64 (24 + 11 significand bits) and, with weights
    in [0.5, 2) and scales in [0.5, 2), so is every partial sum; with R a power
    of two Delta is then the correctly rounded exact weighted mean (R#17, R#20)."""
    rng = np.random.default_rng(30 + R)
    n = 4096
    for trial in range(6):
        w = rng.uniform(0.5, 2.0, R).astype(np.float32)
        w[0] = np.float32(1.0) + np.float32(2.0 ** -23)   # full-width mantissa
        recs, exact = [], [Fraction(0)] * n
        for r in range(R):
            pos = np.sort(rng.choice(n, 64, replace=False)) if trial % 2 else np.arange(64) * 3
            codes = rng.integers(0, 4, 64)
            lo = np.float16(rng.uniform(0.5, 1.0)).view(np.uint16)
            hi = np.float16(rng.uniform(1.0, 2.0)).view(np.uint16)
            recs.append(pack_record(pos, codes, lo, hi, 64, 12))
            S = [F(np.uint16(lo).view(np.float16)), F(np.uint16(hi).view(np.float16))]
            for p, cd in zip(pos, codes):
                v = S[(cd >> 1) & 1] * (-1 if cd & 1 else 1)
                exact[p] += F(w[r]) * v
        ids = rng.integers(0, 256, (R, 16)).astype(np.uint8)
        d = oracle.aggregate_chunk(recs, n, peer_ids=ids, weights=w)
        want = np.array([rn32(x / R) for x in exact], np.float32)
        assert np.array_equal(d.view(np.uint32), want.view(np.uint32))


# ---------------------------------------------------------------- outer step rounding (R#18)
def test_outer_update_f32_is_one_rounding_of_exact():
    """theta <- fma(-alpha, Delta, theta): a single rounding of the exact
    theta - alpha*Delta (alpha = 0.65), checked with exact rationals."""
    rng = np.random.default_rng(40)
    theta = (rng.standard_normal(3000) * 0.02).astype(np.float32)
    delta = (rng.standard_normal(3000) * 1e-3).astype(np.float32)
    alpha = np.float32(0.65)
    new = oracle.outer_update(theta, delta, float(alpha))
    want = np.array([rn32(F(t) - F(alpha) * F(d)) for t, d in zip(theta, delta)], np.float32)
    assert np.array_equal(new.view(np.uint32), want.view(np.uint32))
    two_step = np.array([rn32(F(t) - F(rn32(F(alpha) * F(d)))) for t, d in zip(theta, delta)], np.float32)
    assert (two_step != want).sum() > 10      # the case set separates fused from unfused


def _bf16_witnesses(alpha: np.float32):
    """(theta_bf16_bits, Delta) pairs where rnbf(fma32(-alpha, Delta, theta))
    and rnbf(theta - fl32(alpha*Delta)) differ: theta = 1, and alpha*Delta
    placed just under 3*2^-9 - 2^-25 so that the fused fp32 result sits one
    ulp above the bf16 midpoint 1 - 3*2^-9 and the unfused one on it."""
    out = []
    target = Fraction(3, 2 ** 9) - Fraction(1, 2 ** 25)
    d0 = np.float32(float(target / F(alpha)))
    for t in range(-64, 65):
        d = np.float32(d0 + np.float32(t) * np.spacing(d0))
        s = F(alpha) * F(d)
        fused = rnbf(F(rn32(1 - s)))
        unfused = rnbf(F(rn32(1 - F(rn32(s)))))
        if fused != unfused:
            out.append((d, fused))
    return out


def test_outer_update_bf16_is_rnbf_of_fused_fp32():
    """bf16 theta (R#18): rnbf(fma32(-alpha, Delta, f32(theta))) — the fp32 fma
    result is rounded once more to bf16; built cases where an unfused fp32
    evaluation lands on a bf16 tie and rounds the other way."""
    alpha = np.float32(0.65)
    wit = _bf16_witnesses(alpha)
    assert wit, "no separating case found"
    theta = np.full(len(wit), 0x3F80, np.uint16)   # bf16 1.0
    delta = np.array([d for d, _ in wit], np.float32)
    new = oracle.outer_update(theta, delta, float(alpha))
    want = np.array([np.float32(float(f)) for _, f in wit], np.float32).view(np.uint32) >> 16
    assert np.array_equal(new.astype(np.uint32), want.astype(np.uint32))
