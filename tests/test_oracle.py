"""Pins for the CPU oracle (oracle/, test infrastructure) — no GPU needed.

Each test pins the oracle to something other than itself: values printed in
PAPER.md, SPEC.md worked examples (tests/golden/), closed forms, brute force
on tiny inputs, exact rational arithmetic, and independent library routines
(numpy float16, torch bfloat16).  A plausible slip in the oracle (dropped beta,
wrong sign in the EF update, transposed block index, wrong tie-break, wrong
divisor in the mean) fails at least one of them.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from slcgen import layouts

G = oracle.geom()  # 64x64 / 4096 / k=64 / 12 bits


def ulp32(x: float) -> float:
    x = abs(np.float32(x))
    if x == 0:
        return float(np.float32(2.0 ** -149))
    return float(np.spacing(x))


# ------------------------------------------------------------------ printed values
def test_paper_printed_values(golden):
    pv = golden["paper_values"]
    C, k = pv["chunk_size_C"]["value"], pv["top_k"]["value"]
    assert C == G.chunk == G.block ** 2 and pv["block_side"]["value"] == G.block and k == G.k
    assert G.index_bits == pv["index_bits_per_value"]["value"]
    eb = oracle.index_entropy_bound(C, k)
    assert abs(eb - pv["index_entropy_bound_bits_per_value"]["value"]) < pv["index_entropy_bound_bits_per_value"]["tolerance"]
    # idealised ratio: dense fp32 over (index bits + value bits) per transmitted value
    r = oracle.compression_ratio(C, k, 32, pv["index_bits_per_value"]["value"] + pv["value_bits"]["value"])
    assert r > pv["compression_ratio_more_than"]["value"]
    assert abs(r - 32 * 4096 / (64 * 14)) < 1e-12
    # actual record: k*12 + k*2 bits + 2 fp16 scales = 29 words = 116 bytes
    assert oracle.record_words(G) * 4 == 116
    assert 4 * C / (oracle.record_words(G) * 4) > 140  # measured ratio incl. scales


def test_entropy_bound_brute_force():
    # binom by exact integer arithmetic, not lgamma
    for C, k in [(8, 2), (16, 5), (4096, 64), (1024, 16), (16384, 256)]:
        exact = math.log2(math.comb(C, k)) / k
        assert abs(oracle.index_entropy_bound(C, k) - exact) < 1e-9


def test_72b_layout_matches_paper(golden):
    pv = golden["paper_values"]
    lay = layouts.LAYOUTS["covenant-72b"]
    assert layouts.total_params(lay) == pv["covenant_72b_parameters"]["value"]
    sh = pv["covenant_72b_shape"]["value"]
    assert lay[0][1] == (sh["vocab"], sh["d_model"])
    assert sum(1 for n, _ in lay if n.endswith(".q")) == sh["layers"]
    q = dict(lay)["l0.q"]; kk = dict(lay)["l0.k"]
    assert q == (8192, 8192) and kk == (8192 // sh["q_heads"] * sh["kv_heads"], 8192)
    assert "lm_head" not in dict(lay)  # tied
    assert layouts.total_params(layouts.LAYOUTS["covenant-72b-b"]) == pv["covenant_72b_parameters"]["value"]


# ------------------------------------------------------------------ geometry
def test_spec_chunk_examples(golden):
    for ex in golden["spec_examples"]["chunk_tensor"]:
        shape = tuple(ex["shape"])
        assert oracle.tensor_chunks(shape) == ex["chunks"]
        assert [len(oracle.chunk_offsets(shape, c)) for c in range(ex["chunks"])] == ex["lengths"]
    for ex in golden["spec_examples"]["effective_k"]:
        assert oracle.effective_k(ex["chunk_len"]) == ex["k_eff"]


@pytest.mark.parametrize("shape", [(64, 64), (128, 192), (130, 64), (64, 130), (100,), (1,), (3, 40, 70),
                                   (4097,), (192, 256), (8192,)])
def test_chunking_is_a_partition(shape):
    n = int(np.prod(shape))
    seen = np.zeros(n, np.int32)
    for c in range(oracle.tensor_chunks(shape)):
        off = oracle.chunk_offsets(shape, c)
        assert 1 <= len(off) <= 4096
        seen[off] += 1
    assert (seen == 1).all()


def test_block_geometry_by_hand():
    # (128, 192): 2 x 3 blocks, row-major block order, p = 64*r + c (R#7, R#8)
    shape = (128, 192)
    assert oracle.is_blocked(shape) and oracle.tensor_chunks(shape) == 6
    off = oracle.chunk_offsets(shape, 4)  # block (1, 1)
    for r, c in [(0, 0), (0, 63), (5, 7), (63, 63)]:
        assert off[64 * r + c] == (64 + r) * 192 + 64 + c
    # non-divisible 2-D is flattened (R#9): (130, 64) -> 8320 flat -> 2 full + 1 partial of 128
    assert not oracle.is_blocked((130, 64))
    assert [len(oracle.chunk_offsets((130, 64), c)) for c in range(3)] == [4096, 4096, 128]
    assert oracle.effective_k(128) == 2 and oracle.effective_k(2051) == 32 and oracle.effective_k(4095) == 63


def test_llama_1b_partial_chunks():
    lay = layouts.LAYOUTS["llama3.2-1b"]
    partial = [n for n, s in lay if not oracle.is_blocked(s) and int(np.prod(s)) % 4096]
    assert len(partial) == 33  # 16*2 norms + final norm, each 2048 long -> k_eff = 32
    assert oracle.effective_k(2048) == 32


# ------------------------------------------------------------------ Top-k
def test_spec_topk_examples(golden):
    for ex in golden["spec_examples"]["topk"]:
        sel = oracle.topk(np.array(ex["buffer"], np.float32), ex["k_eff"])
        assert sel.tolist() == ex["indices"]
        if "values" in ex:
            assert np.array(ex["buffer"], np.float32)[sel].tolist() == ex["values"]


def _brute_topk(b, k):
    """The unique k-subset S with: for i in S, j not in S: |b_i| > |b_j| or
    (|b_i| == |b_j| and i < j).  Found by enumerating every subset."""
    n = len(b)
    m = [abs(float(x)) for x in b]
    found = []
    for S in itertools.combinations(range(n), k):
        Sset = set(S)
        ok = all((m[i] > m[j]) or (m[i] == m[j] and i < j) for i in S for j in range(n) if j not in Sset)
        if ok:
            found.append(list(S))
    assert len(found) == 1
    return found[0]


def test_topk_brute_force_tiny():
    rng = np.random.default_rng(1)
    for trial in range(400):
        n = int(rng.integers(1, 11))
        k = int(rng.integers(1, n + 1))
        kind = trial % 4
        if kind == 0:
            b = rng.standard_normal(n).astype(np.float32)
        elif kind == 1:   # heavy ties incl. signed zeros
            b = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, 2.0, -2.0], np.float32), n)
        elif kind == 2:   # all equal magnitude
            b = (rng.choice([-1.0, 1.0], n) * 0.5).astype(np.float32)
        else:             # subnormals and zeros
            b = (rng.integers(-3, 4, n) * np.float32(2.0 ** -149)).astype(np.float32)
        assert oracle.topk(b, k).tolist() == _brute_topk(b, k), (b, k)


def test_topk_full_chunk_properties():
    rng = np.random.default_rng(2)
    for _ in range(20):
        b = (rng.standard_normal(4096) * 2.0 ** rng.integers(-8, 0, 4096)).astype(np.float32)
        sel = oracle.topk(b, 64)
        assert len(sel) == 64 and (np.diff(sel) > 0).all()
        uns = np.setdiff1d(np.arange(4096), sel)
        assert np.abs(b[sel]).min() >= np.abs(b[uns]).max()
    # k = n -> identity
    b = rng.standard_normal(37).astype(np.float32)
    assert oracle.topk(b, 37).tolist() == list(range(37))
    with pytest.raises(ValueError):
        oracle.topk(np.array([1.0, np.nan], np.float32), 1)


# ------------------------------------------------------------------ rounding primitives
def test_rn16_matches_numpy_float16():
    rng = np.random.default_rng(3)
    xs = np.concatenate([
        rng.standard_normal(20000).astype(np.float32) * np.float32(2.0) ** rng.integers(-30, 17, 20000).astype(np.float32),
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e9, -1e9, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.5,
                  2.0 ** -26, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], np.float32)])
    with np.errstate(over="ignore"):
        ref = xs.astype(np.float16).view(np.uint16)
    got = np.array([oracle.rn16(float(x)) for x in xs], np.uint16)
    assert (got == ref).all()
    for h in [0, 1, 0x3C00, 0x7BFF, 0x8001, 0xFC00]:
        assert oracle.f16_to_f32(h) == np.uint16(h).view(np.float16).astype(np.float32)


def test_rnbf_matches_torch_bfloat16():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(4)
    xs = (rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000)).astype(np.float32)
    xs[:4] = [0.0, -0.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8]
    ref = torch.from_numpy(xs).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([oracle.rnbf(float(x)) for x in xs], np.uint16)
    assert (got == ref).all()


def test_tree_sum_exact_and_bounded():
    rng = np.random.default_rng(5)
    for n in [1, 2, 31, 32, 33, 63, 64]:
        ints = rng.integers(0, 1000, n).astype(np.float32)          # exact sums
        assert oracle.tree_sum(ints, 64) == np.float32(ints.sum(dtype=np.float64))
        x = np.abs(rng.standard_normal(n)).astype(np.float32)
        exact = math.fsum(float(v) for v in x)
        # recursive-summation bound: |err| <= (depth) * u * sum|x|, depth <= 2 + 5
        assert abs(float(oracle.tree_sum(x, 64)) - exact) <= 7 * 2.0 ** -24 * exact + 1e-45
    # k up to 256: W = 8 slots per lane
    x = np.ones(256, np.float32)
    assert oracle.tree_sum(x, 256) == 256.0


# ------------------------------------------------------------------ quantiser Q (R#1; parity unpinned by the paper)
def test_spec_quantizer_examples(golden):
    for ex in golden["spec_examples"]["quantize"]:
        vals = ex["values"]
        g = oracle.geom(block=2, k=4)   # k = C: every position of the (partial) chunk is sent
        n = len(vals)
        st, rec, en = oracle.compress_chunk(np.array(vals, np.float32), np.zeros(n, np.float32),
                                            np.zeros(n, np.float32), 0.95, g)
        assert st == 0
        pos, dq = oracle.decode_chunk(rec, n, g)
        assert pos.tolist() == list(range(n))
        assert dq.tolist() == [float(np.float16(x)) for x in ex["decode"]]
        lo = oracle.f16_to_f32(rec[-1] & 0xFFFF)
        hi = oracle.f16_to_f32(rec[-1] >> 16)
        if "scale_lo" in ex:
            assert lo == ex["scale_lo"]
        if "scale_hi" in ex:
            assert hi == ex["scale_hi"]


def test_quantizer_invariants():
    rng = np.random.default_rng(6)
    for trial in range(200):
        b = (rng.standard_normal(4096) * 2.0 ** rng.integers(-12, -4)).astype(np.float32)
        z = np.zeros(4096, np.float32)
        st, rec, en = oracle.compress_chunk(b, z, z, 0.95, G)
        assert st == 0
        pos, dq = oracle.decode_chunk(rec, 4096, G)
        v = b[pos]
        S_lo = oracle.f16_to_f32(rec[-1] & 0xFFFF)
        S_hi = oracle.f16_to_f32(rec[-1] >> 16)
        assert S_lo <= S_hi
        nz = v != 0
        assert (np.sign(dq[nz]) == np.sign(v[nz])).all()                # sign preserved
        assert set(np.abs(dq).tolist()) <= {float(S_lo), float(S_hi)}  # 2 magnitudes = 2 bits with sign
        tau = np.abs(v.astype(np.float64)).mean()
        mag = np.abs(v).astype(np.float64)
        # buckets split at the mean (within fp32 summation error of tau)
        hi_b = np.abs(dq) == S_hi
        if S_lo != S_hi:
            assert (mag[hi_b] >= tau * (1 - 1e-5)).all() and (mag[~hi_b] <= tau * (1 + 1e-5)).all()
            # scales are bucket means, rounded to fp16
            assert abs(S_hi - mag[hi_b].mean()) <= 2.0 ** -10 * S_hi + 1e-30
            if (~hi_b).any():
                assert abs(S_lo - mag[~hi_b].mean()) <= 2.0 ** -10 * max(S_lo, 1e-30) + 2.0 ** -24
        # |dq - v| <= max(|v - lo|, |v - hi|) + fp16 rounding
        err = np.abs(dq.astype(np.float64) - v)
        bound = np.maximum(np.abs(mag - S_lo), np.abs(mag - S_hi)) + 2.0 ** -10 * S_hi
        assert (err <= bound).all()


def test_fp16_overflow_and_nonfinite_are_invalid_data():
    z = np.zeros(4096, np.float32)
    big = np.zeros(4096, np.float32); big[:64] = 1e6
    st, _, _ = oracle.compress_chunk(big, z, z, 0.95, G)
    assert st == oracle.INVALID_DATA
    for bad in [np.inf, -np.inf, np.nan]:
        x = np.ones(4096, np.float32); x[77] = bad
        assert oracle.compress_chunk(x, z, z, 0.95, G)[0] == oracle.INVALID_DATA
        assert oracle.compress_chunk(z, x, z, 0.95, G)[0] == oracle.INVALID_DATA
        assert oracle.compress_chunk(z, z, x, 0.95, G)[0] == oracle.INVALID_DATA
    # overflow in the sum itself: a - l = inf
    a = np.zeros(4096, np.float32); a[0] = 3e38
    l = np.zeros(4096, np.float32); l[0] = -3e38
    assert oracle.compress_chunk(a, l, z, 0.95, G)[0] == oracle.INVALID_DATA


# ------------------------------------------------------------------ Eq. 1 identity
def test_ef_identity_exact_arithmetic():
    """e_new + hatDelta == beta*e + (theta - theta_local) (Eq. 1), each
    side evaluated exactly with Fractions; the only slack is one rounding of
    the difference, one of the fma and one of the residual subtraction."""
    rng = np.random.default_rng(7)
    beta = np.float32(0.95)
    for trial in range(6):
        n = 4096 if trial < 4 else 2051
        a = (rng.standard_normal(n) * 0.02).astype(np.float32)
        d_t = (rng.uniform(-1, 1, n) * 2.0 ** -9 * 2.0 ** -rng.integers(0, 8, n)).astype(np.float32)
        l = (a - d_t).astype(np.float32)
        e = (rng.uniform(-1, 1, n) * 2.0 ** -7 * 2.0 ** -rng.integers(0, 8, n)).astype(np.float32)
        st, rec, en = oracle.compress_chunk(a, l, e, float(beta), G)
        assert st == 0
        pos, dq = oracle.decode_chunk(rec, n, G)
        assert len(pos) == oracle.effective_k(n)
        hat = np.zeros(n, np.float64); hat[pos] = dq
        for p in range(0, n, 7):
            d = float(a[p]) - float(l[p])
            exact_b = Fraction(float(beta)) * Fraction(float(e[p])) + Fraction(d)
            d32 = float(np.float32(float(a[p]) - float(l[p])))
            slack = 0.5 * ulp32(d32) + 0.5 * ulp32(float(en[p]) + hat[p]) + 0.5 * ulp32(float(en[p]))
            lhs = Fraction(float(en[p])) + Fraction(float(hat[p]))
            assert abs(float(lhs - exact_b)) <= slack + 1e-45, (p, float(lhs), float(exact_b))
        unsel = np.setdiff1d(np.arange(n), pos)
        # unselected positions keep b = fma(beta, e, a - l) exactly
        d32 = (a - l).astype(np.float32)
        b_ref = np.array([np.float32(Fraction(float(beta)) * Fraction(float(x)) + Fraction(float(y)))
                          for x, y in zip(e[unsel[:200]], d32[unsel[:200]])], np.float32)
        assert (en[unsel[:200]] == b_ref).all()


def test_selection_uses_ef_accumulated_buffer():
    # the selection ranks beta*e + Delta, not Delta alone: e flips which positions win
    n = 4096
    a = np.zeros(n, np.float32); l = np.zeros(n, np.float32); e = np.zeros(n, np.float32)
    a[:64] = 1.0                      # Delta large on 0..63
    e[100:164] = 2.0                  # beta*e = 1.9 on 100..163 beats it
    st, rec, en = oracle.compress_chunk(a, l, e, 0.95, G)
    pos, dq = oracle.decode_chunk(rec, n, G)
    assert pos.tolist() == list(range(100, 164))
    assert np.allclose(dq, np.float16(np.float32(0.95) * np.float32(2.0)))
    assert (en[:64] == 1.0).all()     # untransmitted Delta stays in EF


def test_lossless_single_peer_identity():
    """k = C and values Q represents exactly -> e_new = 0, hatDelta = b, and
    with one peer and alpha = 1 the outer step lands on theta_local."""
    g = oracle.geom(block=8, k=64)          # C = 64 = k: every position transmitted
    rng = np.random.default_rng(8)
    theta = (rng.integers(-2 ** 14, 2 ** 14, 64) * 2.0 ** -20).astype(np.float32)  # theta -+ c exact
    c = np.float32(2.0 ** -10)
    sign = rng.choice(np.array([-1.0, 1.0], np.float32), 64)
    theta_local = (theta - c * sign).astype(np.float32)
    assert ((theta - theta_local) == c * sign).all()        # exact difference
    st, rec, en = oracle.compress_chunk(theta, theta_local, np.zeros(64, np.float32), 0.95, g)
    assert st == 0 and (en == 0).all()
    delta = oracle.aggregate_chunk([rec], 64, g=g)
    assert (delta == c * sign).all()
    new = oracle.outer_update(theta, delta, 1.0)
    assert (new.view(np.uint32) == theta_local.view(np.uint32)).all()


# ------------------------------------------------------------------ Eq. 2 aggregation
def _records(rng, R, n=4096, g=G):
    recs = []
    for r in range(R):
        a = (rng.standard_normal(n) * 2.0 ** -int(rng.integers(6, 12))).astype(np.float32)
        z = np.zeros(n, np.float32)
        st, rec, _ = oracle.compress_chunk(a, z, z, 0.95, g)
        assert st == 0
        recs.append(rec)
    return recs


def test_spec_aggregate_example(golden):
    ex = golden["spec_examples"]["aggregate"][0]
    g = oracle.geom(block=2, k=2)  # chunk of n=2 -> k_eff = 1
    recs = []
    for vec in ex["decoded"]:
        v = np.array(vec, np.float32)
        st, rec, _ = oracle.compress_chunk(v, np.zeros(2, np.float32), np.zeros(2, np.float32), 0.95, g)
        assert st == 0
        pos, dq = oracle.decode_chunk(rec, 2, g)
        dense = np.zeros(2, np.float32); dense[pos] = dq
        assert dense.tolist() == vec
        recs.append(rec)
    assert oracle.aggregate_chunk(recs, 2, g=g).tolist() == ex["mean"]


def test_aggregate_equals_exact_mean():
    rng = np.random.default_rng(9)
    for R in [1, 2, 3, 8, 20, 64]:
        recs = _records(rng, R)
        delta = oracle.aggregate_chunk(recs, 4096)
        exact = [Fraction(0)] * 4096
        for rec in recs:
            pos, dq = oracle.decode_chunk(rec, 4096)
            for p, v in zip(pos, dq):
                exact[p] += Fraction(float(v))
        for p in range(4096):
            m = exact[p] / R
            if R & (R - 1) == 0:        # 1/R exact -> correctly rounded mean, bitwise
                assert delta[p] == np.float32(float(m))
            else:                        # one fp64 product rounding then fp32
                assert abs(float(delta[p]) - float(m)) <= 0.5 * ulp32(float(delta[p])) + abs(float(m)) * 2.0 ** -52
        if R == 1:
            pos, dq = oracle.decode_chunk(recs[0], 4096)
            dense = np.zeros(4096, np.float32); dense[pos] = dq
            assert (delta.view(np.uint32) == dense.view(np.uint32)).all()


def test_aggregate_permutation_invariant_bitwise():
    rng = np.random.default_rng(10)
    R = 20
    recs = _records(rng, R)
    ids = rng.integers(0, 256, (R, 16)).astype(np.uint8)
    w = rng.uniform(0.1, 2.0, R).astype(np.float32)
    base = oracle.aggregate_chunk(recs, 4096)
    base_w = oracle.aggregate_chunk(recs, 4096, peer_ids=ids, weights=w)
    for _ in range(5):
        perm = rng.permutation(R)
        got = oracle.aggregate_chunk([recs[i] for i in perm], 4096)
        assert (got.view(np.uint32) == base.view(np.uint32)).all()
        got_w = oracle.aggregate_chunk([recs[i] for i in perm], 4096, peer_ids=ids[perm], weights=w[perm])
        assert (got_w.view(np.uint32) == base_w.view(np.uint32)).all()


# ------------------------------------------------------------------ Eq. 2 outer step
def test_outer_update_spec_examples(golden):
    rng = np.random.default_rng(11)
    theta = (rng.standard_normal(1000) * 0.02).astype(np.float32)
    delta = rng.standard_normal(1000).astype(np.float32)
    assert (oracle.outer_update(theta, delta, 0.0).view(np.uint32) == theta.view(np.uint32)).all()
    ones = np.ones(1000, np.float32)
    new = oracle.outer_update(theta, ones, 0.65)
    exact = theta.astype(np.float64) - np.float64(np.float32(0.65))
    assert (new == exact.astype(np.float32)).all()   # fma: one rounding of theta - alpha*1
    # general: theta - alpha*delta with a single rounding
    new = oracle.outer_update(theta, delta, 1.0)
    assert (new == (theta.astype(np.float64) - delta.astype(np.float64)).astype(np.float32)).all()


def test_outer_update_bf16():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    th32 = (rng.standard_normal(5000) * 0.02).astype(np.float32)
    th = torch.from_numpy(th32).to(torch.bfloat16)
    bits = th.view(torch.int16).numpy().view(np.uint16)
    delta = (rng.standard_normal(5000) * 1e-3).astype(np.float32)
    new = oracle.outer_update(bits, delta, 0.65)
    newf = torch.from_numpy(new.view(np.int16)).view(torch.bfloat16).float().numpy()
    exact = th.float().numpy().astype(np.float64) - np.float64(np.float32(0.65)) * delta
    # one bf16 rounding (plus fp32 fma rounding, far below)
    assert (np.abs(newf - exact) <= 0.5 * np.abs(exact) * 2.0 ** -7 + 1e-30).all()


# ------------------------------------------------------------------ tensor drivers / determinism
def test_tensor_driver_matches_chunk_calls_and_is_deterministic():
    rng = np.random.default_rng(13)
    shape = (130, 64)  # flattened, partial last chunk
    n = 130 * 64
    a = (rng.standard_normal(n) * 0.02).astype(np.float32)
    l = (a - rng.standard_normal(n).astype(np.float32) * 1e-3).astype(np.float32)
    e = (rng.standard_normal(n) * 1e-4).astype(np.float32)
    recs, en = oracle.compress_tensor(shape, a, l, e)
    recs2, en2 = oracle.compress_tensor(shape, a, l, e)
    assert (recs == recs2).all() and (en.view(np.uint32) == en2.view(np.uint32)).all()
    for c in range(oracle.tensor_chunks(shape)):
        off = oracle.chunk_offsets(shape, c)
        st, rec, e_c = oracle.compress_chunk(a[off], l[off], e[off], 0.95)
        assert st == 0 and (rec == recs[c]).all() and (en[off] == e_c).all()
    delta = oracle.aggregate_tensor(shape, [recs])
    th = oracle.aggregate_update_tensor(shape, a, [recs], 1.0)
    assert (th == oracle.outer_update(a, delta, 1.0)).all()


def test_bf16_inputs_are_widened_exactly():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(14)
    a32 = (rng.standard_normal(4096) * 0.02).astype(np.float32)
    l32 = (a32 - rng.standard_normal(4096).astype(np.float32) * 1e-3).astype(np.float32)
    a = torch.from_numpy(a32).to(torch.bfloat16)
    l = torch.from_numpy(l32).to(torch.bfloat16)
    ab = a.view(torch.int16).numpy().view(np.uint16)
    lb = l.view(torch.int16).numpy().view(np.uint16)
    e = np.zeros(4096, np.float32)
    st1, r1, e1 = oracle.compress_chunk(ab, lb, e, 0.95)
    st2, r2, e2 = oracle.compress_chunk(a.float().numpy(), l.float().numpy(), e, 0.95)
    assert st1 == st2 == 0 and (r1 == r2).all() and (e1.view(np.uint32) == e2.view(np.uint32)).all()


# ---------------------------------------------------------------- median-norm (R#20)
def test_median_normalize_spec_example_norms_1_2_4():
    """norms [1, 2, 4] -> every output has norm 2 (rescale factors 2, 1, 0.5)."""
    rng = np.random.default_rng(5)
    base = [rng.normal(size=50) for _ in range(3)]
    deltas = [b / np.linalg.norm(b) * s for b, s in zip(base, [1.0, 2.0, 4.0])]
    out = oracle.median_normalize(deltas)
    for o in out:
        assert abs(np.linalg.norm(o) - 2.0) < 1e-12
    w = oracle.median_norm_weights([1.0, 2.0, 4.0])
    assert list(w) == [2.0, 1.0, 0.5]


def test_median_norm_weights_properties():
    # all equal -> unchanged; zero norms pass through; lower median for even counts
    assert list(oracle.median_norm_weights([3.0, 3.0, 3.0])) == [1.0, 1.0, 1.0]
    assert list(oracle.median_norm_weights([0.0, 2.0, 2.0])) == [1.0, 1.0, 1.0]
    assert list(oracle.median_norm_weights([1.0, 2.0, 4.0, 8.0])) == [2.0, 1.0, 0.5, 0.25]
    # one adversarial peer: its contribution is bounded by the median
    n = [1.0, 1.1, 0.9, 1e6]
    w = oracle.median_norm_weights(n)
    assert abs(float(w[3]) * 1e6 - 1.0) < 1e-6
    # permutation invariance and scale equivariance: weights unchanged when
    # every norm is scaled by a power of two
    rng = np.random.default_rng(9)
    n = list(rng.uniform(0.1, 5.0, 9))
    w = oracle.median_norm_weights(n)
    perm = rng.permutation(9)
    assert np.array_equal(oracle.median_norm_weights([n[i] for i in perm]), w[perm])
    assert np.array_equal(oracle.median_norm_weights([x * 8.0 for x in n]), w)


def _f16_fraction(h):
    from fractions import Fraction
    e, m = (h >> 10) & 0x1F, h & 0x3FF
    return Fraction(m, 1 << 24) if e == 0 else Fraction(1024 + m, 1 << 24) * (1 << (e - 1))


def test_payload_norm_is_exact_sum_of_squares():
    """payload_norm (decode + fsum) equals sqrt(RN(exact rational sum)) built
    directly from the fp16 bit patterns and codes, on random payloads whose
    scales span the whole fp16 range (subnormal to 2^15)."""
    import math
    from helpers import pack_record
    g = oracle.geom()
    rng = np.random.default_rng(11)
    for trial in range(20):
        chunks, exact = [], 0
        for _ in range(int(rng.integers(1, 6))):
            n = int(rng.choice([4096, 1000]))
            ke = oracle.effective_k(n, g)
            pos = np.sort(rng.choice(n, ke, replace=False))
            codes = rng.integers(0, 4, ke)
            sc = [(int(rng.integers(0, 31)) << 10) | int(rng.integers(0, 1024)) for _ in range(2)]
            chunks.append((pack_record(pos, codes, sc[0], sc[1], 64, 12), n))
            exact += sum(_f16_fraction(sc[(int(c) >> 1) & 1]) ** 2 for c in codes)
        assert oracle.payload_norm(chunks, g) == math.sqrt(float(exact))


def test_payload_norm_closed_form():
    # one chunk, every slot in the hi bucket with scale S: ||.||^2 = k * S^2
    from helpers import pack_record
    g = oracle.geom()
    S = 0x3C00  # 1.0 in fp16
    rec = pack_record(np.arange(64) * 3, np.full(64, 2), 0, S, 64, 12)
    assert oracle.payload_norm([(rec, 4096)], g) == 8.0
