"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Bars (BASELINE.json north_star): indices / codes / records
bit-exact; EF, scales, Delta and theta within 1e-6 relative (fp32) / 1e-2
(bf16) — the kernels are written to the oracle's operation order, so the
tests demand bitwise equality, which is stricter."""
import numpy as np
import pytest

import oracle
import slcgen
from helpers import (bits, craft_records, host_segment, make_device_inputs, oracle_compress_shard,
                     oracle_update_shard, seg_view)
from slcgen import layouts

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")


def _compress_gpu(plan, layout, seed, peer, dtype, special_period, warm, theta=None):
    theta, tl, ef = make_device_inputs(plan, layout, seed, peer, dtype, special_period, warm, theta=theta)
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    plan.compress(theta, tl, ef, rec)
    return theta, tl, ef, rec


@pytest.mark.parametrize("name", ["ragged", "1m-2d", "1m-1d"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("special", [0, 4])
def test_compress_parity(name, dtype, special):
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype=dtype)
    warm = special == 0
    theta, tl, ef, rec = _compress_gpu(plan, layout, 3, 1, dtype, special, warm)
    assert plan.get_status() == slc.OK
    ref_rec, ref_ef, _ = oracle_compress_shard(plan, layout, 3, 1, dtype, special, warm)
    got = rec.cpu().numpy().view(np.uint32)
    mism = np.nonzero(got != ref_rec)[0]
    assert mism.size == 0, f"{mism.size} record words differ, first at word {mism[:5]}"
    for s, e in zip(plan.segments, ref_ef):
        g = seg_view(ef, s).cpu().numpy()
        assert np.array_equal(bits(g), bits(e)), f"EF differs in segment {s.tensor}"


@pytest.mark.parametrize("R", [1, 3, 8, 20])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_aggregate_update_parity(R, dtype, agg_kernel):
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout, dtype=dtype)
    recs, ref_recs = [], []
    theta = None
    for r in range(R):
        theta, tl, ef, rec = _compress_gpu(plan, layout, 5, r, dtype, 8, True, theta=theta)
        recs.append(rec)
        rr, _, thetas = oracle_compress_shard(plan, layout, 5, r, dtype, 8, True)
        assert np.array_equal(rec.cpu().numpy().view(np.uint32), rr)
        ref_recs.append(rr)
    alpha = 0.65
    # unfused: decode_aggregate -> Delta, then update from Delta
    agg = torch.zeros(plan.shard_elems, dtype=torch.float32, device=DEV)
    plan.decode_aggregate(recs, agg)
    ref_delta = oracle_update_shard(plan, thetas, ref_recs, alpha, only_delta=True)
    for s, d in zip(plan.segments, ref_delta):
        assert np.array_equal(bits(seg_view(agg, s).cpu().numpy()), bits(d))
    th_unfused = theta.clone()
    plan.outer_update(th_unfused, alpha, agg=agg)
    # fused
    th_fused = theta.clone()
    plan.outer_update(th_fused, alpha, records=recs)
    assert plan.get_status() == slc.OK
    ref_theta = oracle_update_shard(plan, thetas, ref_recs, alpha)
    for s, t in zip(plan.segments, ref_theta):
        tb = bits(t)
        fu = seg_view(th_fused, s).cpu()
        un = seg_view(th_unfused, s).cpu()
        if dtype == "bf16":
            fu, un = fu.view(torch.int16), un.view(torch.int16)
        assert np.array_equal(bits(fu.numpy()), tb)
        assert np.array_equal(bits(un.numpy()), tb)


@pytest.mark.parametrize("R", [1, 2, 20, 64])
@pytest.mark.parametrize("exps", [(4, 9), (0, 30), (1, 16)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_aggregate_crafted_records(R, exps, dtype, agg_kernel):
    """Decode / aggregate / update on random well-formed payloads whose fp16
    scales span a chosen exponent range: (4, 9) keeps every chunk on the
    single-int32 accumulator, (0, 30) (subnormal to 2^15) forces the wide
    one, (1, 16) mixes both per chunk and R."""
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout, dtype=dtype)
    rng = np.random.default_rng(1000 * R + exps[1])
    theta, _, _ = make_device_inputs(plan, layout, 21, 0, dtype)
    thetas = [host_segment(layout, s, slcgen.WHAT_THETA, 21, 0, dtype) for s in plan.segments]
    ref_recs = [craft_records(plan, rng, *exps) for _ in range(R)]
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    agg = torch.zeros(plan.shard_elems, dtype=torch.float32, device=DEV)
    plan.decode_aggregate(recs, agg)
    for s, d in zip(plan.segments, oracle_update_shard(plan, thetas, ref_recs, 1.0, only_delta=True)):
        assert np.array_equal(bits(seg_view(agg, s).cpu().numpy()), bits(d))
    alpha = 0.65
    plan.outer_update(theta, alpha, records=recs)
    assert plan.get_status() == slc.OK
    for s, t in zip(plan.segments, oracle_update_shard(plan, thetas, ref_recs, alpha)):
        got = seg_view(theta, s).cpu()
        if dtype == "bf16":
            got = got.view(torch.int16)
        assert np.array_equal(bits(got.numpy()), bits(t))


@pytest.mark.parametrize("R", [2, 20, 40])
@pytest.mark.parametrize("exps,wspan", [((4, 9), 1.0), ((4, 9), 64.0), ((0, 30), 1.0), ((2, 14), 1e4)])
def test_weighted_aggregate_crafted(R, exps, wspan, agg_kernel):
    """Weighted Eq. 2 (median-norm weights enter as w_r) on crafted
    payloads: narrow scale / weight ranges take the exact fixed-point path
    (bitwise the oracle's fp64 canonical-order sum, which is exact there),
    wide ones the sequential fp64 path."""
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout)
    rng = np.random.default_rng(500 + R + exps[1] + int(wspan))
    ref_recs = [craft_records(plan, rng, *exps) for _ in range(R)]
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    ids = [bytes(rng.integers(0, 256, 16, dtype=np.uint8)) for _ in range(R)]
    hdrs = [slc.make_header(plan, ids[r], base_round=2) for r in range(R)]
    w = np.exp(rng.uniform(-np.log(wspan), np.log(wspan), R)).astype(np.float32) if wspan > 1 else \
        rng.uniform(0.5, 1.5, R).astype(np.float32)
    got = torch.zeros(plan.shard_elems, device=DEV)
    plan.decode_aggregate(recs, got, hdrs=hdrs, weights=w)
    wd = torch.from_numpy(w).to(DEV)
    got2 = torch.zeros(plan.shard_elems, device=DEV)
    plan.decode_aggregate(recs, got2, hdrs=hdrs, weights_dev=wd)
    assert plan.get_status() == slc.OK
    thetas = [np.zeros(s.n_elems, np.float32) for s in plan.segments]
    ref = oracle_update_shard(plan, thetas, ref_recs, 1.0, peer_ids=np.frombuffer(b"".join(ids), np.uint8),
                              weights=w, only_delta=True)
    for s, d in zip(plan.segments, ref):
        assert np.array_equal(bits(seg_view(got, s).cpu().numpy()), bits(d))
        assert np.array_equal(bits(seg_view(got2, s).cpu().numpy()), bits(d))


@pytest.mark.parametrize("R", [3, 20])
@pytest.mark.parametrize("offset", [4, 8, 12])
def test_aggregate_misaligned_record_buffers(R, offset, agg_kernel):
    """Record buffers that are only 4-B aligned (the C ABI's requirement) take
    the word-by-word staging path; results are unchanged."""
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout)
    rng = np.random.default_rng(77 + R + offset)
    theta, _, _ = make_device_inputs(plan, layout, 23, 0)
    thetas = [host_segment(layout, s, slcgen.WHAT_THETA, 23, 0) for s in plan.segments]
    ref_recs = [craft_records(plan, rng, 2, 12) for _ in range(R)]
    recs = []
    for r in ref_recs:
        buf = torch.zeros(r.nbytes + 16, dtype=torch.uint8, device=DEV)
        v = buf[offset:offset + r.nbytes]
        v.copy_(torch.from_numpy(r.view(np.uint8).copy()))
        recs.append(v)
    plan.outer_update(theta, 1.0, records=recs)
    assert plan.get_status() == slc.OK
    for s, t in zip(plan.segments, oracle_update_shard(plan, thetas, ref_recs, 1.0)):
        assert np.array_equal(bits(seg_view(theta, s).cpu().numpy()), bits(t))


def test_permutation_invariance_and_weights(agg_kernel):
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout)
    R = 12
    recs, ref_recs, theta = [], [], None
    for r in range(R):
        theta, tl, ef, rec = _compress_gpu(plan, layout, 9, r, "f32", 0, True, theta=theta)
        recs.append(rec)
        rr, _, thetas = oracle_compress_shard(plan, layout, 9, r, "f32", 0, True)
        ref_recs.append(rr)
    rng = np.random.default_rng(0)
    base = torch.zeros(plan.shard_elems, device=DEV)
    plan.decode_aggregate(recs, base)
    for _ in range(3):
        perm = rng.permutation(R)
        got = torch.zeros(plan.shard_elems, device=DEV)
        plan.decode_aggregate([recs[i] for i in perm], got)
        assert torch.equal(got.view(torch.int32), base.view(torch.int32))
    # weighted (median-norm style weights), canonical peer-id order via headers
    ids = [bytes(rng.integers(0, 256, 16, dtype=np.uint8)) for _ in range(R)]
    w = rng.uniform(0.25, 2.0, R).astype(np.float32)
    hdrs = [slc.make_header(plan, ids[r], base_round=7) for r in range(R)]
    ref = oracle_update_shard(plan, thetas, ref_recs, 1.0, peer_ids=np.frombuffer(b"".join(ids), np.uint8),
                              weights=w, only_delta=True)
    for _ in range(3):
        perm = rng.permutation(R)
        got = torch.zeros(plan.shard_elems, device=DEV)
        plan.decode_aggregate([recs[i] for i in perm], got, hdrs=[hdrs[i] for i in perm], weights=w[perm])
        for s, d in zip(plan.segments, ref):
            assert np.array_equal(bits(seg_view(got, s).cpu().numpy()), bits(d))


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_sharding_invariance(nranks):
    """Records of every shard concatenated in rank order == the 1-shard records;
    EF identical (compression is independent per shard)."""
    layout = layouts.LAYOUTS["ragged"] + [("w_big", (512, 256))]
    full = slc.Plan(layout)
    _, _, ef1, rec1 = _compress_gpu(full, layout, 11, 2, "f32", 4, True)
    parts, first = [], 0
    for g in range(nranks):
        p = slc.Plan(layout, rank=g, nranks=nranks)
        assert p.info.first_chunk == first
        first += p.n_chunks
        if p.n_chunks == 0:
            continue
        _, _, ef, rec = _compress_gpu(p, layout, 11, 2, "f32", 4, True)
        parts.append(rec.cpu())
        for s in p.segments:
            ref = [t for t in full.segments if t.tensor == s.tensor][0]
            lo = ref.shard_offset + s.tensor_begin - ref.tensor_begin
            assert torch.equal(seg_view(ef, s).cpu().view(torch.int32),
                               ef1[lo:lo + s.n_elems].cpu().view(torch.int32))
    assert first == full.n_chunks
    assert torch.equal(torch.cat(parts), rec1.cpu())


@pytest.mark.parametrize("block,k", [(32, 4), (32, 16), (32, 64), (64, 16), (64, 32), (64, 128), (64, 256),
                                     (128, 64), (128, 256)])
def test_geometry_sweep_parity(block, k, agg_kernel):
    g = slc.geometry(block=block, k=k)
    og = oracle.geom(block=block, k=k)
    B = block
    layout = [("w", (2 * B, 3 * B)), ("v", (B * B * 2 + 77,)), ("r", (B + 3, B))]
    plan = slc.Plan(layout, geom=g)
    recs, ref_recs, theta = [], [], None
    for r in range(3):
        theta, tl, ef, rec = _compress_gpu(plan, layout, 13, r, "f32", 2, True, theta=theta)
        rr, ref_ef, thetas = oracle_compress_shard(plan, layout, 13, r, "f32", 2, True, g=og)
        assert np.array_equal(rec.cpu().numpy().view(np.uint32), rr)
        for s, e in zip(plan.segments, ref_ef):
            assert np.array_equal(bits(seg_view(ef, s).cpu().numpy()), bits(e))
        recs.append(rec)
        ref_recs.append(rr)
    plan.outer_update(theta, 1.0, records=recs)
    ref = oracle_update_shard(plan, thetas, ref_recs, 1.0, g=og)
    for s, t in zip(plan.segments, ref):
        assert np.array_equal(bits(seg_view(theta, s).cpu().numpy()), bits(t))


def test_error_injection():
    layout = [("w", (64, 128)), ("b", (4096,))]
    plan = slc.Plan(layout)
    theta, tl, ef = make_device_inputs(plan, layout, 1, 0)
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    plan.compress(theta, tl, ef, rec)
    assert plan.get_status() == slc.OK
    for buf, val in [(theta, float("nan")), (tl, float("inf")), (ef, float("-inf"))]:
        t2, l2, e2 = theta.clone(), tl.clone(), ef.clone()
        {id(theta): t2, id(tl): l2, id(ef): e2}[id(buf)][100] = val
        plan.compress(t2, l2, e2, rec)
        assert plan.get_status() == slc.INVALID_DATA
        assert plan.get_status() == slc.OK  # cleared
    # fp16 scale overflow
    t2 = theta.clone()
    t2[:64] = 1e6
    plan.compress(t2, tl, ef.clone(), rec)
    assert plan.get_status() == slc.INVALID_DATA
    # stale / mismatched headers
    good = slc.make_header(plan, b"peer-a", base_round=3)
    stale = slc.make_header(plan, b"peer-b", base_round=4)
    agg = torch.zeros(plan.shard_elems, device=DEV)
    with pytest.raises(slc.SlcError) as ei:
        plan.decode_aggregate([rec, rec], agg, hdrs=[good, stale])
    assert ei.value.status == slc.STALE
    other = slc.Plan([("w", (64, 64)), ("b", (8192,))])  # same chunk count, other layout digest
    with pytest.raises(slc.SlcError) as ei:
        plan.decode_aggregate([rec, rec], agg, hdrs=[good, slc.make_header(other, b"peer-b", 3)])
    assert ei.value.status == slc.STALE
    wrong_range = slc.make_header(plan, b"peer-b", base_round=3)
    wrong_range.first_chunk = 1
    with pytest.raises(slc.SlcError) as ei:
        plan.decode_aggregate([rec, rec], agg, hdrs=[good, wrong_range])
    assert ei.value.status == slc.INVALID_ARGUMENT
    dup = slc.make_header(plan, b"peer-a", base_round=3)
    with pytest.raises(slc.SlcError) as ei:
        plan.decode_aggregate([rec, rec], agg, hdrs=[good, dup])
    assert ei.value.status == slc.INVALID_ARGUMENT
    # misaligned dense buffer
    big = torch.zeros(plan.shard_elems + 4, device=DEV)
    with pytest.raises(slc.SlcError) as ei:
        plan.compress(big[1:plan.shard_elems + 1], tl, ef, rec)
    assert ei.value.status == slc.INVALID_ARGUMENT


def test_generator_cuda_twin_bitwise():
    rng = np.random.default_rng(1)
    for what in [slcgen.WHAT_THETA, slcgen.WHAT_THETA_LOCAL, slcgen.WHAT_EF]:
        for _ in range(3):
            G0 = int(rng.integers(0, 2 ** 40))
            n = 100003
            ref = slcgen.generate(what, 42, 7, G0, n, special_period=3, warm_ef=True)
            buf = torch.empty(n, dtype=torch.float32, device=DEV)
            slcgen.fill_cuda(buf, what, 42, 7, G0, special_period=3, warm_ef=True)
            assert np.array_equal(bits(buf.cpu().numpy()), bits(ref))
    ref = slcgen.generate(slcgen.WHAT_THETA, 1, 0, 999, 5000, dtype="bf16")
    buf = torch.empty(5000, dtype=torch.bfloat16, device=DEV)
    slcgen.fill_cuda(buf, slcgen.WHAT_THETA, 1, 0, 999)
    assert np.array_equal(buf.view(torch.int16).cpu().numpy().view(np.uint16), ref)


# ---------------------------------------------------------------- median-norm (R#20)
def _chunks_of(plan, rec_words):
    from helpers import shard_chunk_lengths
    RW = plan.record_bytes // 4
    lens = shard_chunk_lengths(plan)
    return [(rec_words[i * RW:(i + 1) * RW], n) for i, n in enumerate(lens)]


def _limbs_value(limbs_row):
    return sum(int(x) << (32 * i) for i, x in enumerate(np.asarray(limbs_row, np.int64).view(np.uint64)))


def _exact_sq_units(plan, rec_words):
    """sum of dq^2 over the payload, as an integer in units of 2^-48 (Fractions, oracle decode)."""
    from fractions import Fraction
    tot = Fraction(0)
    for rec, n in _chunks_of(plan, rec_words):
        _, dq = oracle.decode_chunk(rec, n)
        tot += sum(Fraction(float(x)) ** 2 for x in dq)
    v = tot * (1 << 48)
    assert v.denominator == 1
    return int(v)


@pytest.mark.parametrize("exps", [(2, 12), (0, 30)])
def test_median_norm_weights_parity(exps):
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout)
    rng = np.random.default_rng(300 + exps[1])
    R = 7
    ref_recs = [craft_records(plan, rng, *exps) for _ in range(R)]
    ref_recs[3] = ref_recs[0].copy()
    ref_recs[3].reshape(-1, plan.record_bytes // 4)[:, -1] = 0  # a zero-norm peer passes through
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    limbs = torch.zeros((R, 4), dtype=torch.int64, device=DEV)
    plan.payload_sqnorm(recs, limbs)
    w = torch.zeros(R, dtype=torch.float32, device=DEV)
    nrm = torch.zeros(R, dtype=torch.float64, device=DEV)
    plan.median_norm_weights(limbs, w, nrm)
    assert plan.get_status() == slc.OK
    L = limbs.cpu().numpy()
    for r in range(R):
        assert _limbs_value(L[r]) == _exact_sq_units(plan, ref_recs[r])
    ref_norms = [oracle.payload_norm(_chunks_of(plan, rr)) for rr in ref_recs]
    assert np.array_equal(nrm.cpu().numpy(), np.array(ref_norms))
    ref_w = oracle.median_norm_weights(ref_norms)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), ref_w.view(np.uint32))
    assert float(w[3]) == 1.0
    # the weighted fused update with the device weights == the oracle's weighted Eq. 2
    ids = [bytes(rng.integers(0, 256, 16, dtype=np.uint8)) for _ in range(R)]
    hdrs = [slc.make_header(plan, ids[r], base_round=1) for r in range(R)]
    theta, _, _ = make_device_inputs(plan, layout, 31, 0)
    thetas = [host_segment(layout, s, slcgen.WHAT_THETA, 31, 0) for s in plan.segments]
    plan.outer_update(theta, 1.0, records=recs, hdrs=hdrs, weights_dev=w)
    assert plan.get_status() == slc.OK
    ref = oracle_update_shard(plan, thetas, ref_recs, 1.0, peer_ids=np.frombuffer(b"".join(ids), np.uint8),
                              weights=ref_w)
    for s, t in zip(plan.segments, ref):
        assert np.array_equal(bits(seg_view(theta, s).cpu().numpy()), bits(t))


@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_payload_sqnorm_sharding_invariance(nranks):
    """Limbs of the shards add up exactly to the single-shard limbs' value."""
    layout = layouts.LAYOUTS["ragged"]
    full = slc.Plan(layout)
    rng = np.random.default_rng(40 + nranks)
    R = 3
    ref_recs = [craft_records(full, rng, 0, 30) for _ in range(R)]
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    limbs = torch.zeros((R, 4), dtype=torch.int64, device=DEV)
    full.payload_sqnorm(recs, limbs)
    want = [_limbs_value(x) for x in limbs.cpu().numpy()]
    tot = [0] * R
    for g in range(nranks):
        p = slc.Plan(layout, rank=g, nranks=nranks)
        rb = p.record_bytes
        lo = p.info.first_chunk * rb
        part = [r[lo:lo + p.payload_bytes] for r in recs]
        lg = torch.zeros((R, 4), dtype=torch.int64, device=DEV)
        if p.n_chunks:
            p.payload_sqnorm(part, lg)
        tot = [a + _limbs_value(x) for a, x in zip(tot, lg.cpu().numpy())]
    assert tot == want


# ---------------------------------------------------------------- SLC1 wire format (NEXT row f2)
@pytest.mark.parametrize("name,nranks", [("ragged", 1), ("ragged", 3), ("1m-1d", 2)])
def test_wire_encode_decode_parity(name, nranks):
    """GPU encode of compress output == the oracle's bit-string encoding of the
    same records (byte for byte); decode(encode(x)) == x bit for bit;
    the shards' bodies concatenate to the whole message body."""
    from oracle import wire
    from helpers import shard_chunk_lengths
    layout = layouts.LAYOUTS[name]
    g = oracle.geom()
    bodies = []
    for rank in range(nranks):
        plan = slc.Plan(layout, rank=rank, nranks=nranks)
        if plan.n_chunks == 0:
            continue
        theta, tl, ef, rec = _compress_gpu(plan, layout, 17, 1, "f32", 4, True)
        body_bytes, body_off = plan.wire_layout()
        w = torch.zeros(body_bytes, dtype=torch.uint8, device=DEV)
        plan.wire_encode(rec, w)
        rw = rec.cpu().numpy().view(np.uint32).reshape(-1, plan.record_bytes // 4)
        lens = shard_chunk_lengths(plan)
        want = b"".join(wire.encode_chunk(*wire.record_to_chunk(r, oracle.effective_k(n, g))) for r, n in zip(rw, lens))
        got = bytes(w.cpu().numpy())
        assert got == want
        back = torch.zeros_like(rec)
        plan.wire_decode(w, back)
        assert plan.get_status() == slc.OK
        assert torch.equal(back, rec)
        bodies.append((body_off, got))
    off = 0
    for o, b in bodies:
        assert o == off
        off += len(b)


def test_wire_decode_rejects_invalid_chunks():
    from oracle import wire
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout)
    theta, tl, ef, rec = _compress_gpu(plan, layout, 19, 2, "f32", 0, True)
    nb, _ = plan.wire_layout()
    w = torch.zeros(nb, dtype=torch.uint8, device=DEV)
    plan.wire_encode(rec, w)
    good = w.cpu().numpy().copy()
    size0 = wire.chunk_wire_bytes(64)
    cases = {
        "count": lambda b: b.__setitem__(1, b[1] ^ 1),
        "scale_inf": lambda b: b.__setitem__(4, 0x7C),
        "lo_gt_hi": lambda b: (b.__setitem__(2, 0x7B), b.__setitem__(3, 0xFF)),
        "order": lambda b: b.__setitem__(6, 0xFF),  # first index -> >= 0xFF0 > the second
        "padding": None,
    }
    for name, f in cases.items():
        b = good.copy()
        if f is None:
            continue  # 64 indices x 12 bits and 64 codes x 2 bits fill whole bytes: no padding at k = 64
        f(b)
        back = torch.zeros_like(rec)
        plan.wire_decode(torch.from_numpy(b).to(DEV), back)
        assert plan.get_status() == slc.INVALID_DATA, name
    # a truncated body is a format error and nothing is read
    with pytest.raises(slc.SlcError) as ei:
        plan.wire_decode(torch.from_numpy(good[:-1]).to(DEV), torch.zeros_like(rec))
    assert ei.value.status == slc.FORMAT_ERROR
    # untouched bytes decode cleanly again (the latch was cleared by get_status)
    back = torch.zeros_like(rec)
    plan.wire_decode(torch.from_numpy(good).to(DEV), back)
    assert plan.get_status() == slc.OK and torch.equal(back, rec)
    assert size0 == 118


@pytest.mark.parametrize("release", [False, True])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ef_offload_parity(release, dtype):
    """Row f3: EF kept in pinned host memory, swapped in for slc_compress and out after it
    (overlapping the fused update on the compute stream).  Records and the host EF after the swap-out are
    bit-identical to the oracle; a second step from the swapped-out EF equals the oracle's second step."""
    from paper_2603_08163_b200.offload import EFOffload
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout, dtype=dtype)
    theta, tl, ef = make_device_inputs(plan, layout, 5, 2, dtype, 0, True)
    off = EFOffload(plan, release=release)
    off.host.copy_(ef.cpu())
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    stream = torch.cuda.current_stream()
    off.compress(theta, tl, rec, beta=0.95, stream=stream)
    plan.outer_update(theta, 1.0, records=[rec], stream=stream)  # overlaps the swap-out
    off.wait(stream)
    torch.cuda.synchronize()
    assert plan.get_status() == slc.OK
    ref_rec, ref_ef, _ = oracle_compress_shard(plan, layout, 5, 2, dtype, 0, True)
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), ref_rec)
    host = off.host.clone()
    for s, e in zip(plan.segments, ref_ef):
        assert np.array_equal(bits(seg_view(host, s).numpy()), bits(e)), f"EF differs in segment {s.tensor}"
    # second step: resident EF path on copies of the same state must agree bitwise with the offloaded one
    ef2 = host.to(DEV)
    th2, tl2 = theta.clone(), tl.clone()
    rec2 = torch.zeros_like(rec)
    plan.compress(th2, tl2, ef2, rec2)
    off.compress(theta, tl, rec, beta=0.95, stream=stream)
    off.wait(stream)
    torch.cuda.synchronize()
    assert torch.equal(rec, rec2)
    assert torch.equal(off.host, ef2.cpu())


@pytest.mark.parametrize("name", ["ragged", "1m-2d", "1m-1d"])
@pytest.mark.parametrize("n_pieces", [1, 3, 16])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_compress_range_and_pipelined_offload(name, n_pieces, dtype):
    """slc_compress_range over the pieces of shard_pieces is bitwise slc_compress (chunks are independent);
    the pipelined EF swap (row f3) gives the oracle's records and EF."""
    from paper_2603_08163_b200.offload import EFOffload, shard_pieces
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype=dtype)
    theta, tl, ef = make_device_inputs(plan, layout, 7, 1, dtype, 4, False)
    ef0 = ef.clone()
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    for c0, nc, _, _ in reversed(shard_pieces(plan, n_pieces)):
        plan.compress_range(c0, nc, theta, tl, ef, rec)
    ref_rec, ref_ef, _ = oracle_compress_shard(plan, layout, 7, 1, dtype, 4, False)
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), ref_rec)
    for s, e in zip(plan.segments, ref_ef):
        assert np.array_equal(bits(seg_view(ef, s).cpu().numpy()), bits(e))
    with pytest.raises(slc.SlcError):
        plan.compress_range(plan.n_chunks, 1, theta, tl, ef, rec)
    off = EFOffload(plan, n_pieces=n_pieces, release=n_pieces == 3)
    off.host.copy_(ef0.cpu())
    rec2 = torch.zeros_like(rec)
    off.compress_pipelined(theta, tl, rec2)
    off.wait()
    torch.cuda.synchronize()
    assert plan.get_status() == slc.OK
    assert torch.equal(rec2, rec)
    for s, e in zip(plan.segments, ref_ef):
        assert np.array_equal(bits(seg_view(off.host, s).numpy()), bits(e))


@pytest.mark.parametrize("name", ["ragged", "1m-2d", "1m-1d"])
@pytest.mark.parametrize("special", [0, 4])
def test_index_rank_parity(name, special):
    """Row f4 (R#28): slc_index_rank on ORACLE records equals the oracle's colex rank of the decoded
    positions, limb for limb; every rank fits in ceil(log2 binom(C_eff, k_eff)) bits."""
    from oracle import index_coding as ic
    from helpers import shard_chunk_lengths
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype="f32")
    ref_rec, _, _ = oracle_compress_shard(plan, layout, 11, 3, "f32", special, special == 0)
    rec = torch.from_numpy(ref_rec.view(np.uint8).copy()).to(DEV)
    ranks = torch.full((plan.n_chunks * 16,), -1, dtype=torch.int32, device=DEV)
    plan.index_rank(rec, ranks)
    torch.cuda.synchronize()
    got = ranks.cpu().numpy().view(np.uint32).reshape(plan.n_chunks, 16)
    RW = ref_rec.size // plan.n_chunks
    g = oracle.geom(plan.geom.block, plan.geom.k, plan.geom.index_bits)
    for c, n in enumerate(shard_chunk_lengths(plan)):
        pos = [int(p) for p in oracle.decode_chunk(ref_rec[c * RW:(c + 1) * RW], n, g)[0]]
        want = ic.rank(pos, n)
        assert want.bit_length() <= ic.code_bits(n, len(pos))
        assert sum(int(w) << (32 * l) for l, w in enumerate(got[c])) == want, f"chunk {c}"


def test_index_rank_unsupported_geometry():
    plan = slc.Plan(layouts.LAYOUTS["ragged"], geom=slc.geometry(32, 16))
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    ranks = torch.zeros(plan.n_chunks * 16, dtype=torch.int32, device=DEV)
    with pytest.raises(slc.SlcError):
        plan.index_rank(rec, ranks)


@pytest.mark.parametrize("name", ["ragged", "1m-2d", "1m-1d"])
@pytest.mark.parametrize("special", [0, 4])
def test_index_ec_encode_decode_parity(name, special):
    """Row f4 (R#28): GPU entropy-coded records equal the oracle's EC records word
    for word; the GPU unrank (slc_index_decode) gives back the fixed-width records
    bit for bit, from the GPU's and from the oracle's EC records."""
    from oracle import index_coding as ic
    from helpers import shard_chunk_lengths
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype="f32")
    ref_rec, _, _ = oracle_compress_shard(plan, layout, 13, 2, "f32", special, special == 0)
    rec = torch.from_numpy(ref_rec.view(np.uint8).copy()).to(DEV)
    assert plan.ec_record_bytes == 80
    ec = torch.zeros(plan.n_chunks * plan.ec_record_bytes, dtype=torch.uint8, device=DEV)
    plan.index_encode(rec, ec)
    RW = ref_rec.size // plan.n_chunks
    lens = shard_chunk_lengths(plan)
    want = np.array([ic.ec_from_record(ref_rec[c * RW:(c + 1) * RW], n) for c, n in enumerate(lens)], np.uint32)
    got = ec.cpu().numpy().view(np.uint32).reshape(plan.n_chunks, -1)
    assert np.array_equal(got, want)
    back = torch.zeros_like(rec)
    plan.index_decode(ec, back)
    assert plan.get_status() == slc.OK
    assert torch.equal(back, rec)
    back2 = torch.zeros_like(rec)
    plan.index_decode(torch.from_numpy(want.view(np.uint8).copy().reshape(-1)).to(DEV), back2)
    assert plan.get_status() == slc.OK and torch.equal(back2, rec)
    # a rank beyond binom(C_eff, k_eff) is not a code: INVALID_DATA
    bad = want.copy()
    bad[0, 14] = 0x00FFFFFF
    plan.index_decode(torch.from_numpy(bad.view(np.uint8).copy().reshape(-1)).to(DEV), back2)
    assert plan.get_status() == slc.INVALID_DATA
