"""Parity at the target configuration's scale (BASELINE.json configs[3],
north_star: Covenant-72B sharded over 8 B200, R = 20) and on the paths only
large inputs reach:

* one GPU's shard of the 8-way 72B job (rank 0 and rank 7; 9.09 G elements, so
  shard offsets pass 2^32), fp32 and bf16, R = 20 — compress + fused update
  exactly as bench.py runs them, then sampled chunks (random, first, last,
  every flat partial chunk) recomputed one by one by the oracle;
* a 64-row blocked tensor with 2^24 columns (row stride >= 2^24 routes
  slc_compress to the warp-per-chunk kernel, compress_warp.cu);
* crafted payloads with R = 128 and R = 256 (the ABI maximum);
* bf16 theta with median-norm style weights through the fused update;
* bf16 with cold EF (round 0, e = 0): d = theta - theta_local is a small
  multiple of the bf16 ulp, so many magnitudes tie.
"""
import gc

import numpy as np
import pytest

import oracle
import slcgen
from helpers import bits, craft_records, host_segment, make_device_inputs, oracle_compress_shard, \
    oracle_update_shard, seg_view
from slcgen import layouts

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")
BETA, ALPHA = 0.95, 1.0


def _free():
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _fill(plan, layout, buf, what, peer, **kw):
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in layout])
    for s in plan.segments:
        slcgen.fill_cuda(buf[s.shard_offset:s.shard_offset + s.n_elems], what, 0, peer,
                         int(offs[s.tensor]) + s.tensor_begin, **kw)


def _seg_chunks(plan, layout):
    """Per shard chunk: (segment, chunk within the segment's own shape)."""
    out = []
    for s in plan.segments:
        for j in range(s.n_chunks):
            out.append((s, j))
    return out


def _chunk_positions(plan, layout, s, j):
    """Shard offsets and global element indices of chunk j of segment s."""
    offs = np.cumsum([0] + [int(np.prod(sh)) for _, sh in layout])
    shape = (s.rows, s.cols) if s.blocked else (s.n_elems,)
    loc = oracle.chunk_offsets(shape, j)
    return s.shard_offset + loc, int(offs[s.tensor]) + s.tensor_begin + loc


def _sampled_parity(layout, plan, dtype, R, special, n_random, seed=123, warm=True):
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n = plan.shard_elems
    theta = torch.empty(n, dtype=tdt, device=DEV)
    tl = torch.empty(n, dtype=tdt, device=DEV)
    ef = torch.empty(n, dtype=torch.float32, device=DEV)
    _fill(plan, layout, theta, slcgen.WHAT_THETA, 0, special_period=special)
    chunks = _seg_chunks(plan, layout)
    rng = np.random.default_rng(seed)
    last_flat = [i for i, (s, j) in enumerate(chunks) if not s.blocked and j == s.n_chunks - 1]
    sample = sorted(set(rng.choice(len(chunks), n_random, replace=False).tolist() + last_flat[:40] +
                        [0, len(chunks) - 1]))
    pos = {c: _chunk_positions(plan, layout, *chunks[c]) for c in sample}
    idx_all = torch.from_numpy(np.concatenate([pos[c][0] for c in sample]).astype(np.int64)).to(DEV)
    th_before = theta.index_select(0, idx_all).cpu()
    recs, ef0 = [], None
    for r in range(R):
        _fill(plan, layout, tl, slcgen.WHAT_THETA_LOCAL, r, special_period=special)
        _fill(plan, layout, ef, slcgen.WHAT_EF, r, special_period=special, warm_ef=warm)
        rec = torch.empty(plan.payload_bytes, dtype=torch.uint8, device=DEV)
        plan.compress(theta, tl, ef, rec, beta=BETA)
        recs.append(rec)
        if r == 0:
            ef0 = ef.index_select(0, idx_all).cpu()
    del tl, ef
    plan.outer_update(theta, ALPHA, records=recs)
    torch.cuda.synchronize()
    assert plan.get_status() == slc.OK
    th_after = theta.index_select(0, idx_all).cpu()
    RW = oracle.record_words()
    sample_rows = torch.tensor([c for c in sample], dtype=torch.int64, device=DEV)
    rec_rows = [r.view(torch.int32).view(-1, RW).index_select(0, sample_rows).cpu().numpy().view(np.uint32)
                for r in recs]
    del theta, recs
    _free()
    o = 0
    for i, c in enumerate(sample):
        shard_off, G = pos[c]
        m = len(G)
        sl = slice(o, o + m)
        o += m
        a = slcgen.generate_at(0, 0, 0, G, dtype=dtype, special_period=special)
        tb = th_before[sl]
        got_a = tb.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else tb.numpy()
        assert np.array_equal(bits(got_a), bits(a)), f"theta input differs at chunk {c}"
        ref_recs = []
        for r in range(R):
            l = slcgen.generate_at(1, 0, r, G, dtype=dtype, special_period=special)
            e = slcgen.generate_at(2, 0, r, G, special_period=special, warm_ef=warm)
            st, rec, e_new = oracle.compress_chunk(a, l, e, BETA)
            assert st == 0
            assert np.array_equal(rec_rows[r][i], rec), f"record mismatch chunk {c} peer {r}"
            if r == 0:
                assert np.array_equal(bits(ef0[sl].numpy()), bits(e_new)), f"EF mismatch chunk {c}"
            ref_recs.append(rec)
        delta = oracle.aggregate_chunk(ref_recs, m)
        ref_theta = oracle.outer_update(a, delta, ALPHA)
        ta = th_after[sl]
        got = ta.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else ta.numpy()
        assert np.array_equal(bits(got), bits(ref_theta)), f"theta mismatch chunk {c}"
    return sample


@pytest.mark.parametrize("rank,dtype", [(0, "f32"), (7, "f32"), (7, "bf16")])
def test_covenant72b_shard_of_8_sampled_parity(rank, dtype):
    """One GPU's shard of the target job (north_star config 4), R = 20, exactly
    as `bench.py --workload covenant-72b --shard-of 8 --shard-rank R` runs it."""
    free, total = torch.cuda.mem_get_info()
    layout = layouts.LAYOUTS["covenant-72b"]
    plan = slc.Plan(layout, rank=rank, nranks=8, dtype=dtype)
    need = plan.shard_elems * (3 * (4 if dtype == "f32" else 2) + 4) + 21 * plan.payload_bytes
    if free < need + (2 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB free")
    assert plan.shard_elems > 2 ** 32
    sample = _sampled_parity(layout, plan, dtype, R=20, special=64, n_random=60, seed=rank)
    assert plan.n_chunks - 1 in sample
    _free()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_wide_blocked_tensor_takes_warp_kernel(dtype):
    """(64, 2^24) is 64x64-blocked with a row stride of 2^24 elements: the
    persistent kernel's 32-bit in-chunk offsets do not fit and slc_compress
    runs compress_warp.cu; sampled chunks (incl. the last block column)."""
    layout = [("wide", (64, 1 << 24))]
    plan = slc.Plan(layout, dtype=dtype)
    sample = _sampled_parity(layout, plan, dtype, R=3, special=32, n_random=40, seed=5)
    assert plan.n_chunks - 1 in sample
    _free()


@pytest.mark.parametrize("R", [128, 256])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_crafted_many_peers(R, dtype, agg_kernel):
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout, dtype=dtype)
    rng = np.random.default_rng(R)
    theta, _, _ = make_device_inputs(plan, layout, 21, 0, dtype)
    thetas = [host_segment(layout, s, slcgen.WHAT_THETA, 21, 0, dtype) for s in plan.segments]
    ref_recs = [craft_records(plan, rng, 1, 16) for _ in range(R)]
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    agg = torch.zeros(plan.shard_elems, dtype=torch.float32, device=DEV)
    plan.decode_aggregate(recs, agg)
    for s, d in zip(plan.segments, oracle_update_shard(plan, thetas, ref_recs, 1.0, only_delta=True)):
        assert np.array_equal(bits(seg_view(agg, s).cpu().numpy()), bits(d))
    plan.outer_update(theta, 0.65, records=recs)
    assert plan.get_status() == slc.OK
    for s, t in zip(plan.segments, oracle_update_shard(plan, thetas, ref_recs, 0.65)):
        got = seg_view(theta, s).cpu()
        if dtype == "bf16":
            got = got.view(torch.int16)
        assert np.array_equal(bits(got.numpy()), bits(t))


@pytest.mark.parametrize("exps,wspan", [((4, 9), 1.0), ((2, 14), 1e4)])
def test_bf16_weighted_fused_update(exps, wspan, agg_kernel):
    """bf16 theta + weights (median-norm) through the fused update, both the
    exact fixed-point (narrow) and the sequential fp64 (wide) weighted paths."""
    layout = layouts.LAYOUTS["ragged"]
    plan = slc.Plan(layout, dtype="bf16")
    rng = np.random.default_rng(900 + exps[1])
    R = 20
    theta, _, _ = make_device_inputs(plan, layout, 33, 0, "bf16")
    thetas = [host_segment(layout, s, slcgen.WHAT_THETA, 33, 0, "bf16") for s in plan.segments]
    ref_recs = [craft_records(plan, rng, *exps) for _ in range(R)]
    recs = [torch.from_numpy(r.view(np.uint8).copy()).to(DEV) for r in ref_recs]
    ids = [bytes(rng.integers(0, 256, 16, dtype=np.uint8)) for _ in range(R)]
    hdrs = [slc.make_header(plan, ids[r], base_round=2) for r in range(R)]
    w = (np.exp(rng.uniform(-np.log(wspan), np.log(wspan), R)) if wspan > 1
         else rng.uniform(0.5, 1.5, R)).astype(np.float32)
    th2 = theta.clone()
    plan.outer_update(theta, 0.65, records=recs, hdrs=hdrs, weights=w)
    plan.outer_update(th2, 0.65, records=recs, hdrs=hdrs, weights_dev=torch.from_numpy(w).to(DEV))
    assert plan.get_status() == slc.OK
    ref = oracle_update_shard(plan, thetas, ref_recs, 0.65, peer_ids=np.frombuffer(b"".join(ids), np.uint8),
                              weights=w)
    for s, t in zip(plan.segments, ref):
        for th in (theta, th2):
            assert np.array_equal(bits(seg_view(th, s).cpu().view(torch.int16).numpy()), bits(t))


@pytest.mark.parametrize("name", ["1m-2d", "1m-1d", "llama-tiny"])
def test_bf16_cold_ef_compress_parity(name):
    """Round 0 (e = 0) with bf16 params: b = theta - theta_local exactly, a small
    multiple of the bf16 ulp, so many chunk magnitudes tie at the k-th value."""
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype="bf16")
    theta, tl, ef = make_device_inputs(plan, layout, 3, 1, "bf16", 0, False)
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    plan.compress(theta, tl, ef, rec)
    assert plan.get_status() == slc.OK
    ref_rec, ref_ef, _ = oracle_compress_shard(plan, layout, 3, 1, "bf16", 0, False)
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), ref_rec)
    for s, e in zip(plan.segments, ref_ef):
        assert np.array_equal(bits(seg_view(ef, s).cpu().numpy()), bits(e))
