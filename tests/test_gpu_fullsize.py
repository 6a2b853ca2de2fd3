"""Full-size parity in bench.py's launch configuration: the Llama-3.2-1B-shaped
param set (1,235,814,400 params, BASELINE.json configs[1]) with R = 8 peers,
compress + fused aggregate/update through the C ABI exactly as bench.py runs
them; then a seeded sample of chunks (random ones, every partial chunk, the
first and the last) is recomputed one by one by the oracle from the same
seeded inputs and compared bit for bit (records, EF, theta)."""
import numpy as np
import pytest

import oracle
import slcgen
from slcgen import layouts

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")
BETA, ALPHA = 0.95, 1.0


def _fill(plan, layout, buf, what, peer, **kw):
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in layout])
    for s in plan.segments:
        slcgen.fill_cuda(buf[s.shard_offset:s.shard_offset + s.n_elems], what, 0, peer,
                         int(offs[s.tensor]) + s.tensor_begin, **kw)


def _chunk_map(plan, layout, c):
    """(tensor index, chunk within tensor, shard offsets of its positions, global indices)."""
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in layout])
    for s in plan.segments:
        if s.first_chunk <= c < s.first_chunk + s.n_chunks:
            shape = layout[s.tensor][1]
            tc = c - s.first_chunk + oracle_first_chunk(shape, s)
            toff = oracle.chunk_offsets(shape, tc)
            return s.tensor, tc, s.shard_offset + (toff - s.tensor_begin), offs[s.tensor] + toff
    raise IndexError(c)


def oracle_first_chunk(shape, s):
    if s.blocked:
        return s.tensor_begin // (64 * shape[1]) * (shape[1] // 64)
    return s.tensor_begin // 4096


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_llama1b_sampled_parity(dtype):
    layout = layouts.LAYOUTS["llama3.2-1b"]
    R = 8
    plan = slc.Plan(layout, dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n = plan.shard_elems
    theta = torch.empty(n, dtype=tdt, device=DEV)
    tl = torch.empty(n, dtype=tdt, device=DEV)
    ef = torch.empty(n, dtype=torch.float32, device=DEV)
    _fill(plan, layout, theta, slcgen.WHAT_THETA, 0, special_period=64)
    recs = []
    ef0 = None
    for r in range(R):
        _fill(plan, layout, tl, slcgen.WHAT_THETA_LOCAL, r, special_period=64)
        _fill(plan, layout, ef, slcgen.WHAT_EF, r, special_period=64, warm_ef=True)
        rec = torch.empty(plan.payload_bytes, dtype=torch.uint8, device=DEV)
        plan.compress(theta, tl, ef, rec, beta=BETA)
        recs.append(rec)
        if r == 0:
            ef0 = ef.clone()
    theta_new = theta.clone()
    plan.outer_update(theta_new, ALPHA, records=recs)
    torch.cuda.synchronize()
    assert plan.get_status() == slc.OK
    del tl, ef

    rng = np.random.default_rng(123)
    partial = [s.first_chunk + s.n_chunks - 1 for s in plan.segments if not s.blocked]
    sample = sorted(set(rng.choice(plan.n_chunks, 120, replace=False).tolist() + partial +
                        [0, plan.n_chunks - 1]))
    RW = oracle.record_words()
    rec_host = [r.view(torch.int32) for r in recs]
    for c in sample:
        ti, tc, shard_off, G = _chunk_map(plan, layout, c)
        idx = torch.from_numpy(shard_off.astype(np.int64)).to(DEV)
        th_gpu = theta.index_select(0, idx).cpu()
        th_new = theta_new.index_select(0, idx).cpu()
        a = slcgen.generate_at(0, 0, 0, G, dtype=dtype, special_period=64)
        if dtype == "bf16":
            assert np.array_equal(th_gpu.view(torch.int16).numpy().view(np.uint16), a)
        else:
            assert np.array_equal(th_gpu.numpy().view(np.uint32), a.view(np.uint32))
        ref_recs = []
        for r in range(R):
            l = slcgen.generate_at(1, 0, r, G, dtype=dtype, special_period=64)
            e = slcgen.generate_at(2, 0, r, G, special_period=64, warm_ef=True)
            st, rec, e_new = oracle.compress_chunk(a, l, e, BETA)
            assert st == 0
            got = rec_host[r][c * RW:(c + 1) * RW].cpu().numpy().view(np.uint32)
            assert np.array_equal(got, rec), f"record mismatch chunk {c} peer {r}"
            if r == 0:
                assert np.array_equal(ef0.index_select(0, idx).cpu().numpy().view(np.uint32),
                                      e_new.view(np.uint32)), f"EF mismatch chunk {c}"
            ref_recs.append(rec)
        delta = oracle.aggregate_chunk(ref_recs, len(G))
        ref_theta = oracle.outer_update(a, delta, ALPHA)
        got = th_new.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else th_new.numpy()
        assert np.array_equal(got.view(ref_theta.dtype), ref_theta), f"theta mismatch chunk {c}"
