"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool,
profiles/r02_compute_sanitizer_refused.txt): every buffer the C ABI touches is
placed inside a larger allocation whose guard bands (before and after) and
inter-segment padding hold a poison pattern — NaN for the dense fp32 / bf16
buffers, so a stray READ of padding would also surface as a latched
INVALID_DATA in compress, 0xA5 bytes for records / wire / ranks.  After each
entry point runs (compress, compress_range, decode_aggregate, fused and
weighted updates on every decode kernel, payload_sqnorm, median weights, wire
encode / decode, index rank / encode / decode, fast checks) the guards and the
padding must be untouched and the status OK."""
import numpy as np
import pytest

from helpers import make_device_inputs
from slcgen import layouts

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")
GUARD = 4096  # elements / bytes of guard on each side (keeps 16-B alignment)


def _guarded(n, dtype, poison):
    big = torch.empty(n + 2 * GUARD, dtype=dtype, device=DEV)
    if dtype == torch.uint8:
        big.fill_(0xA5)
    elif dtype == torch.int32:
        big.fill_(-0x5A5A5A5B)
    else:
        big.fill_(float("nan"))
    return big, big[GUARD:GUARD + n]


def _guards_intact(big, n, dtype):
    g = torch.cat([big[:GUARD], big[GUARD + n:]])
    if dtype in (torch.uint8, torch.int32):
        ref = big[:1].clone().fill_(0xA5 if dtype == torch.uint8 else -0x5A5A5A5B)
        return bool((g == ref).all())
    return bool(torch.isnan(g.float()).all())


def _padding_mask(plan):
    m = torch.ones(plan.shard_elems, dtype=torch.bool)
    for s in plan.segments:
        m[s.shard_offset:s.shard_offset + s.n_elems] = False
    return m.to(DEV)


@pytest.mark.parametrize("name,dtype", [("ragged", "f32"), ("ragged", "bf16"), ("llama-tiny", "f32")])
def test_guard_bands_and_padding(name, dtype, agg_kernel):
    layout = layouts.LAYOUTS[name]
    plan = slc.Plan(layout, dtype=dtype)
    n = plan.shard_elems
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    pad = _padding_mask(plan)
    assert pad.any() or name == "llama-tiny"
    th0, tl0, ef0 = make_device_inputs(plan, layout, 3, 1, dtype, special_period=8, warm_ef=True)
    bufs = {}
    for key, src, dt in (("theta", th0, tdt), ("tl", tl0, tdt), ("ef", ef0, torch.float32)):
        big, v = _guarded(n, dt, None)
        v.copy_(src)
        v[pad] = float("nan")  # padding poisoned: never read (compress would latch INVALID_DATA)
        bufs[key] = (big, v, dt)
    R = 3
    recs = []
    for r in range(R):
        big, rec = _guarded(plan.payload_bytes, torch.uint8, 0xA5)
        _, tl_r, ef_r = make_device_inputs(plan, layout, 3, r, dtype, special_period=8, warm_ef=True, theta=th0)
        bufs["tl"][1][~pad] = tl_r[~pad]
        bufs["ef"][1][~pad] = ef_r[~pad]
        plan.compress(bufs["theta"][1], bufs["tl"][1], bufs["ef"][1], rec)
        assert plan.get_status() == slc.OK
        recs.append((big, rec))
    recv = [r for _, r in recs]
    c0 = plan.n_chunks // 3
    plan.compress_range(c0, plan.n_chunks // 3, bufs["theta"][1], bufs["tl"][1], bufs["ef"][1], recv[0])
    agg_big, agg = _guarded(n, torch.float32, None)
    agg[pad] = float("nan")
    plan.decode_aggregate(recv, agg)
    assert bool(torch.isnan(agg[pad]).all())
    plan.outer_update(bufs["theta"][1], 0.65, records=recv)
    plan.outer_update(bufs["theta"][1], 1.0, records=recv, weights=[0.5, 1.0, 2.0])
    l64 = torch.empty(R * 4 + 2 * GUARD // 8, dtype=torch.int64, device=DEV).fill_(-0x5A5A5A5A5A5A5A5B)
    lv = l64[GUARD // 8:GUARD // 8 + R * 4].view(R, 4)
    plan.payload_sqnorm(recv, lv)
    w = torch.empty(R + 64, dtype=torch.float32, device=DEV).fill_(float("nan"))
    plan.median_norm_weights(lv, w[32:32 + R])
    plan.outer_update(bufs["theta"][1], 1.0, records=recv, weights_dev=w[32:32 + R])
    assert bool(torch.isnan(w[:32]).all()) and bool(torch.isnan(w[32 + R:]).all())
    assert bool((l64[:GUARD // 8] == -0x5A5A5A5A5A5A5A5B).all())
    assert bool((l64[GUARD // 8 + R * 4:] == -0x5A5A5A5A5A5A5A5B).all())
    body, _ = plan.wire_layout()
    wb, wv = _guarded(body, torch.uint8, 0xA5)
    plan.wire_encode(recv[0], wv)
    back_big, back = _guarded(plan.payload_bytes, torch.uint8, 0xA5)
    plan.wire_decode(wv, back)
    assert torch.equal(back, recv[0])
    rk_big, rk = _guarded(plan.n_chunks * 64, torch.uint8, 0xA5)
    plan.index_rank(recv[0], rk)
    ec_big, ec = _guarded(plan.n_chunks * plan.ec_record_bytes, torch.uint8, 0xA5)
    plan.index_encode(recv[0], ec)
    plan.index_decode(ec, back)
    assert torch.equal(back, recv[0])
    fl_big, fl = _guarded(R, torch.int32, 0)
    plan.fast_checks(recv, fl, sqnorm=lv, norm_history=[1.0])
    torch.cuda.synchronize()
    assert plan.get_status() == slc.OK
    for key, (big, v, dt) in bufs.items():
        assert _guards_intact(big, n, dt), f"{key}: guard band written"
        assert bool(torch.isnan(v[pad].float()).all()), f"{key}: padding written"
    for big, _ in recs:
        assert _guards_intact(big, plan.payload_bytes, torch.uint8), "records: guard band written"
    assert _guards_intact(agg_big, n, torch.float32)
    for big, m in ((wb, body), (back_big, plan.payload_bytes), (rk_big, plan.n_chunks * 64),
                   (ec_big, plan.n_chunks * plan.ec_record_bytes)):
        assert _guards_intact(big, m, torch.uint8)
    assert _guards_intact(fl_big, R, torch.int32)
