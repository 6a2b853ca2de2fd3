"""The hand-worked cases of tests/golden/oracle_pins.json through the CUDA path
(C ABI): the GPU must reach the same hand-derived values as the oracle — the
partial-chunk threshold (R#10), the |v| == tau boundary, the tau
fallback, the sign bit of a selected -0 (R#25), the canonical-order fp64 sum
with w = 2^60 (R#17; the sequential weighted path), and the R = 49 invR
product (R#17)."""
import numpy as np
import pytest

from helpers import record_from_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")
def _expand(ranges, n):
    v = np.zeros(n, np.float32)
    for a, b, x in ranges:
        v[a:b] = x
    return v


@pytest.mark.parametrize("case", [0, 2, 3, 4])
@pytest.mark.parametrize("shape", ["flat", "block"])
def test_quantizer_hand_worked_cases_gpu(golden, case, shape):
    c = golden["oracle_pins"]["quantizer"][case]
    n = c["n"]
    if shape == "block" and n != 4096:
        pytest.skip("partial chunks are flat")
    layout = [("v", (n,))] if shape == "flat" else [("w", (64, 64))]  # one 64x64 block: p = 64r + c = flat order
    plan = slc.Plan(layout)
    a = _expand(c["values"], n)
    e = np.zeros(n, np.float32)
    for p in c.get("negative_zero_positions", []):
        a[p] = np.float32(-0.0)
        e[p] = np.float32(-0.0)
    theta = torch.from_numpy(a).to(DEV)
    tl = torch.zeros(n, dtype=torch.float32, device=DEV)
    ef = torch.from_numpy(e).to(DEV)
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
    plan.compress(theta, tl, ef, rec)
    assert plan.get_status() == slc.OK
    w = rec.cpu().numpy().view(np.uint32)
    assert w[-1] & 0xFFFF == int(c["scale_lo_f16"], 16) and w[-1] >> 16 == int(c["scale_hi_f16"], 16)
    # decode through the GPU aggregate (R = 1: Delta = decoded values)
    agg = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.decode_aggregate([rec], agg)
    got = agg.cpu().numpy()
    if "decode" in c:
        assert np.array_equal(got, _expand(c["decode"], n))
    if "sign_bit_slots" in c:
        for p in c["negative_zero_positions"]:
            assert got[p].view(np.uint32) == 0          # acc = +0.0 + (-0) = +0 (R#17 starts at +0.0)
            assert ef.cpu().numpy()[p].view(np.uint32) == 0       # -0 - (-0) = +0


@pytest.mark.parametrize("case", [0, 1])
def test_canonical_peer_order_gpu(golden, case, agg_kernel):
    c = golden["oracle_pins"]["aggregate_order"][case]
    n = 4096
    plan = slc.Plan([("v", (n,))])
    recs = [torch.from_numpy(record_from_values({0: p["dq"]}, n, 64).view(np.uint8).copy()).to(DEV)
            for p in c["peers"]]
    ids = [bytes([0] * 15 + [p["id"]]) for p in c["peers"]]
    hdrs = [slc.make_header(plan, ids[i], base_round=1) for i in range(3)]
    w = np.array([p["w"] for p in c["peers"]], np.float32)
    order = c["pass_order"]
    agg = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.decode_aggregate([recs[i] for i in order], agg, hdrs=[hdrs[i] for i in order], weights=w[order])
    assert agg[0].item() == np.float32(c["delta"]) and agg[1:].abs().max().item() == 0
    agg2 = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.decode_aggregate([recs[i] for i in order], agg2, hdrs=[hdrs[i] for i in order],
                          weights_dev=torch.from_numpy(w[order]).to(DEV))
    assert torch.equal(agg2, agg)
    th = torch.full((n,), 1.0, dtype=torch.float32, device=DEV)
    plan.outer_update(th, 1.0, records=[recs[i] for i in order], hdrs=[hdrs[i] for i in order], weights=w[order])
    assert plan.get_status() == slc.OK
    assert th[0].item() == np.float32(np.float32(1.0) - np.float32(c["delta"]))


def test_delta_is_acc_times_inv_r_gpu(golden, agg_kernel):
    c = golden["oracle_pins"]["aggregate_inv_r"]
    R, n = c["R"], 4096
    plan = slc.Plan([("v", (n,))])
    recs = []
    for r in range(R):
        vals = {0: c["parts_units_2^-24"][r] * 2.0 ** -24} if r < 3 else {1 + r: 0.5}
        recs.append(torch.from_numpy(record_from_values(vals, n, 64).view(np.uint8).copy()).to(DEV))
    agg = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.decode_aggregate(recs, agg)
    assert plan.get_status() == slc.OK
    assert agg[0].item() == np.float32(c["delta"]) != np.float32(c["delta_if_divided"])
    th = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.outer_update(th, -1.0, records=recs)
    assert th[0].item() == np.float32(c["delta"])
