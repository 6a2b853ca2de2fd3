"""Drive every CUDA entry point of libslc.so once, at small sizes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Usage (GPU box):
  compute-sanitizer --tool racecheck --kernel-name regex:'^(?!slcgen)' \
      python tools/sanitize_paths.py [--quick]
No oracle involvement: this only exercises the kernels (every path: compress
on clean / special / bf16 chunks, the fused pipelined and simple decode /
aggregate / update, weighted, median-norm, wire, index rank)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import slcgen  # noqa: E402
from slcgen import layouts  # noqa: E402
from paper_2603_08163_b200 import slc  # noqa: E402

DEV = torch.device("cuda:0")


def fill(plan, layout, buf, what, seed, peer, **kw):
    offs, o = [], 0
    for _, shape in layout:
        offs.append(o)
        o += int(np.prod(shape))
    for s in plan.segments:
        slcgen.fill_cuda(buf[s.shard_offset:s.shard_offset + s.n_elems], what, seed, peer,
                         offs[s.tensor] + s.tensor_begin, **kw)


def run(layout_name: str, dtype: str, R: int, special: int):
    layout = layouts.LAYOUTS[layout_name]
    plan = slc.Plan(layout, dtype=dtype)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n = plan.shard_elems
    theta = torch.zeros(n, dtype=tdt, device=DEV)
    fill(plan, layout, theta, slcgen.WHAT_THETA, 1, 0, special_period=special)
    recs = []
    for r in range(R):
        tl = torch.zeros(n, dtype=tdt, device=DEV)
        ef = torch.zeros(n, dtype=torch.float32, device=DEV)
        fill(plan, layout, tl, slcgen.WHAT_THETA_LOCAL, 1, r, special_period=special)
        fill(plan, layout, ef, slcgen.WHAT_EF, 1, r, special_period=special, warm_ef=(r % 2 == 0))
        rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device=DEV)
        plan.compress(theta, tl, ef, rec)
        recs.append(rec)
    plan.check()
    agg = torch.zeros(n, dtype=torch.float32, device=DEV)
    plan.decode_aggregate(recs, agg)
    th = theta.clone()
    plan.outer_update(th, 0.65, agg=agg)
    th = theta.clone()
    plan.outer_update(th, 0.65, records=recs)
    w = [0.5 + 0.25 * r for r in range(R)]
    plan.decode_aggregate(recs, agg, weights=w)
    plan.outer_update(th, 1.0, records=recs, weights=w)
    sq = torch.zeros(R, 4, dtype=torch.int64, device=DEV)
    plan.payload_sqnorm(recs, sq)
    wd = torch.zeros(R, dtype=torch.float32, device=DEV)
    plan.median_norm_weights(sq, wd)
    plan.decode_aggregate(recs, agg, weights_dev=wd)
    plan.outer_update(th, 1.0, records=recs, weights_dev=wd)
    plan.check()
    body, _ = plan.wire_layout()
    wire = torch.zeros(body, dtype=torch.uint8, device=DEV)
    plan.wire_encode(recs[0], wire)
    back = torch.zeros_like(recs[0])
    plan.wire_decode(wire, back)
    ranks = torch.zeros(plan.n_chunks * 16, dtype=torch.int32, device=DEV)
    plan.index_rank(recs[0], ranks)
    plan.check()
    torch.cuda.synchronize()
    print(f"ok {layout_name} {dtype} R={R} special={special}", flush=True)


def main():
    quick = "--quick" in sys.argv
    cases = [("ragged", "f32", 3, 4), ("ragged", "bf16", 2, 0)]
    if not quick:
        cases += [("1m-2d", "f32", 2, 8), ("1m-1d", "bf16", 2, 32)]
    for c in cases:
        run(*c)
    for variant in (2, 3):  # pipelined, one CTA per chunk
        slc.Plan.default_options = {slc.OPT_AGG_KERNEL: variant}
        run("ragged", "f32", 3, 4)
    print("sanitize_paths done")


if __name__ == "__main__":
    main()
