"""Per-phase cycle breakdown of the batched decode kernel (SLC_BATCH_TIMING build):
  python tools/build_variants.py bt=SLC_BATCH_TIMING
  SLC_LIB=build/variants/libslc_bt.so python tools/batch_timing.py [layout] [nranks] [R] [dtype]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import make_device_inputs  # noqa: E402
from paper_2603_08163_b200 import slc  # noqa: E402
from slcgen import layouts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
nranks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
R = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dtype = sys.argv[4] if len(sys.argv) > 4 else "f32"
lib = ctypes.CDLL(slc.LIB_PATH)
layout = layouts.LAYOUTS[name]
plan = slc.Plan(layout, rank=0, nranks=nranks, dtype=dtype)
plan.set_option(slc.OPT_AGG_KERNEL, 1)
theta = None
recs = []
for r in range(R):
    theta, tl, ef = make_device_inputs(plan, layout, 1, r, dtype, warm_ef=True, theta=theta)
    rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device="cuda")
    plan.compress(theta, tl, ef, rec)
    recs.append(rec)
del tl, ef
buf = (ctypes.c_ulonglong * 8)()
plan.outer_update(theta, 1.0, records=recs)
torch.cuda.synchronize()
lib.slc_debug_batch_cycles(buf, 1)
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); plan.outer_update(theta, 1.0, records=recs); b.record(); torch.cuda.synchronize()
lib.slc_debug_batch_cycles(buf, 0)
n = plan.n_chunks
names = ["top (TMA issue, desc)", "scatter", "B1 wait", "build (warp 0)", "wait tile + convert/update", "B2 wait",
         "store issue"]
tot = sum(buf[i] for i in range(7))
print(f"fused update {a.elapsed_time(b):.3f} ms, {n} chunks, R={R}, {dtype}; warp-cycles per chunk (8 warps):")
for i, nm in enumerate(names):
    print(f"  {nm:24s} {buf[i] / n:10.0f}  {100 * buf[i] / tot:5.1f}%")
print(f"  {'total':24s} {tot / n:10.0f}")
