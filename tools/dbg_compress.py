"""Run slc_compress once on a named layout (fresh process per layout) and compare
against the non-TMA kernel path; prints OK / the CUDA error.  Debug aid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import make_device_inputs  # noqa: E402
from paper_2603_08163_b200 import slc  # noqa: E402

LAYOUTS = {
    "one_big": [("w", (4096, 512))],
    "two_big": [("a", (4096, 512)), ("b", (2048, 512))],
    "mat_norm": [("a", (4096, 512)), ("n", (512,)), ("b", (2048, 512))],
    "flat_full": [("a", (4096 * 600,))],
    "tiny": None,
    "x2": [("w", (64 * 296, 64))],
    "m1": [("w", (1024, 1024))],
    "m1b": [("w", (1024, 2048))],
    "m1c": [("w", (2048, 1024))],
    "x3": [("w", (64 * 444, 64))],
    "x4": [("w", (64 * 592, 64))],
    "x13": [("w", (64 * 148 * 13, 64))],
}
name = sys.argv[1]
if name == "tiny":
    from slcgen import layouts
    layout = layouts.LAYOUTS["llama-tiny"]
else:
    layout = LAYOUTS[name]
plan = slc.Plan(layout)
th, tl, ef = make_device_inputs(plan, layout, 1, 0, warm_ef=True)
rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device="cuda")
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    print("rep", rep, flush=True)
    plan.compress(th, tl, ef, rec)
    torch.cuda.synchronize()
print(name, "chunks", plan.n_chunks, "OK status", plan.get_status())
