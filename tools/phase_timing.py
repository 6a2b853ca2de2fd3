"""Per-phase cycle breakdown of the compress warp kernel (SLC_PHASE_TIMING build)."""
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

lib = ctypes.CDLL(slc.LIB_PATH)
layout = layouts.LAYOUTS[sys.argv[1] if len(sys.argv) > 1 else "llama3.2-1b"]
plan = slc.Plan(layout, geom=slc.geometry(int(os.environ.get("BLOCK", 64)), int(os.environ.get("K", 64))),
                rank=0, nranks=int(os.environ.get("NRANKS", 1)), dtype=os.environ.get("DTYPE", "f32"))
th, tl, ef = make_device_inputs(plan, layout, 1, 0, warm_ef=not os.environ.get("COLD"), special_period=int(os.environ.get("SPECIAL", 0)),
                                dtype=os.environ.get("DTYPE", "f32"))
rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device="cuda")
buf = (ctypes.c_ulonglong * 8)()
plan.compress(th, tl, ef, rec)
torch.cuda.synchronize()
fn = getattr(lib, "slc_debug_phase_cycles_ws" if os.environ.get("WS") else "slc_debug_phase_cycles")
fn(buf, 1)
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); plan.compress(th, tl, ef, rec); b.record(); torch.cuda.synchronize()
fn(buf, 0)
n = plan.n_chunks
names = ["A stream", "S threshold", "B candidates", "R rank+slots (incl. fallbacks)", "Q quantise+pack",
         "F EF fix-ups", "stream: wait empty", "select: wait full"]
tot = sum(buf[i] for i in range(8))
print(f"kernel {a.elapsed_time(b):.3f} ms, {n} chunks; cycles per chunk per warp:")
for i, nm in enumerate(names):
    print(f"  {nm:18s} {buf[i] / n:10.0f}  {100 * buf[i] / tot:5.1f}%")
print(f"  {'total':18s} {tot / n:10.0f}")
if os.environ.get("WS"):
    pc = (ctypes.c_ulonglong * 16)()
    lib.slc_debug_path_count_ws(pc)
    print("  selection paths (chunks): candidates %d, tie %d, tie->rank %d, radix %d" % tuple(pc[:4]))
    nt = max(1, pc[1] + pc[2] + pc[3]); nr = max(1, pc[3])
    print("  cycles per call: tie_select %.0f, radix rounds %.0f, radix mark+fill %.0f; radix chunks: mean G %.1f, mean M %.1f"
          % (pc[4] / nt, pc[5] / nr, pc[6] / nr, pc[7] / nr, pc[8] / nr))
    print("  reg_select: %d chunks, %.0f cycles per call" % (pc[9], pc[10] / max(1, pc[9])))
