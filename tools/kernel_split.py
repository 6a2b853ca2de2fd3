"""Per-kernel device times of slc_compress (streaming kernel + deferred-chunk
fallback kernel) under torch.profiler, back to back as in a step:
python tools/kernel_split.py [layout] [special_period] [dtype] [cold]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import make_device_inputs  # noqa: E402
from paper_2603_08163_b200 import slc  # noqa: E402
from slcgen import layouts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama3.2-1b"
sp = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dtype = sys.argv[3] if len(sys.argv) > 3 else "f32"
cold = len(sys.argv) > 4 and sys.argv[4] == "cold"
layout = layouts.LAYOUTS[name]
plan = slc.Plan(layout, dtype=dtype)
th, tl, ef = make_device_inputs(plan, layout, 0, 0, dtype, special_period=sp, warm_ef=not cold)
ef0 = ef.clone()
rec = torch.zeros(plan.payload_bytes, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ef.copy_(ef0); flush.zero_(); plan.compress(th, tl, ef, rec)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
times = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        ef.copy_(ef0); flush.zero_()
        a.record(); plan.compress(th, tl, ef, rec); b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
d = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "compress" in e.name:
        d[e.name[:60]].append(e.device_time_total / 1e3)
print(f"{name} special {sp} {dtype}{' cold' if cold else ''}: event ms {sorted(times)[2]:.3f}")
for k, v in d.items():
    print(f"   {k}: median {sorted(v)[len(v) // 2]:.3f} ms")
