"""Per-kernel device times over a whole bench.py run under torch.profiler
(median per kernel name): python tools/bench_kernels.py <bench args>"""
import collections
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

sys.argv = ["bench.py"] + sys.argv[1:]
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    try:
        runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
    except SystemExit:
        pass
d = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        d[e.name[:70]].append(e.device_time_total / 1e3)
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    if sum(v) > 0.5:
        print(f"   {len(v):4d} x median {sorted(v)[len(v) // 2]:.3f} ms  max {max(v):.3f}  {k}", file=sys.stderr)
        if os.environ.get("SEQ") and os.environ["SEQ"] in k:
            print("      in order: " + " ".join(f"{x:.3f}" for x in v), file=sys.stderr)
