"""Build libslc variants with different -D tuning macros into build/variants/
(for one-call GPU sweeps: SLC_LIB=<path> python bench.py ...)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402


def build(name, defines):
    out_dir = os.path.join(ROOT, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libslc_{name}.so")
    csrc = os.path.join(ge.PKG, "csrc")
    cmd = [ge.NVCC, *ge.ARCH, *ge.NVFLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", out, *[os.path.join(csrc, s) for s in ge.SLC_SOURCES]]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition("=")
        print(build(name, [d for d in defs.split(",") if d]))
