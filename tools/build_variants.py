"""Build libslc variants with different -D tuning macros into build/variants/
(for one-call GPU sweeps: SLC_LIB=<path> python bench.py ...)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402


def build(name, defines):
    """defines: -D macros; an entry "@<git rev>" builds that revision's csrc/ instead."""
    out_dir = os.path.join(ROOT, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libslc_{name}.so")
    csrc = os.path.join(ge.PKG, "csrc")
    revs = [d[1:] for d in defines if d.startswith("@")]
    defines = [d for d in defines if not d.startswith("@")]
    if revs:
        tmp = os.path.join(out_dir, f"src_{name}")
        os.makedirs(tmp, exist_ok=True)
        rel = os.path.relpath(csrc, ROOT)
        subprocess.check_call(f"git -C {ROOT} archive {revs[0]} {rel} include | tar -x -C {tmp}", shell=True)
        csrc = os.path.join(tmp, rel)
    srcs = list(ge.SLC_SOURCES)
    if any(d.startswith("SLC_USE_TMA") for d in defines):
        srcs += ge.SLC_TMA_SOURCES
    if revs:
        srcs = sorted(f for f in os.listdir(csrc) if f.endswith((".cu", ".cpp")))
    cmd = [ge.NVCC, *ge.ARCH, *ge.NVFLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", out, *[os.path.join(csrc, s) for s in srcs]]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition("=")
        print(build(name, [d for d in defs.split(",") if d]))
