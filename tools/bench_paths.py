"""Selection-path counts of the compress kernels over a whole bench.py run
(SLC_LIB must be a SLC_PHASE_TIMING build): python tools/bench_paths.py <bench args>"""
import ctypes
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_08163_b200 import slc  # noqa: E402

lib = ctypes.CDLL(slc.LIB_PATH)
z = (ctypes.c_ulonglong * 8)()
lib.slc_debug_phase_cycles_ws(z, 1)
sys.argv = ["bench.py"] + sys.argv[1:]
try:
    runpy.run_path(os.path.join(ROOT, "bench.py"), run_name="__main__")
except SystemExit:
    pass
pc = (ctypes.c_ulonglong * 16)()
lib.slc_debug_path_count_ws(pc)
print("paths over the run: candidates %d, tie %d, tie->rank %d, radix %d, key_select %d, hist->key %d" %
      (pc[0], pc[1], pc[2], pc[3], pc[9], pc[11]), file=sys.stderr)
nt = max(1, pc[1] + pc[2] + pc[3]); nr = max(1, pc[3])
print("  cycles per call: tie_select %.0f, radix rounds %.0f, radix mark+fill %.0f, key_select %.0f; "
      "radix chunks: mean G %.1f, mean M %.1f" % (pc[4] / nt, pc[5] / nr, pc[6] / nr, pc[10] / max(1, pc[9]),
                                                   pc[7] / nr, pc[8] / nr), file=sys.stderr)
