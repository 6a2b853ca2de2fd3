"""Per-source-line instruction counts and stall samples from an ncu report
(--import-source on, -lineinfo): python tools/ncu_source_lines.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
lines = []
cur = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 1:
        if r and r[0] == "File Path":
            fname = r[1]
        continue
    if r[0]:  # a source line row (aggregated)
        try:
            cur = {"line": int(r[0]), "src": r[1][:90], "samples": int(r[4] or 0), "inst": int(r[7] or 0),
                   "file": fname.split("/")[-1]}
        except ValueError:
            continue
        lines.append(cur)
tot_s = sum(l["samples"] for l in lines) or 1
tot_i = sum(l["inst"] for l in lines) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for l in sorted(lines, key=lambda l: -l["samples"])[:top]:
    print(f"{l['file'][:18]:18s}:{l['line']:4d} samp {100*l['samples']/tot_s:5.1f}% inst {100*l['inst']/tot_i:5.1f}%  {l['src']}")
