"""Summarise ncu artefacts into profiles/ (committed evidence).

  python tools/profile_summary.py launches <launches.csv> <out.txt>
      per-kernel launch count / mean device time and share of the step
  python tools/profile_summary.py full <prof.ncu-rep> <out.txt> [units_per_launch]
      per-kernel key metrics (time, DRAM bytes, throughput, issue, occupancy,
      top stall reasons) + per-source-line hot spots; also updates
      profiles/ncu_traffic.json with dram read+write bytes per launch
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = [f"# ncu launch list ({os.path.basename(path)}): gpu__time_duration.sum, --clock-control none",
             "# cold-cache serialised launches: compare SHARES, not absolute times",
             f"{'kernel':92s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:92s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__sass_inst_executed_op_local_ld.sum", "sm__cycles_elapsed.avg.per_second"]


def full(rep, out, units=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, unitrow = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {os.path.basename(rep)}"]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        lines.append(f"\n## {name}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:60s} {d[k]:>20s} {unitrow[h.index(k)]}")
        st = {k[33:]: float(d[k]) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and d[k] not in ("", "n/a")}
        tot = sum(st.values()) or 1
        lines.append("  top stall reasons (pc sampling):")
        for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]:
            lines.append(f"    {k:50s} {100 * v / tot:5.1f}%")
        rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        rd *= scale.get(unitrow[h.index("dram__bytes_read.sum")], 1)
        wr *= scale.get(unitrow[h.index("dram__bytes_write.sum")], 1)
        short = "compress" if "compress" in name else ("aggregate" if ("aggregate" in name or "agg_pipe" in name) else name)
        traffic[short] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "kernel": name,
                          "source": os.path.basename(rep)}
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    open("/tmp/_src.csv", "w").write(src)
    if units:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import io
        from contextlib import redirect_stdout

        import ncu_lines
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_lines.main("/tmp/_src.csv", float(units), 30)
        lines.append("\n## source hot spots (all kernels in the report; instr per unit = per chunk)")
        lines.extend("  " + l for l in buf.getvalue().splitlines())
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
