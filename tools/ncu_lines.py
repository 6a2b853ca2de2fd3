"""Summarise an ncu source page (--print-source cuda,sass) per CUDA source line:
instructions executed per unit and stall-sample share.  Usage:
  ncu -i rep --page source --csv -k regex:K --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv UNITS [TOP]"""
import csv
import sys


def main(path, units, top=40):
    rows = list(csv.reader(open(path)))
    out = []
    fname = None
    hdr = None
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0] != "":
            d = dict(zip(hdr[2:], r[2:]))
            cur = [fname, r[0], r[1][:90], 0.0, 0.0]
            out.append(cur)
            try:
                cur[3] = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
                cur[4] = float(d.get("Instructions Executed", 0) or 0)
            except ValueError:
                pass
    tot_s = sum(o[3] for o in out) or 1
    tot_i = sum(o[4] for o in out)
    print(f"total instr/unit {tot_i / units:.1f}")
    for o in sorted(out, key=lambda o: -(o[3] / tot_s + o[4] / max(tot_i, 1)))[:top]:
        print(f"{o[0][:14]:14s}:{o[1]:>4s} stall {100 * o[3] / tot_s:5.1f}%  instr/unit {o[4] / units:8.1f}  {o[2]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
