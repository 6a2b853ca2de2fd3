#!/bin/bash
# per-kernel durations of compress (main + fallback), warm caches (--cache-control none)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for sp in ${SPS:-0 32 8}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:compress --csv --log-file gpurun_out/fb_$sp.csv \
    python bench.py --steps 3 --warmup 3 --special-period $sp --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "special $sp"; python - <<PY
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/fb_$sp.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
d=collections.defaultdict(list)
for r in rows[1:]:
    v=float(r[vi].replace(",","")); v = v/1e3 if r[ui].startswith("n") else v
    d[r[ki][:40]].append(v)
for k,v in d.items(): print("  ", k, len(v), "median us %.1f" % sorted(v)[len(v)//2])
PY
done
