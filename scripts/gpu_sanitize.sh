#!/bin/bash
# compute-sanitizer over every libslc.so entry point at small sizes
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_paths.py ${QUICK:-} \
    > gpurun_out/san_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_$tool.log >> gpurun_out/san_summary.txt
done
