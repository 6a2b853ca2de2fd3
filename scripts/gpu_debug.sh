mkdir -p gpurun_out
for v in dbgb; do
for l in m1; do
  SLC_LIB=build/variants/libslc_$v.so SLC_DEBUG=1 timeout 300 python tools/dbg_compress.py $l 1 > gpurun_out/dbg_${v}_$l.log 2>&1; echo "$v $l rc=$? $(grep -E "OK|libslc|SLC_CHECK" gpurun_out/dbg_${v}_$l.log | head -3 | tr '\n' ' ')"
done
done
