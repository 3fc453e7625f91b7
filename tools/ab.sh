# A/B: lib (current) vs lib_alt
for v in lib lib_alt; do
  if [ $v = lib_alt ]; then cp paper_2201_13191_b200/lib/libxscatgpu.so /tmp/cur.so; cp paper_2201_13191_b200/lib_alt/libxscatgpu.so paper_2201_13191_b200/lib/libxscatgpu.so; fi
  timeout 100 python tools/sweep.py 1e7 | sed "s/^/$v /"; XSCAT_SKIP=0 timeout 100 python tools/sweep.py 1e7 | sed "s/^/$v exact /"
  if [ $v = lib_alt ]; then cp /tmp/cur.so paper_2201_13191_b200/lib/libxscatgpu.so; fi
done
