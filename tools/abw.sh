# A/B/n of paper_2201_13191_b200/lib_v*/ on the wavefront engine (C3)
cp paper_2201_13191_b200/lib/libxscatgpu.so /tmp/cur.so
for d in paper_2201_13191_b200/lib_v*; do
  cp $d/libxscatgpu.so paper_2201_13191_b200/lib/libxscatgpu.so
  timeout 120 python tools/wsweep.py ${N:-1e7} | sed "s/^/$(basename $d) /"
  XSCAT_SKIP=0 timeout 120 python tools/wsweep.py ${N:-1e7} | sed "s/^/$(basename $d) exact /"
done
cp /tmp/cur.so paper_2201_13191_b200/lib/libxscatgpu.so
