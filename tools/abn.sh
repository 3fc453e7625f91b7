# A/B/n: run the C3 sweep (macro + exact) with each paper_2201_13191_b200/lib_v*/libxscatgpu.so
cp paper_2201_13191_b200/lib/libxscatgpu.so /tmp/cur.so
for d in paper_2201_13191_b200/lib_v*; do
  v=$(basename $d)
  cp $d/libxscatgpu.so paper_2201_13191_b200/lib/libxscatgpu.so
  timeout 100 python tools/sweep.py ${N:-1e7} | sed "s/^/$v /"
  XSCAT_SKIP=0 timeout 100 python tools/sweep.py ${N:-1e7} | sed "s/^/$v exact /"
done
cp /tmp/cur.so paper_2201_13191_b200/lib/libxscatgpu.so
