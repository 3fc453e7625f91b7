# bit-identity + speed of lib_v* builds on C3
cp paper_2201_13191_b200/lib/libxscatgpu.so /tmp/cur.so
for d in paper_2201_13191_b200/lib_v*; do
  cp $d/libxscatgpu.so paper_2201_13191_b200/lib/libxscatgpu.so
  timeout 200 python tools/imghash.py ${N:-2e6} | sed "s/^/$(basename $d) /"
  timeout 120 python tools/wsweep.py ${NS:-1e7} | head -1 | sed "s/^/$(basename $d) /"
done
cp /tmp/cur.so paper_2201_13191_b200/lib/libxscatgpu.so
