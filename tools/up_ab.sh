#!/bin/bash
# staged phantom upload, product lib against an A/B build (tools/ab.sh upold "" on the old revision)
for rep in 1 2 3; do for lib in product upold; do
 if [ $lib = product ]; then unset XSCAT_LIB; else export XSCAT_LIB=build_ab/$lib/libxscatgpu.so; fi
 echo "== $lib"; python tools/upload_split.py 2>&1 | grep ms:
done; done
