#!/bin/bash
# per-kernel device time (XSCAT_KTIME, one pipeline) of the product lib and A/B builds, twice each
for rep in 1 2; do for lib in product "$@"; do
 if [ $lib = product ]; then unset XSCAT_LIB; else export XSCAT_LIB=build_ab/$lib/libxscatgpu.so; fi
 XSCAT_KTIME=1 XSCAT_WAVE_PIPES=1 python tools/ktime.py 1e8 1
done; done
