#!/bin/bash
# bench each A/B build (and the product lib) on the same box: tools/ab_bench.sh name1 name2 ...
for n in product "$@"; do
  if [ "$n" = product ]; then unset XSCAT_LIB; else export XSCAT_LIB=build_ab/$n/libxscatgpu.so; fi
  python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$n', round(d['value']/1e6,2), 'Mhist/s', round(d['ms_per_step'],1), 'ms', 'walk', round(d['roofline']['walk_ms'],1))"
done
