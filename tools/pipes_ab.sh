#!/bin/bash
# bench with 1..4 concurrent wavefront pipelines
for p in ${PIPES:-1 2 3 1 2 3}; do
  XSCAT_WAVE_PIPES=$p python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-ktime 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('pipes $p', round(d['value']/1e6,2), 'Mhist/s', round(d['ms_per_step'],1), 'ms')"
done
