# space sharing: walk blocks per SM x concurrent pipelines (bench ms per projection)
for rep in 1 2; do
for v in "6 2" "3 2" "4 2" "2 3" "3 3"; do set -- $v
  XSCAT_WALK_BPS=$1 XSCAT_WAVE_PIPES=$2 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --no-ktime 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bps $1 pipes $2', round(d['value']/1e6,2), 'Mhist/s', round(d['ms_per_step'],1), 'ms')"
done; done
