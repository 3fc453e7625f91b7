# run-field A/B (XSCAT_RUNS=0/1) on the C3 projection: per-kernel device time
for rep in 1 2; do for r in 0 1; do
 XSCAT_RUNS=$r XSCAT_KTIME=1 XSCAT_WAVE_PIPES=1 python tools/ktime.py 1e8 1 2>&1 | sed "s/^/runs=$r /"
done; done
