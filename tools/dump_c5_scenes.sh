#!/bin/bash
# C5 loop, 2 iterations, with the segmented scenes dumped and compressed into gpurun_out/
mkdir -p /tmp/scenes
XSCAT_DUMP_SCENE=/tmp/scenes python tools/bench_loop.py ${1:-3} > gpurun_out/c5_dump.log 2>&1
python - <<'PY'
import numpy as np, glob
for f in sorted(glob.glob('/tmp/scenes/scene_*.u8')):
    a = np.fromfile(f, np.uint8)
    np.savez_compressed('gpurun_out/' + f.split('/')[-1].replace('.u8', '.npz'), ids=a)
    print(f, a.size, np.bincount(a, minlength=3))
PY
