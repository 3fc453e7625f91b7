"""C4-style scan (C3 phantom and panel, 1e7 histories per angle) with several
angles per wavefront run: seconds per angle for scan_jobs x wave_pipes.
usage: [XSCAT_WAVE_SLOTS=n] python tools/scan_jobs_probe.py [n_angles] [JOBSxPIPES ...]"""
import sys
import time
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 90
w = configs.c4()
ctx = X.Context(0)
proj = X.Projector(w.phantom, w.response, ctx=ctx)
sub = list(range(n))
out = np.empty((n, w.geometry.nv, w.geometry.nu))
ref = None
CASES = [(int(a), int(b)) for a, b in (c.split('x') for c in sys.argv[2:])] or \
    [(1, 2), (8, 2), (16, 2), (1, 3), (8, 3), (16, 3), (24, 3), (16, 4)]
for jobs, pipes in CASES:
    ctx.set_option("scan_jobs", jobs)
    ctx.set_option("wave_pipes", pipes)
    proj.run_scan(w.geometry, w.spectrum, w.config, sub, X.SCATTER)  # warm: buffers at full size
    t = time.perf_counter()
    r = proj.run_scan(w.geometry, w.spectrum, w.config, sub, X.SCATTER)
    dt = time.perf_counter() - t
    img = r.scatter.images
    same = ref is None or np.array_equal(img, ref)
    if ref is None:
        ref = img.copy()
    print(f"scan_jobs {jobs:2d} pipes {pipes}: {1e3 * dt / n:.2f} ms/angle, identical {same}", flush=True)
