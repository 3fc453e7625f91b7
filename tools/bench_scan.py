"""C4-style scan timing: run_scan over n angles of the C3 panel, 1e7 photons each
(scatter only), against the per-angle transport time."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
n_ang = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = configs.c4(photons=10_000_000)
proj = X.Projector(w.phantom, w.response)
proj.run_scan(w.geometry, w.spectrum, w.config, [0], what=X.SCATTER)  # warm
t = time.perf_counter()
r = proj.run_scan(w.geometry, w.spectrum, w.config, list(range(n_ang)), what=X.SCATTER)
wall = time.perf_counter() - t
k = proj.ctx.launch_stats()["kernel_ms"]
print(f"run_scan {n_ang} angles x 1e7: {wall:.3f} s wall ({wall / n_ang * 1e3:.1f} ms/angle); "
      f"last angle transport {k:.1f} ms; {n_ang * 1e7 / wall:.3e} hist/s")
