"""Run-to-run variance of the C3 projection: device time of 8 consecutive
projections in one process (transport kernel_ms from the launch stats)."""
import sys
sys.path.insert(0, ".")
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
w = configs.c3()
proj = X.Projector(w.phantom, w.response)
out = []
for i in range(9):
    s = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config).stats
    out.append(round(s["kernel_ms"], 1))
print("kernel_ms per projection:", out[1:], flush=True)
