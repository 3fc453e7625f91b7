"""One C3 scatter launch on the wavefront engine (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2_000_000
slots = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1 << 19
w = configs.c3(photons=n)
proj = X.Projector(w.phantom, w.response)
proj.ctx.set_option("engine", 1)
proj.ctx.set_option("wave_slots", slots)
r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
print(r.stats)
