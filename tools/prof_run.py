"""One warm + one measured scatter launch of a config (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 200000
w = getattr(configs, name)(photons=n)
proj = X.Projector(w.phantom, w.response)
for _ in range(2):
    r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
print(name, n, r.stats)
