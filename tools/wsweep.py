import sys
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
w = configs.c3(photons=n)
proj = X.Projector(w.phantom, w.response)
proj.ctx.set_option("engine", 1)
proj.scatter_stats(w.geometry, 0, w.spectrum, configs.c3(photons=500000, phantom=w.phantom).config)
r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
s = r.stats
print(f"n={n} kernel {s['kernel_ms']:.1f} ms hist/s {n/(s['kernel_ms']/1e3):.3e} lane-occ {s['walk_iterations']/max(1,s['walk_lane_slots']):.3f} "
      f"walk-blk/SM {s['blocks_per_sm']} waves {s['waves']}", flush=True)
print(f"  walk_iterations {s['walk_iterations']:.3e} uniform {s['uniform_iterations']:.3e} ({s['uniform_iterations']/max(1,s['walk_iterations']):.3f}) "
      f"REF visits {s['free_path_steps']+s['scoring_steps']:.3e}")
