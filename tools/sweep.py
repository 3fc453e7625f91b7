import os, sys, time
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
w = configs.c3(photons=n)
proj = X.Projector(w.phantom, w.response)
r = proj.scatter_stats(w.geometry, 0, w.spectrum, configs.c3(photons=200000, phantom=w.phantom).config)
r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
s = r.stats
st = s['free_path_steps'] + s['scoring_steps']
occ = s['walk_iterations'] / s['walk_lane_slots'] if s.get('walk_lane_slots') else float('nan')
print(f"n={n} kernel {s['kernel_ms']:.0f} ms  hist/s {n/(s['kernel_ms']/1e3):.3e}  Gsteps/s {st/(s['kernel_ms']/1e3)/1e9:.1f}  lane-occ {occ:.3f} blk/sm {s.get("blocks_per_sm")} smem {s.get("smem_per_block")} H {s.get("slots_per_warp")}", flush=True)
