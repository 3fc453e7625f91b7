"""Megakernel vs wavefront engine: bit-identity of the outputs and timing."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs

def run(w, engine, exact=False, slots=None, warm=True):
    proj = X.Projector(w.phantom, w.response)
    proj.ctx.set_option("engine", engine)
    proj.ctx.set_option("exact_walk", 1 if exact else 0)
    if slots:
        proj.ctx.set_option("wave_slots", slots)
    if warm:
        proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
    return proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)

for name, n in [("c1", 200000), ("c2", 1000000)]:
    w = getattr(configs, name)(photons=n)
    for exact in (False, True):
        a = run(w, 0, exact)
        b = run(w, 1, exact)
        same = np.array_equal(a.image, b.image) and a.total == b.total
        print(f"{name} n={n} exact={exact}: bit-identical={same} total {a.total:.12g} {b.total:.12g} "
              f"mk {a.stats['kernel_ms']:.1f} ms  wf {b.stats['kernel_ms']:.1f} ms waves {b.stats['waves']}", flush=True)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
w = configs.c3(photons=n)
a = run(w, 0)
print(f"c3 megakernel: {a.stats['kernel_ms']:.0f} ms  {n / a.stats['kernel_ms'] * 1e3:.3e} hist/s", flush=True)
for slots in (1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20):
    b = run(w, 1, slots=slots)
    s = b.stats
    occ = s['walk_iterations'] / max(s['walk_lane_slots'], 1)
    print(f"c3 wavefront slots={slots}: {s['kernel_ms']:.0f} ms  {n / s['kernel_ms'] * 1e3:.3e} hist/s  waves {s['waves']} "
          f"lane-occ {occ:.3f} walk-blocks/SM {s['blocks_per_sm']} identical={np.array_equal(a.image, b.image)}", flush=True)
