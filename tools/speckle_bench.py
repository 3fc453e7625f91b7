"""Speckled-phantom transport (the C5 iterations-2+ regime): the C3 phantom
with 15% of the air voxels flipped to aluminium and 2% of the body to air,
one 512^2 MC-grid projection at 1e7 photons; walk mode from the upload probe
(argv[1] forces 0/1)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs, inputs as I
w = configs.c3()
ph = w.phantom
rng = np.random.default_rng(5)
ids, dens = ph.material_id.copy(), ph.density.copy()
air = ids == 0
f1 = air & (rng.uniform(size=ids.size) < 0.15)
f2 = (~air) & (rng.uniform(size=ids.size) < 0.02)
ids[f1], dens[f1] = 1, np.float32(2.699)
ids[f2], dens[f2] = 0, np.float32(0.0)
sp = I.VoxelPhantom(ph.dims, ph.voxel_size, ph.origin, ids, dens, ph.materials)
g = I.make_circular_geometry(configs.SDD, configs.SOD, 512, 512, configs.pitch(512), 1)
cfg = I.SimConfig(photons_total=10_000_000, splitting=10, seed=configs.SEED)
ctx = X.Context(0)
if len(sys.argv) > 1:
    ctx.set_option("walk_mode", int(sys.argv[1]))
proj = X.Projector(sp, w.response, ctx=ctx)
proj.scatter_stats(g, 0, w.spectrum, cfg)
for _ in range(2):
    r = proj.scatter_stats(g, 0, w.spectrum, cfg)
    s = ctx.launch_stats()
    print(f"mode {sys.argv[1] if len(sys.argv) > 1 else 'auto'}: block_walk {s['block_walk']} kernel {s['kernel_ms']:.1f} ms "
          f"walk {s['walk_ms']:.1f} ms ({1e7 / s['kernel_ms'] * 1e3:.3e} hist/s), walk iters/hist "
          f"{s['walk_iterations'] / s['histories']:.0f}, visits/hist {(s['free_path_steps'] + s['scoring_steps']) / s['histories']:.0f}, total {r.total:.6g}")
