"""Speckled-phantom transport check: walk_mode x engine (argv)."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I
from cases import poly
mode, engine, frac = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 9
ph, g, angle, spec, resp, cfg = poly()
import os
if os.environ.get('NOVAR'):
    cfg.track_variance = False
if os.environ.get('SPLIT'):
    cfg.splitting = int(os.environ['SPLIT'])
rng = np.random.default_rng(seed)
sp = I.VoxelPhantom(ph.dims, ph.voxel_size, ph.origin, ph.material_id.copy(), ph.density.copy(), ph.materials)
flip = (rng.uniform(size=ph.material_id.size) < frac) & (ph.material_id > 0)
sp.material_id[flip] = 2
sp.density[flip] = 7.874
ctx = X.Context(0)
ctx.set_option("walk_mode", mode)
ctx.set_option("engine", engine)
proj = X.Projector(sp, resp, ctx=ctx)
r = proj.scatter_stats(g, angle, spec, cfg)
print(f"mode {mode} engine {engine} frac {frac} seed {seed}: block_walk {ctx.launch_stats()['block_walk']} total {r.total}", flush=True)
