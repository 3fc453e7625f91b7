"""Speckled-phantom stress matrix (the regime where the first wavefront event
kernel hung): flip fractions x seeds x walk modes x 1 / 2
pipelines, variance tracking on; every wavefront run must finish and equal the
megakernel bit for bit.  Prints one line per case and "ALL OK" at the end.
usage: python tools/stress_cases.py [n_seeds] [photons]"""
import sys
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import inputs as I  # noqa: E402
from cases import poly  # noqa: E402

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
photons = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
ph, g, angle, spec, resp, cfg = poly()
if photons:
    cfg.photons_total = photons
ctx = X.Context(0)
bad = 0
for frac in (0.1, 0.3, 0.5):
    for seed in range(9, 9 + n_seeds):
        rng = np.random.default_rng(seed)
        sp = I.VoxelPhantom(ph.dims, ph.voxel_size, ph.origin, ph.material_id.copy(), ph.density.copy(),
                            ph.materials)
        flip = (rng.uniform(size=ph.material_id.size) < frac) & (ph.material_id > 0)
        sp.material_id[flip] = 2
        sp.density[flip] = 7.874
        for mode in (0, 1):
            ctx.set_option("walk_mode", mode)
            ctx.set_option("engine", 0)
            proj = X.Projector(sp, resp, ctx=ctx)
            ref = proj.scatter_stats(g, angle, spec, cfg)
            ctx.set_option("engine", 1)
            for pipes in (1, 2):
                ctx.set_option("wave_pipes", pipes)
                r = proj.scatter_stats(g, angle, spec, cfg)
                ok = (np.array_equal(r.image, ref.image) and np.array_equal(r.variance, ref.variance)
                      and r.total == ref.total and r.ledger == ref.ledger)
                bad += not ok
                print(f"frac {frac} seed {seed} walk_mode {mode} pipes {pipes}: "
                      f"{'ok' if ok else 'MISMATCH'} total {r.total:.9g}", flush=True)
print("ALL OK" if bad == 0 else f"{bad} MISMATCHES", flush=True)
