"""Diagnostic: per-(super-)pixel z statistics of independent-seed scatter
images (GPU vs GPU, GPU vs oracle) at several binnings and photon counts.
usage: python tools/diag_stats.py c3 <gpu_photons> <cpu_photons>"""
import os
import sys
import pathlib

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import configs  # noqa: E402
import oracle_lib  # noqa: E402

name = sys.argv[1]
pg, pc = int(float(sys.argv[2])), int(float(sys.argv[3]))
make = getattr(configs, name)
w = make(photons=pg, seed=11)
proj = X.Projector(w.phantom, w.response)


def gpu(seed, p):
    c = make(photons=p, seed=seed, **({"phantom": w.phantom} if name == "c3" else {})).config
    c.track_variance = True
    return proj.scatter_stats(w.geometry, 0, w.spectrum, c)


def binz(a, va, b, vb, k):
    def bn(x):
        nv, nu = x.shape
        return x.reshape(nv // k, k, nu // k, k).sum(axis=(1, 3)).ravel()
    A, B, V = bn(a), bn(b), bn(va) + bn(vb)
    ok = V > 0
    z = (A - B)[ok] / np.sqrt(V[ok])
    return dict(k=k, n=int(z.size), f3=round(float(np.mean(np.abs(z) > 3)), 5),
                mz=round(float(np.mean(z)), 4), l2=round(float(np.sum((A - B) ** 2) / np.sum(V)), 4))


g1, g2 = gpu(101, pg), gpu(202, pg)
print("gpu/gpu totals", g1.total, g2.total, (g1.total - g2.total) / np.hypot(g1.total_std_error, g2.total_std_error))
for k in (1, 2, 4, 8, 16, 32):
    if w.geometry.nu % k == 0:
        print(" gpu/gpu", binz(g1.image, g1.variance, g2.image, g2.variance, k), flush=True)
orc = oracle_lib.oracle()
c = make(photons=pc, seed=303, **({"phantom": w.phantom} if name == "c3" else {}))
c.config.track_variance = True
cpu = orc.simulate_scatter_stats(c.phantom, c.geometry, 0, c.spectrum, c.response, c.config, os.cpu_count())
g3 = gpu(404, pc)
print("gpu/cpu totals", g3.total, cpu["total"], (g3.total - cpu["total"]) / np.hypot(g3.total_std_error, cpu["total_std_error"]))
for k in (1, 2, 4, 8, 16, 32):
    if w.geometry.nu % k == 0:
        print(" gpu/cpu", binz(g3.image, g3.variance, cpu["image"], cpu["variance"], k), flush=True)
