"""Diagnostic: find single histories whose scatter tallies differ between the
device and the oracle (same seed), by bisection over history ranges.

usage: python tools/diag_replay.py [c1|c2|c3] [photons] [walk_mode] [n_probe]
"""
import sys
import pathlib

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import _capi as A  # noqa: E402
from paper_2201_13191_b200 import configs  # noqa: E402
import oracle_lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
photons = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
walk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n_probe = int(sys.argv[4]) if len(sys.argv) > 4 else 4000

w = getattr(configs, name)(photons=photons)
g, spec, cfg = w.geometry, w.spectrum, w.config
orc = oracle_lib.oracle()
ctx = X.projector.Context(0)
ctx.set_option("walk_mode", walk)
proj = X.Projector(w.phantom, w.response, ctx=ctx)
L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
n = X.history_count(spec, cfg.photons_total)
counts = orc.apportion(spec, cfg.photons_total)
starts = np.concatenate([[0], np.cumsum(counts)])


def gpu_img(h0, h1):
    acc = torch.zeros(L["words"], dtype=torch.int64, device="cuda")
    proj.accumulate(g, 0, spec, cfg, h0, h1, acc.data_ptr())
    a = acc.cpu().numpy().view(np.uint64)
    return a


def cpu_img(h0, h1):
    a = np.zeros(L["words"], np.uint64)
    orc.accumulate_range(w.phantom, g, 0, spec, w.response, cfg, h0, h1, a)
    return a


def image_of(acc, h0, h1):
    return X.projector.finalize_host(g, spec, cfg, acc, h0, h1).image.ravel()


def differs(h0, h1, tol=1e-9):
    a, b = gpu_img(h0, h1), cpu_img(h0, h1)
    ia, ib = image_of(a, h0, h1), image_of(b, h0, h1)
    nzb = ib > 0
    bad = (np.abs(ia - ib) > tol * np.maximum(np.abs(ib), 1e-300))
    return int(bad.sum()), ia, ib


def bisect(h0, h1):
    while h1 - h0 > 1:
        m = (h0 + h1) // 2
        if differs(h0, m)[0]:
            h1 = m
        else:
            h0 = m
    return h0


rng = np.random.default_rng(1)
found = 0
for trial in range(12):
    h0 = int(rng.integers(0, n - n_probe))
    nb, ia, ib = differs(h0, h0 + n_probe)
    print(f"range [{h0}, {h0 + n_probe}): {nb} pixels differ", flush=True)
    if nb and found < 3:
        h = bisect(h0, h0 + n_probe)
        nb, ia, ib = differs(h, h + 1)
        bin_ = int(np.searchsorted(starts, h, side="right") - 1)
        print(f"  history {h} (bin {bin_}, E {spec.energy_kev[bin_]} keV, photon {h - starts[bin_]}): "
              f"{nb} pixels differ")
        pa, pb = np.nonzero(ia)[0], np.nonzero(ib)[0]
        print("   gpu pixels:", list(pa[:40]), "sum", ia.sum())
        print("   cpu pixels:", list(pb[:40]), "sum", ib.sum())
        common = np.intersect1d(pa, pb)
        for p in common[:10]:
            print(f"     pix {p}: gpu {ia[p]!r} cpu {ib[p]!r} rel {(ia[p] - ib[p]) / ib[p]:.3e}")
        found += 1
