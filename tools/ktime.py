"""Per-kernel device time of one C3 projection (XSCAT_KTIME=1, one pipeline).
usage: XSCAT_KTIME=1 XSCAT_WAVE_PIPES=1 python tools/ktime.py [photons] [reps]"""
import os
import sys
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("XSCAT_KTIME", "1")
import paper_2201_13191_b200 as X  # noqa: E402
from paper_2201_13191_b200 import configs  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = configs.c3(photons=n)
proj = X.Projector(w.phantom, w.response)
proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
for _ in range(reps):
    s = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config).stats
    ks = ("setup_ms", "walk_ms", "score_ms", "event_ms", "admit_ms")
    tot = sum(s[k] for k in ks)
    print(f"lib={os.environ.get('XSCAT_LIB', 'product')} pipes={os.environ.get('XSCAT_WAVE_PIPES', '2')} "
          f"transport {s['kernel_ms']:.1f} ms | " + " ".join(f"{k[:-3]} {s[k]:.1f} ({100 * s[k] / tot:.0f}%)" for k in ks)
          + f" | iters/hist {s['walk_iterations'] / s['histories']:.1f} uniform {s['uniform_iterations'] / max(1, s['walk_iterations']):.2f}"
          f" lanes {s['walk_iterations'] / max(1, s['walk_lane_slots']):.2f} visits/hist "
          f"{(s['free_path_steps'] + s['scoring_steps']) / s['histories']:.0f} rays/hist {s['scoring_rays'] / s['histories']:.2f}",
          flush=True)
