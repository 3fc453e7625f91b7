import sys; sys.path.insert(0, ".")
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
w = configs.c3()
proj = X.Projector(w.phantom, w.response)
for n in (1e7, 2e7, 5e7, 1e8):
    wc = configs.c3(photons=int(n), phantom=w.phantom)
    proj.scatter_stats(w.geometry, 0, w.spectrum, wc.config)
    ks = [proj.scatter_stats(w.geometry, 0, w.spectrum, wc.config).stats for _ in range(3)]
    k = min(s["kernel_ms"] for s in ks)
    print(f"photons {n:.0e}: {k:.1f} ms, {k / n * 1e8:.1f} ms per 1e8, waves {ks[0]['waves']}", flush=True)
