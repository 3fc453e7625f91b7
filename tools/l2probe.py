"""C3 transport throughput vs detector resolution (same physical panel):
probes how much the image accumulator's L2 footprint costs."""
import sys
sys.path.insert(0, '.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs, inputs as I
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
ph = configs.c3_phantom()
w = configs.c3(photons=n, phantom=ph)
proj = X.Projector(ph, w.response)
for res in (2048, 1024, 512, 256):
    g = I.make_circular_geometry(configs.SDD, configs.SOD, res, res, configs.pitch(res), 1)
    proj.scatter_stats(g, 0, w.spectrum, configs.c3(photons=200000, phantom=ph).config)
    r = proj.scatter_stats(g, 0, w.spectrum, w.config)
    s = r.stats
    print(f"detector {res}^2: kernel {s['kernel_ms']:.0f} ms  hist/s {n / (s['kernel_ms'] / 1e3):.3e}", flush=True)
