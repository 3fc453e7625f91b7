import sys, time, os
sys.path.insert(0,'.')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
w = configs.c3(photons=10_000_000)
proj = X.Projector(w.phantom, w.response)
for _ in range(2): proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
t=time.perf_counter(); n=5
for _ in range(n): r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
dt=(time.perf_counter()-t)/n
s=r.stats
print(os.environ.get('XSCAT_LIB','product'), f"call {dt*1e3:.1f} ms kernel {s['kernel_ms']:.1f} waves {s['waves']} launches {s['launches']}")
g = X.inputs.make_circular_geometry(configs.SDD, configs.SOD, 2048, 2048, configs.pitch(2048), 360)
t = time.perf_counter()
sc = proj.run_scan(g, w.spectrum, w.config, list(range(24)), X.SCATTER)
print(f"run_scan 24 angles: {(time.perf_counter() - t) / 24 * 1e3:.1f} ms/angle")
