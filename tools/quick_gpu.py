"""Quick device timing of the configs at reduced photon counts (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs

for name, fn, n in [("C1", configs.c1, 1_000_000), ("C2", configs.c2, 2_000_000), ("C3", configs.c3, 2_000_000)]:
    t = time.time(); w = fn(photons=n); tb = time.time() - t
    t = time.time(); proj = X.Projector(w.phantom, w.response); tu = time.time() - t
    r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)  # warm
    t = time.time(); r = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config); ts = time.time() - t
    s = r.stats
    steps = s['free_path_steps'] + s['scoring_steps']
    t = time.time(); p = proj.primary(w.geometry, 0, w.spectrum, w.config); tp = time.time() - t
    print(f"{name}: build {tb:.2f}s upload {tu:.3f}s fmt={s['voxel_format']} pal={s['palette_size']} "
          f"scatter {ts:.3f}s kernel {s['kernel_ms']:.1f}ms hist/s={r.histories/(s['kernel_ms']/1e3):.3e} "
          f"steps/hist={steps/r.histories:.1f} (fp {s['free_path_steps']/r.histories:.1f}) rays/hist={s['scoring_rays']/r.histories:.2f} "
          f"Gsteps/s={steps/(s["kernel_ms"]/1e3)/1e9:.1f} iters/hist={s["walk_iterations"]/r.histories:.1f} total={r.total:.6g}±{r.total_std_error:.2g} primary {tp*1e3:.1f}ms", flush=True)
