"""Per-angle cost of run_scan on the C4 scene: fresh (untouched) host outputs
as Projector.run_scan allocates them, against caller-owned pre-touched ones."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, configs

w = configs.c4()
proj = X.Projector(w.phantom, w.response)
g, spec, cfg = w.geometry, w.spectrum, w.config
proj.run_scan(g, spec, cfg, list(range(4)), X.SCATTER)
sub = np.arange(10, 30, dtype=np.int32)
for rep in range(2):
    t = time.perf_counter()
    proj.run_scan(g, spec, cfg, list(sub), X.SCATTER)
    a = (time.perf_counter() - t) / sub.size
    out = np.ones((sub.size, g.nv, g.nu))  # touched
    secs = np.zeros(sub.size)
    pk = A.Packed()
    t = time.perf_counter()
    proj.ctx.check(A.lib().xs_run_scan(proj.ctx.h, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
                                       C.byref(pk.config(cfg)), sub.ctypes.data_as(C.POINTER(C.c_int32)),
                                       int(sub.size), X.SCATTER, None, A.dptr(out), A.dptr(secs)))
    b = (time.perf_counter() - t) / sub.size
    print(f"fresh outputs {1e3*a:.1f} ms/angle | touched outputs {1e3*b:.1f} ms/angle", flush=True)
