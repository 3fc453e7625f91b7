"""Where the C3 e2e step's time goes beyond the transport: the phantom upload,
the scatter call with a device image, and with a host image (D2H into a
fresh host buffer, as bench.py's e2e arm does)."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, configs

w = configs.c3()
ctx = X.Context(0)
proj = X.Projector(w.phantom, w.response, ctx=ctx)
ctx.comm_init(1, 0, X.Context.comm_unique_id())
g, spec, cfg = w.geometry, w.spectrum, w.config
dimg = torch.empty(g.nu * g.nv, dtype=torch.float64, device="cuda")
for rep in range(3):
    t0 = time.perf_counter()
    pk = A.Packed()
    A.check(A.lib().xs_upload_phantom(ctx.h, C.byref(pk.phantom(w.phantom))), ctx.h)
    t1 = time.perf_counter()
    proj.scatter_stats_mgpu(g, 0, spec, cfg, root=0, d_image_ptr=dimg.data_ptr(), host_image=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = proj.scatter_stats_mgpu(g, 0, spec, cfg, root=0, host_image=True)
    t3 = time.perf_counter()
    img = np.empty(g.nu * g.nv)
    img[:] = r.image.ravel()
    t4 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms | scatter, device image {1e3*(t2-t1):.1f} ms | "
          f"scatter, host image {1e3*(t3-t2):.1f} ms | copy out {1e3*(t4-t3):.1f} ms", flush=True)
