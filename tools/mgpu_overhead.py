"""Host-observed time of the bench's step (xs_simulate_scatter_stats_mgpu,
one rank, device image) against its transport device time (kernel_ms), and
the same for the plain xs_simulate_scatter_stats."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs
w = configs.c3()
ctx = X.Context(0)
proj = X.Projector(w.phantom, w.response, ctx=ctx)
ctx.comm_init(1, 0, X.Context.comm_unique_id())
g, spec, cfg = w.geometry, w.spectrum, w.config
img = torch.empty(g.nu * g.nv, dtype=torch.float64, device="cuda")
for i in range(7):
    t = time.perf_counter()
    r = proj.scatter_stats_mgpu(g, 0, spec, cfg, root=0, d_image_ptr=img.data_ptr(), host_image=False)
    torch.cuda.synchronize()
    a = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter()
    q = proj.scatter_stats(g, 0, spec, cfg)
    b = 1e3 * (time.perf_counter() - t)
    print(f"mgpu {a:.1f} ms (kernel {r.stats['kernel_ms']:.1f}) | plain {b:.1f} ms (kernel {q.stats['kernel_ms']:.1f})", flush=True)
