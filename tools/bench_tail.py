"""C5-scale timing of the fused correction tail:
720 views at 2048^2, MC grid 512^2, scatter on every 2nd angle.  Device
buffers (torch); the REF CPU composition (oracle/_ref) on 8 views, scaled."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A

n_full = int(sys.argv[1]) if len(sys.argv) > 1 else 720
nu = nv = 512
nu_out = nv_out = 2048
full = np.linspace(0.0, 2 * np.pi, n_full, endpoint=False)
sub = full[::2]
sg = X.default_sg_spec(nu, nv)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
scat = (0.2 + 0.05 * torch.rand((sub.size, nv, nu), device=dev, dtype=torch.float64, generator=g)).contiguous()
prim = (0.5 + 0.5 * torch.rand((n_full, nv, nu), device=dev, dtype=torch.float64, generator=g)).contiguous()
a = (2.0 * torch.rand((n_full, nv_out, nu_out), device=dev, dtype=torch.float64, generator=g)).contiguous()
out = torch.empty_like(a)
ctx = X.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
frac, cl = C.c_double(0.0), C.c_uint64(0)
sa, fa = np.ascontiguousarray(sub), np.ascontiguousarray(full)


def run():
    ctx.check(A.lib().xs_correction_tail(ctx.h, scat.data_ptr(), A.dptr(sa), sub.size, prim.data_ptr(),
                                         A.dptr(fa), n_full, nu, nv, sg.window, sg.polyorder, a.data_ptr(),
                                         nu_out, nv_out, out.data_ptr(), C.byref(frac), C.byref(cl), 1))


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    run()
e1.record()
torch.cuda.synchronize()
gpu_ms = e0.elapsed_time(e1) / 3
alg = n_full * nv_out * nu_out * 16  # a read + corrected write (8 B each per full-resolution pixel)
print(f"GPU fused tail: {n_full} views {nu}^2 -> {nu_out}^2: {gpu_ms:.1f} ms "
      f"({alg / gpu_ms / 1e6:.0f} GB/s of algorithmic bytes; fp64 log/div bound); "
      f"mean scatter fraction {frac.value:.6f}")
import oracle_lib
ref = oracle_lib.ref()
if ref is not None:
    k = 8
    s8 = scat[: k // 2].cpu().numpy()
    p8 = prim[:k].cpu().numpy()
    a8 = a[:k].cpu().numpy()
    t = time.perf_counter()
    ref.correction_tail(s8, full[:k:2], p8, full[:k], sg.window, sg.polyorder, a8)
    cpu_s = (time.perf_counter() - t) * n_full / k
    print(f"REF CPU composition (1 thread, {k} views scaled to {n_full}): {cpu_s:.1f} s -> {cpu_s * 1e3 / gpu_ms:.0f}x")
