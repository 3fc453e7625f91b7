"""FDK timing at correction-loop scale: n views of nu x nv (device buffers) ->
dims^3 volume; REF on a few views (host cores, 1 worker) scaled by the
operation count."""
import ctypes as C
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, inputs as I, configs

n_views = int(sys.argv[1]) if len(sys.argv) > 1 else 720
nu = nv = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
n3 = int(sys.argv[3]) if len(sys.argv) > 3 else 512
g = I.make_circular_geometry(configs.SDD, configs.SOD, nu, nv, configs.pitch(nu), n_views)
ang = np.asarray(g.angles, dtype=np.float64)
dims = (n3, n3, n3)
voxel = X.default_voxel_size(g, dims)
dev = torch.device("cuda")
stack = torch.rand((n_views, nv, nu), device=dev, dtype=torch.float64)
vol = torch.empty((n3, n3, n3), device=dev, dtype=torch.float32)
ctx = X.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
pk = A.Packed()
gp = pk.geometry(g)
d = (C.c_int32 * 3)(*dims)


def run():
    ctx.check(A.lib().xs_fbp_reconstruct(ctx.h, stack.data_ptr(), A.dptr(ang), n_views, nu, nv, C.byref(gp), d,
                                         A.dptr(voxel), 1, vol.data_ptr(), 1))


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
macs = n_views * nv * nu * nu
print(f"GPU FDK {n_views} x {nu}x{nv} -> {n3}^3: {ms:.1f} ms (filter {macs:.2e} fp64 MACs, "
      f"backprojection {n_views * n3 ** 3:.2e} voxel-views)")
import oracle_lib
ref = oracle_lib.ref()
if ref is not None:
    # REF at reduced size: 8 views x (nu/4)^2 -> (n3/4)^3, scaled by both terms of the cost
    k, s = 8, 4
    gs = I.make_circular_geometry(configs.SDD, configs.SOD, nu // s, nv // s, configs.pitch(nu // s), n_views)
    small = np.random.default_rng(0).random((n_views, nv // s, nu // s))
    t = time.perf_counter()
    try:
        ref.fbp_reconstruct(small, np.asarray(gs.angles), gs, (n3 // s,) * 3, X.default_voxel_size(gs, (n3 // s,) * 3))
    except Exception as e:
        print("ref failed", e)
    cpu = time.perf_counter() - t
    est = cpu * (s ** 3)  # filter ~ views*nv*nu^2 (x s^3), backprojection ~ views*n3^3 (x s^3)
    print(f"REF FDK (1 worker) at 1/{s} linear size: {cpu:.2f} s -> ~{est:.0f} s at full size -> {est * 1e3 / ms:.0f}x")
