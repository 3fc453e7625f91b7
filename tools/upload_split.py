"""Where the C3 e2e step's phantom upload goes: the staged host upload
(xs_upload_phantom, what bench.py's e2e arm times), the device-side part
alone (xs_upload_phantom_device on arrays already in HBM), and a bare pinned
H2D of the same 671 MB."""
import ctypes as C
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, configs
w = configs.c3(photons=1000)
ctx = X.Context(0)
ctx.upload(w.phantom, w.response)


def t(f, n=3):
    out = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append(1e3 * (time.perf_counter() - t0))
    return " ".join(f"{x:.1f}" for x in out)


def staged():
    pk = A.Packed()
    ctx.check(A.lib().xs_upload_phantom(ctx.h, C.byref(pk.phantom(w.phantom))))


ids = torch.from_numpy(w.phantom.material_id).cuda()
dens = torch.from_numpy(w.phantom.density).cuda()


def device():
    pk = A.Packed()
    p = pk.phantom(w.phantom)
    p.material_id = C.cast(C.c_void_p(ids.data_ptr()), C.POINTER(C.c_uint8))
    p.density = C.cast(C.c_void_p(dens.data_ptr()), C.POINTER(C.c_float))
    ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))


hid = torch.from_numpy(w.phantom.material_id).pin_memory()
hde = torch.from_numpy(w.phantom.density).pin_memory()


def h2d():
    ids.copy_(hid, non_blocking=True)
    dens.copy_(hde, non_blocking=True)


print("staged upload ms:", t(staged), flush=True)
print("device-side upload ms:", t(device), flush=True)
print("bare pinned H2D ms:", t(h2d), flush=True)
