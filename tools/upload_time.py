"""Phantom upload paths for the C3 grid (512^3): host encode + H2D of the
encoded grid (xs_upload_phantom) vs H2D of the raw arrays + device
validation / encode (xs_upload_phantom_device)."""
import ctypes as C
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A, configs
w = configs.c3(photons=1000)
ctx = X.Context(0)
for i in range(3):
    t = time.perf_counter()
    ctx.upload(w.phantom, w.response)
    print(f"host-encode upload {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
ids = torch.empty(w.phantom.material_id.size, dtype=torch.uint8, device="cuda")
dens = torch.empty(w.phantom.density.size, dtype=torch.float32, device="cuda")
hid = torch.from_numpy(w.phantom.material_id).pin_memory()
hde = torch.from_numpy(w.phantom.density).pin_memory()
for i in range(3):
    t = time.perf_counter()
    ids.copy_(torch.from_numpy(w.phantom.material_id), non_blocking=False)
    dens.copy_(torch.from_numpy(w.phantom.density), non_blocking=False)
    pk = A.Packed()
    p = pk.phantom(w.phantom)
    p.material_id = C.cast(C.c_void_p(ids.data_ptr()), C.POINTER(C.c_uint8))
    p.density = C.cast(C.c_void_p(dens.data_ptr()), C.POINTER(C.c_float))
    ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))
    print(f"raw H2D (pageable) + device encode {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
for i in range(3):
    t = time.perf_counter()
    ids.copy_(hid, non_blocking=True)
    dens.copy_(hde, non_blocking=True)
    pk = A.Packed()
    p = pk.phantom(w.phantom)
    p.material_id = C.cast(C.c_void_p(ids.data_ptr()), C.POINTER(C.c_uint8))
    p.density = C.cast(C.c_void_p(dens.data_ptr()), C.POINTER(C.c_float))
    ctx.check(A.lib().xs_upload_phantom_device(ctx.h, C.byref(p)))
    print(f"raw H2D (pinned) + device encode {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
