"""The reference's file formats and text inputs through libxscatgpu.so
(csrc/files.cpp, declared in include/xscat_gpu.h).

Same names and meaning as REF's functions:
  save_stack / load_stack        XPRJ1   REF detector_image.cpp:33-87
  save_phantom / load_phantom    XVOX1   REF phantom.cpp:74-161
  load_phantom_header                    REF phantom.cpp:95-118
  save_volume / load_volume      XVOL1   REF volume.cpp:22-62
  load_material                  .mat    REF material.cpp:129-213
  load_spectrum                  CSV     REF spectrum.cpp:32-60
  load_detector_response         CSV     REF detector_response.cpp:50-79
Errors raise the exception types and messages REF throws.  No GPU needed.
"""
import ctypes as C
import dataclasses
from typing import List, Optional

import numpy as np

from . import _capi as A
from . import inputs as I
from .projector import ProjectionStack


def _path(p) -> bytes:
    return str(p).encode()


# ------------------------------------------------------------------ XPRJ1
def save_stack(stack: ProjectionStack, path) -> None:
    imgs = np.ascontiguousarray(stack.images, np.float64)
    n, nv, nu = imgs.shape
    A.check(A.lib().xs_stack_file_save(_path(path), nu, nv, n, A.dptr(imgs)))


def load_stack(path, angle_values=None) -> ProjectionStack:
    """REF load_stack: the f32 pixels widened to double; angle_values (if given)
    must have one entry per image."""
    L = A.lib()
    nu, nv, n = C.c_int32(), C.c_int32(), C.c_int32()
    A.check(L.xs_stack_file_info(_path(path), C.byref(nu), C.byref(nv), C.byref(n)))
    if angle_values is not None and len(angle_values) and len(angle_values) != n.value:
        raise I.XscatError(f"{path}: angle list size does not match file ({len(angle_values)} vs {n.value})")
    imgs = np.empty((n.value, nv.value, nu.value), np.float64)
    A.check(L.xs_stack_file_load(_path(path), A.dptr(imgs)))
    angles = (np.zeros(n.value) if angle_values is None or not len(angle_values)
              else np.asarray(angle_values, np.float64))
    return ProjectionStack(angles, imgs)


# ------------------------------------------------------------------ XVOX1
@dataclasses.dataclass
class PhantomHeader:
    """REF PhantomHeader (phantom.hpp:40-46)."""

    dims: tuple
    voxel_size: tuple
    origin: tuple
    material_count: int


def load_phantom_header(path) -> PhantomHeader:
    d = (C.c_int32 * 3)()
    vs, o = (C.c_double * 3)(), (C.c_double * 3)()
    nm = C.c_uint32()
    A.check(A.lib().xs_phantom_file_info(_path(path), d, vs, o, C.byref(nm)))
    return PhantomHeader(tuple(d), tuple(vs), tuple(o), int(nm.value))


def load_phantom(path, materials: List[Optional[I.Material]]) -> I.VoxelPhantom:
    """REF load_phantom: `materials` are the phantom's ids 1..N (a leading
    vacuum entry, None, is added when absent); validated like REF."""
    mats = list(materials)
    if not mats or mats[0] is not None:
        mats.insert(0, None)
    L = A.lib()
    h = C.c_void_p()
    A.check(L.xs_phantom_file_read(_path(path), len(mats), C.byref(h)))
    try:
        p = L.xs_phantom_file_get(h).contents
        n = int(p.dims[0]) * int(p.dims[1]) * int(p.dims[2])
        ph = I.VoxelPhantom(tuple(p.dims), tuple(p.voxel_size), tuple(p.origin),
                            np.ctypeslib.as_array(p.material_id, (n,)).copy(),
                            np.ctypeslib.as_array(p.density, (n,)).copy(), mats)
    finally:
        L.xs_phantom_file_free(h)
    pk = A.Packed()
    A.check(A.lib().xs_validate_phantom(C.byref(pk.phantom(ph))))
    return ph


def save_phantom(ph: I.VoxelPhantom, path) -> None:
    pk = A.Packed()
    A.check(A.lib().xs_phantom_file_save(_path(path), C.byref(pk.phantom(ph))))


# ------------------------------------------------------------------ XVOL1
@dataclasses.dataclass
class Volume:
    """REF Volume (volume.hpp:11-30): values (nz, ny, nx) float32."""

    values: np.ndarray
    voxel_size: tuple

    @property
    def dims(self):
        nz, ny, nx = self.values.shape
        return (nx, ny, nz)


def save_volume(v: Volume, path) -> None:
    vals = np.ascontiguousarray(v.values, np.float32)
    d = (C.c_int32 * 3)(*v.dims)
    vs = (C.c_double * 3)(*v.voxel_size)
    A.check(A.lib().xs_volume_file_save(_path(path), d, vs, vals.ctypes.data))


def load_volume(path) -> Volume:
    L = A.lib()
    d = (C.c_int32 * 3)()
    vs = (C.c_double * 3)()
    A.check(L.xs_volume_file_info(_path(path), d, vs))
    vals = np.empty((d[2], d[1], d[0]), np.float32)
    A.check(L.xs_volume_file_load(_path(path), vals.ctypes.data))
    return Volume(vals, tuple(vs))


# ------------------------------------------------------------- text inputs
def _table(t) -> I.Table1D:
    n = int(t.n)
    return I.Table1D(np.ctypeslib.as_array(t.x, (n,)).copy(), np.ctypeslib.as_array(t.y, (n,)).copy())


def load_material(path) -> I.Material:
    L = A.lib()
    h = C.c_void_p()
    A.check(L.xs_material_file_load(_path(path), C.byref(h)))
    try:
        m = L.xs_material_file_get(h).contents
        return I.Material(m.name.decode(), float(m.z_eff), float(m.density_ref), _table(m.mu),
                          _table(m.sigma_incoh), _table(m.sigma_coh), _table(m.sigma_pe),
                          _table(m.s_factor), _table(m.f_factor))
    finally:
        L.xs_material_file_free(h)


def load_spectrum(path) -> I.Spectrum:
    L = A.lib()
    h = C.c_void_p()
    A.check(L.xs_spectrum_file_load(_path(path), C.byref(h)))
    try:
        s = L.xs_spectrum_file_get(h).contents
        n = int(s.n_bins)
        return I.Spectrum(np.ctypeslib.as_array(s.energy_kev, (n,)).copy(),
                          np.ctypeslib.as_array(s.weight, (n,)).copy())
    finally:
        L.xs_spectrum_file_free(h)


def load_detector_response(path) -> I.DetectorResponse:
    L = A.lib()
    h = C.c_void_p()
    A.check(L.xs_response_file_load(_path(path), C.byref(h)))
    try:
        r = L.xs_response_file_get(h).contents
        return I.DetectorResponse(_table(r.dqe), _table(r.deposit))
    finally:
        L.xs_response_file_free(h)
