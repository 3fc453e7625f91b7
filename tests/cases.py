"""Shared test inputs (used by the golden generator and the tests)."""
import ctypes as C

import numpy as np

from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200 import synthetic as S

RNG_STREAMS = [(424242, 0, 0, 7), (20240915, 3, 12, 99999), (0xFFFFFFFF00000001, 7, 0, 0)]

SG_KERNELS = [(2, 2, 3), (0, 3, 3), (3, 0, 2), (7, 7, 3), (1, 7, 3), (4, 2, 2)]


def mixed_spectrum():
    """REF test_transport.cpp:296-310 apportionment spectrum."""
    return I.Spectrum(np.array([20.0, 40.0, 60.0, 80.0, 100.0]), np.array([0.001, 1.0, 2.0, 0.0, 0.5]))


def rods(n=32):
    return S.make_rods_phantom(n, 10.0 / n, 4.5, 8.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                               I.material("iron"), 7.874)


def crit2():
    """REF acceptance criterion 2 (acceptance_main.cpp:128-158)."""
    ph = S.make_cube_phantom(32, 0.2, 6.4, I.material("water"), 1.0)
    g = I.make_circular_geometry(60.0, 40.0, 24, 24, 0.55, 1)
    cfg = I.SimConfig(photons_total=100000, splitting=10, seed=424242, step_voxels=1)
    return ph, g, 0, I.monochromatic_spectrum(100.0), I.detector_response(), cfg


def poly(step=1):
    ph = rods(32)
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    cfg = I.SimConfig(photons_total=30000, splitting=5, seed=777, step_voxels=step,
                      roulette_wmin_rel=2.0, roulette_survival=0.6, track_variance=True)
    return ph, g, 2, I.kramers_spectrum(150.0), I.detector_response(), cfg


def head():
    """Scaled-down C3 (cylinder head) with the C3 spectrum and splitting."""
    ph = S.make_cylinder_head_phantom(64, 0.2, I.material("aluminum"), 2.699, I.material("iron"),
                                      7.874)
    g = I.make_circular_geometry(128.2, 86.2, 48, 40, 0.6, 3)
    cfg = I.SimConfig(photons_total=20000, splitting=20, seed=20240915)
    return ph, g, 1, I.kramers_spectrum(150.0), I.detector_response(), cfg


SCATTER_CASES = {"crit2": crit2, "poly1": lambda: poly(1), "poly3": lambda: poly(3),
                 "head": head}


def prim_c1_small():
    ph = S.make_cylinder_phantom(64, 0.2, 5.0, 10.0, I.material("water"), 1.0)
    g = I.make_circular_geometry(128.2, 86.2, 64, 48, 0.45, 5)
    return ph, g, 2, I.monochromatic_spectrum(60.0), I.detector_response()


def prim_head():
    ph, g, a, spec, resp, _ = head()
    return ph, g, 2, spec, resp


PRIMARY_CASES = {"c1_small": prim_c1_small, "head": prim_head}

# name -> (kind, n, voxel, params, density) for REF's generators (xr_make_phantom)
PHANTOMS = {
    "c1": (1, 128, 0.1, [5.0, 10.0], 1.0),
    "c2": (2, 256, 0.05, [5.0, 10.0, 4, 0.6, 3.0, 2.699], 1.0),
    "head96": (3, 96, 0.1, [7.874], 2.699),
    "cube": (0, 32, 0.2, [6.4], 1.0),
}


def our_phantom(name):
    kind, n, vox, p, dens = PHANTOMS[name]
    w, al, fe = I.material("water"), I.material("aluminum"), I.material("iron")
    if kind == 0:
        return S.make_cube_phantom(n, vox, p[0], w, dens)
    if kind == 1:
        return S.make_cylinder_phantom(n, vox, p[0], p[1], w, dens)
    if kind == 2:
        return S.make_rods_phantom(n, vox, p[0], p[1], w, dens, int(p[2]), p[3], p[4], al, p[5])
    return S.make_cylinder_head_phantom(n, vox, al, dens, fe, p[0])


def ref_phantom(ref, kind, n, vox, params, dens):
    ids = np.zeros(n ** 3, np.uint8)
    den = np.zeros(n ** 3, np.float32)
    dims = (C.c_int32 * 3)()
    vs = np.zeros(3)
    org = np.zeros(3)
    par = np.asarray(params, np.float64)
    st = ref.L.xr_make_phantom(kind, n, vox, par.ctypes.data_as(C.POINTER(C.c_double)), dens, dims,
                               vs.ctypes.data_as(C.POINTER(C.c_double)),
                               org.ctypes.data_as(C.POINTER(C.c_double)),
                               ids.ctypes.data_as(C.POINTER(C.c_uint8)),
                               den.ctypes.data_as(C.POINTER(C.c_float)))
    assert st == 0
    return ids, den
