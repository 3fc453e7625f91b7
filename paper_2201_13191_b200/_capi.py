"""ctypes mirror of include/xscat_gpu.h and loader of the CUDA library.

The product path is ``lib/libxscatgpu.so`` (built by the repo Makefile from
``csrc/``).  There is no fallback: if the library or a CUDA device is missing,
the projector raises.  The struct packers here are shared with the test
oracles (which take the same POD structs), but nothing in this package loads
or calls anything under ``oracle/``.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
from typing import List, Optional

import numpy as np

from . import inputs as I

PKG = pathlib.Path(__file__).resolve().parent
# XSCAT_LIB: an alternative build of the library (A/B experiments, tools/ab.sh);
# the product path is the in-tree lib/libxscatgpu.so
LIB_PATH = pathlib.Path(os.environ["XSCAT_LIB"]) if os.environ.get("XSCAT_LIB") else PKG / "lib" / "libxscatgpu.so"

c_double_p = C.POINTER(C.c_double)
c_u64_p = C.POINTER(C.c_uint64)


class XsTable(C.Structure):
    _fields_ = [("n", C.c_int32), ("x", c_double_p), ("y", c_double_p)]


class XsMaterial(C.Structure):
    _fields_ = [("name", C.c_char_p), ("z_eff", C.c_double), ("density_ref", C.c_double),
                ("mu", XsTable), ("sigma_incoh", XsTable), ("sigma_coh", XsTable),
                ("sigma_pe", XsTable), ("s_factor", XsTable), ("f_factor", XsTable)]


class XsPhantom(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("voxel_size", C.c_double * 3),
                ("origin", C.c_double * 3), ("material_id", C.POINTER(C.c_uint8)),
                ("density", C.POINTER(C.c_float)), ("n_materials", C.c_int32),
                ("materials", C.POINTER(XsMaterial))]


class XsGeometry(C.Structure):
    _fields_ = [("sdd", C.c_double), ("sod", C.c_double), ("nu", C.c_int32), ("nv", C.c_int32),
                ("pixel_pitch", C.c_double), ("n_angles", C.c_int32), ("angles", c_double_p)]


class XsSpectrum(C.Structure):
    _fields_ = [("n_bins", C.c_int32), ("energy_kev", c_double_p), ("weight", c_double_p)]


class XsResponse(C.Structure):
    _fields_ = [("dqe", XsTable), ("deposit", XsTable)]


class XsSimConfig(C.Structure):
    _fields_ = [("photons_total", C.c_uint64), ("splitting", C.c_int32),
                ("roulette_survival", C.c_double), ("roulette_wmin_rel", C.c_double),
                ("step_voxels", C.c_int32), ("max_interactions", C.c_int32),
                ("seed", C.c_uint64), ("track_variance", C.c_int32)]


class XsClassSpec(C.Structure):
    _fields_ = [("material_id", C.c_int32), ("density", C.c_double)]


class XsCorrectionConfig(C.Structure):
    _fields_ = [("n_iterations", C.c_int32), ("simulate_every_kth_angle", C.c_int32),
                ("mc_nu", C.c_int32), ("mc_nv", C.c_int32), ("recon_dims", C.c_int32 * 3),
                ("n_classes", C.c_int32), ("class_map", C.POINTER(XsClassSpec)),
                ("sim", XsSimConfig), ("sg_window", C.c_int32), ("sg_polyorder", C.c_int32),
                ("sg_auto_window", C.c_int32)]


class XsIterationReport(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("pad_", C.c_int32)] + [
        (k, C.c_double) for k in ("seconds_fbp", "seconds_segmentation", "seconds_mc_scatter",
                                  "seconds_mc_primary", "seconds_postprocess", "seconds_correction",
                                  "seconds_total", "mc_seconds_per_projection",
                                  "mean_scatter_fraction", "ncc_to_previous")] + [
        ("negative_scatter_clamped", C.c_uint64)]


class XsLedger(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("initial", "escaped", "absorbed", "culled",
                                          "roulette_killed", "roulette_boost")]


class XsScatterResult(C.Structure):
    _fields_ = [("image", c_double_p), ("variance", c_double_p), ("ledger", XsLedger),
                ("histories", C.c_uint64), ("total", C.c_double),
                ("total_std_error", C.c_double)]


class XsLaunchStats(C.Structure):
    _fields_ = [("free_path_steps", C.c_uint64), ("scoring_steps", C.c_uint64),
                ("histories", C.c_uint64), ("scoring_rays", C.c_uint64),
                ("interactions", C.c_uint64), ("kernel_ms", C.c_double),
                ("voxel_format", C.c_int32), ("palette_size", C.c_int32),
                ("upload_bytes", C.c_uint64), ("walk_iterations", C.c_uint64),
                ("walk_lane_slots", C.c_uint64), ("blocks_per_sm", C.c_uint32),
                ("smem_per_block", C.c_uint32), ("slots_per_warp", C.c_uint32),
                ("engine", C.c_uint32), ("waves", C.c_uint32), ("live_histories", C.c_uint32),
                ("uniform_iterations", C.c_uint64), ("walk_ms", C.c_float), ("launches", C.c_uint32),
                ("block_walk", C.c_uint32), ("setup_ms", C.c_float), ("score_ms", C.c_float),
                ("event_ms", C.c_float), ("admit_ms", C.c_float)]


def dptr(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


# --------------------------------------------------------------- packing
class Packed:
    """Owns the numpy buffers behind a set of C structs (keeps them alive)."""

    def __init__(self):
        self._keep: List[object] = []

    def keep(self, *objs):
        self._keep.extend(objs)
        return objs[0] if len(objs) == 1 else objs

    def table(self, t: Optional[I.Table1D]) -> XsTable:
        if t is None:
            return XsTable(0, None, None)
        x = self.keep(np.ascontiguousarray(t.x, np.float64))
        y = self.keep(np.ascontiguousarray(t.y, np.float64))
        return XsTable(int(x.size), dptr(x), dptr(y))

    def material(self, m: Optional[I.Material], out: XsMaterial) -> None:
        if m is None:  # vacuum sentinel
            out.name = b"vacuum"
            out.z_eff = 0.0
            out.density_ref = 0.0
            for f in ("mu", "sigma_incoh", "sigma_coh", "sigma_pe", "s_factor", "f_factor"):
                setattr(out, f, XsTable(0, None, None))
            return
        name = self.keep(m.name.encode())
        out.name = name
        out.z_eff = m.z_eff
        out.density_ref = m.density_ref
        out.mu = self.table(m.mu)
        out.sigma_incoh = self.table(m.sigma_incoh)
        out.sigma_coh = self.table(m.sigma_coh)
        out.sigma_pe = self.table(m.sigma_pe)
        out.s_factor = self.table(m.s_factor)
        out.f_factor = self.table(m.f_factor)

    def materials(self, mats) -> "C.Array":
        """xs_material array of a REF material list (index 0 = vacuum sentinel)."""
        arr = (XsMaterial * len(mats))()
        for i, m in enumerate(mats):
            self.material(m, arr[i])
        return self.keep(arr)

    def class_map(self, cmap) -> "C.Array":
        arr = (XsClassSpec * max(1, len(cmap)))()
        for i, c in enumerate(cmap):
            arr[i].material_id = int(c.material_id)
            arr[i].density = float(c.density)
        return self.keep(arr)

    def correction_config(self, cc) -> XsCorrectionConfig:
        """xs_correction_config of a projector.CorrectionConfig."""
        x = XsCorrectionConfig()
        x.n_iterations = int(cc.n_iterations)
        x.simulate_every_kth_angle = int(cc.simulate_every_kth_angle)
        x.mc_nu, x.mc_nv = int(cc.mc_nu), int(cc.mc_nv)
        x.recon_dims[:] = [int(d) for d in cc.recon_dims]
        x.n_classes = int(cc.n_classes)
        x.class_map = C.cast(self.class_map(cc.class_map), C.POINTER(XsClassSpec))
        x.sim = self.config(cc.sim)
        x.sg_window, x.sg_polyorder = int(cc.sg.window), int(cc.sg.polyorder)
        x.sg_auto_window = 1 if cc.sg_auto_window else 0
        return self.keep(x)

    def phantom(self, ph: I.VoxelPhantom) -> XsPhantom:
        mats = (XsMaterial * len(ph.materials))()
        for i, m in enumerate(ph.materials):
            self.material(m, mats[i])
        ids = self.keep(np.ascontiguousarray(ph.material_id, np.uint8))
        dens = self.keep(np.ascontiguousarray(ph.density, np.float32))
        self.keep(mats)
        p = XsPhantom()
        p.dims[:] = list(ph.dims)
        p.voxel_size[:] = list(ph.voxel_size)
        p.origin[:] = list(ph.origin)
        p.material_id = ids.ctypes.data_as(C.POINTER(C.c_uint8))
        p.density = dens.ctypes.data_as(C.POINTER(C.c_float))
        p.n_materials = len(ph.materials)
        p.materials = C.cast(mats, C.POINTER(XsMaterial))
        return self.keep(p)

    def geometry(self, g: I.ScanGeometry) -> XsGeometry:
        a = self.keep(np.ascontiguousarray(g.angles, np.float64))
        return self.keep(XsGeometry(g.sdd, g.sod, g.nu, g.nv, g.pixel_pitch, int(a.size),
                                    dptr(a)))

    def spectrum(self, s: I.Spectrum) -> XsSpectrum:
        e = self.keep(np.ascontiguousarray(s.energy_kev, np.float64))
        w = self.keep(np.ascontiguousarray(s.weight, np.float64))
        return self.keep(XsSpectrum(int(e.size), dptr(e), dptr(w)))

    def response(self, r: I.DetectorResponse) -> XsResponse:
        return self.keep(XsResponse(self.table(r.dqe), self.table(r.deposit)))

    def config(self, c: I.SimConfig) -> XsSimConfig:
        return self.keep(XsSimConfig(int(c.photons_total), int(c.splitting),
                                     float(c.roulette_survival), float(c.roulette_wmin_rel),
                                     int(c.step_voxels), int(c.max_interactions),
                                     int(c.seed) & 0xFFFFFFFFFFFFFFFF,
                                     1 if c.track_variance else 0))


class XsCommId(C.Structure):
    """include/xscat_gpu.h xs_comm_id (an NCCL unique id, 128 bytes)."""
    _fields_ = [("internal", C.c_char * 128)]


# ------------------------------------------------------ accumulator layout
def accum_layout(nu: int, nv: int, n_bins: int, track_variance: bool) -> dict:
    """include/xscat_gpu.h xs_accum_layout_make."""
    n_pixels = nu * nv
    off_variance = 4 * n_pixels
    off_bins = off_variance + (4 * n_pixels if track_variance else 0)
    off_ledger = off_bins + 8 * n_bins
    off_diag = off_ledger + 24
    return dict(n_pixels=n_pixels, off_image=0, off_variance=off_variance, off_bins=off_bins,
                off_ledger=off_ledger, off_diag=off_diag, words=off_diag + 8)


# ------------------------------------------------------------ the library
_STATUS_EXC = {1: I.XscatError, 2: I.XscatOutOfRange, 3: I.XscatInvalidArgument,
               4: I.XscatDomainError, 5: I.XscatError, 6: I.XscatError}

_lib = None

# symbol -> (restype, argtypes); every function declared in include/xscat_gpu.h
_P = C.c_void_p
SIGNATURES = {
    "xs_version": (C.c_char_p, []),
    "xs_abi_version": (C.c_int, []),
    "xs_last_error": (C.c_char_p, [_P]),
    "xs_sim_config_default": (None, [C.POINTER(XsSimConfig)]),
    "xs_validate_sim_config": (C.c_int, [C.POINTER(XsSimConfig)]),
    "xs_apportion_photons": (C.c_int, [C.POINTER(XsSpectrum), C.c_uint64, c_u64_p]),
    "xs_point_detector_score": (C.c_double, [C.c_double] * 6),
    "xs_scatter_finalize_host": (C.c_int, [C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                                           C.POINTER(XsSimConfig), c_u64_p, C.c_uint64,
                                           C.c_uint64, C.POINTER(XsScatterResult)]),
    "xs_history_count": (C.c_int, [C.POINTER(XsSpectrum), C.c_uint64, c_u64_p]),
    "xs_validate_sg_spec": (C.c_int, [C.c_int32, C.c_int32]),
    "xs_default_sg_spec": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]),
    "xs_sg_kernel": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, c_double_p]),
    "xs_device_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "xs_ctx_create": (C.c_int, [C.c_int32, C.POINTER(_P)]),
    "xs_ctx_destroy": (None, [_P]),
    "xs_ctx_set_stream": (C.c_int, [_P, _P]),
    "xs_ctx_synchronize": (C.c_int, [_P]),
    "xs_ctx_set_option": (C.c_int, [_P, C.c_char_p, C.c_int64]),
    "xs_upload_phantom": (C.c_int, [_P, C.POINTER(XsPhantom)]),
    "xs_upload_response": (C.c_int, [_P, C.POINTER(XsResponse)]),
    "xs_simulate_scatter_stats": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                            C.POINTER(XsSpectrum), C.POINTER(XsSimConfig),
                                            C.POINTER(XsScatterResult)]),
    "xs_simulate_primary": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                      C.POINTER(XsSpectrum), C.POINTER(XsSimConfig),
                                      c_double_p]),
    "xs_run_scan": (C.c_int, [_P, C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                              C.POINTER(XsSimConfig), C.POINTER(C.c_int32), C.c_int32,
                              C.c_int32, c_double_p, c_double_p, c_double_p]),
    "xs_scatter_accumulate_device": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                               C.POINTER(XsSpectrum), C.POINTER(XsSimConfig),
                                               C.c_uint64, C.c_uint64, _P]),
    "xs_scatter_finalize_device": (C.c_int, [_P, C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                                             C.POINTER(XsSimConfig), _P, C.c_uint64,
                                             C.c_uint64, C.POINTER(XsScatterResult), _P]),
    "xs_primary_device": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                    C.POINTER(XsSpectrum), C.POINTER(XsSimConfig), _P]),
    "xs_last_launch_stats": (C.c_int, [_P, C.POINTER(XsLaunchStats)]),
    "xs_sg_smooth": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                               C.c_int32, C.c_int32]),
    "xs_interpolate_angles": (C.c_int, [_P, _P, c_double_p, C.c_int32, _P, c_double_p,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "xs_upsample_image": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32,
                                    C.c_int32, C.c_int32]),
    "xs_downsample_average": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, _P,
                                        C.c_int32, C.c_int32, C.c_int32]),
    "xs_fbp_reconstruct": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(XsGeometry), C.POINTER(C.c_int32), _P, C.c_int32, _P,
                                     C.c_int32]),
    "xs_default_voxel_size": (None, [C.POINTER(XsGeometry), C.POINTER(C.c_int32), _P]),
    "xs_intensity_to_attenuation": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P,
                                              C.c_int32]),
    "xs_correct_projections": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, _P,
                                         C.POINTER(C.c_uint64), C.c_int32]),
    "xs_correction_tail": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32,
                                     _P, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int32]),
    "xs_otsu_thresholds": (C.c_int, [_P, _P, C.POINTER(C.c_int32), C.c_int32, C.c_int32, _P,
                                     C.c_int32]),
    "xs_segment_volume": (C.c_int, [_P, _P, C.c_uint64, _P, C.c_int32, C.c_int32, _P, C.c_int32]),
    "xs_to_density_phantom": (C.c_int, [_P, _P, C.POINTER(C.c_int32), C.POINTER(XsClassSpec),
                                        C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                        C.POINTER(XsMaterial), _P, _P, C.c_int32]),
    "xs_segment_to_scene": (C.c_int, [_P, _P, C.POINTER(C.c_int32), _P, C.c_int32, C.c_int32,
                                      C.POINTER(XsClassSpec), C.POINTER(C.c_int32), C.c_int32,
                                      C.POINTER(XsMaterial), _P, C.c_int32]),
    "xs_upload_phantom_device": (C.c_int, [_P, C.POINTER(XsPhantom)]),
    "xs_run_scan_device": (C.c_int, [_P, C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                                     C.POINTER(XsSimConfig), C.POINTER(C.c_int32), C.c_int32,
                                     C.c_int32, _P, _P, _P]),
    "xs_ctx_copy_scene": (C.c_int, [_P, _P]),
    "xs_comm_unique_id": (C.c_int, [C.POINTER(XsCommId)]),
    "xs_ctx_comm_init": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(XsCommId)]),
    "xs_ctx_comm_size": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "xs_simulate_scatter_stats_mgpu": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                                 C.POINTER(XsSpectrum), C.POINTER(XsSimConfig),
                                                 C.c_int32, C.POINTER(XsScatterResult), _P]),
    "xs_run_scan_mgpu": (C.c_int, [_P, C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                                   C.POINTER(XsSimConfig), C.POINTER(C.c_int32), C.c_int32,
                                   C.c_int32, C.c_int32, C.c_int32, c_double_p, c_double_p,
                                   c_double_p]),
    "xs_group_create": (C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.POINTER(_P)]),
    "xs_group_destroy": (None, [_P]),
    "xs_group_size": (C.c_int32, [_P]),
    "xs_group_context": (_P, [_P, C.c_int32]),
    "xs_group_last_error": (C.c_char_p, [_P]),
    "xs_group_set_option": (C.c_int, [_P, C.c_char_p, C.c_int64]),
    "xs_group_upload_phantom": (C.c_int, [_P, C.POINTER(XsPhantom)]),
    "xs_group_upload_response": (C.c_int, [_P, C.POINTER(XsResponse)]),
    "xs_group_simulate_scatter_stats": (C.c_int, [_P, C.POINTER(XsGeometry), C.c_int32,
                                                  C.POINTER(XsSpectrum), C.POINTER(XsSimConfig),
                                                  C.POINTER(XsScatterResult)]),
    "xs_group_run_scan": (C.c_int, [_P, C.POINTER(XsGeometry), C.POINTER(XsSpectrum),
                                    C.POINTER(XsSimConfig), C.POINTER(C.c_int32), C.c_int32,
                                    C.c_int32, c_double_p, c_double_p, c_double_p]),
    "xs_group_run_iterative_correction": (C.c_int, [_P, _P, _P, C.POINTER(XsGeometry),
                                                    C.POINTER(XsSpectrum),
                                                    C.POINTER(XsCorrectionConfig), C.c_int32,
                                                    C.POINTER(XsMaterial), _P, _P,
                                                    C.POINTER(XsIterationReport), C.c_int32]),
    # files and inputs (csrc/files.cpp)
    "xs_stack_file_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]),
    "xs_stack_file_load": (C.c_int, [C.c_char_p, c_double_p]),
    "xs_stack_file_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, c_double_p]),
    "xs_phantom_file_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), c_double_p, c_double_p,
                                       C.POINTER(C.c_uint32)]),
    "xs_phantom_file_read": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(_P)]),
    "xs_phantom_file_get": (C.POINTER(XsPhantom), [_P]),
    "xs_phantom_file_free": (None, [_P]),
    "xs_phantom_file_save": (C.c_int, [C.c_char_p, C.POINTER(XsPhantom)]),
    "xs_validate_phantom": (C.c_int, [C.POINTER(XsPhantom)]),
    "xs_volume_file_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), c_double_p]),
    "xs_volume_file_load": (C.c_int, [C.c_char_p, _P]),
    "xs_volume_file_save": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), c_double_p, _P]),
    "xs_material_file_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "xs_material_file_get": (C.POINTER(XsMaterial), [_P]),
    "xs_material_file_free": (None, [_P]),
    "xs_spectrum_file_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "xs_spectrum_file_get": (C.POINTER(XsSpectrum), [_P]),
    "xs_spectrum_file_free": (None, [_P]),
    "xs_response_file_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "xs_response_file_get": (C.POINTER(XsResponse), [_P]),
    "xs_response_file_free": (None, [_P]),
    "xs_correction_config_default": (None, [C.POINTER(XsCorrectionConfig)]),
    "xs_run_iterative_correction": (C.c_int, [_P, _P, _P, C.POINTER(XsGeometry),
                                              C.POINTER(XsSpectrum),
                                              C.POINTER(XsCorrectionConfig), C.c_int32,
                                              C.POINTER(XsMaterial), _P, _P,
                                              C.POINTER(XsIterationReport), C.c_int32]),
}


def _preload_nccl():
    """libxscatgpu.so links libnccl.so.2 (its multi-GPU entry points).  When
    PyTorch's newer NCCL wheel is installed, load that one first: the process
    then holds a single NCCL that both libxscatgpu and torch (imported before
    or after) resolve against."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []) if spec else []:
            p = pathlib.Path(d) / "lib" / "libnccl.so.2"
            if p.exists():
                C.CDLL(str(p), mode=C.RTLD_GLOBAL)
                return
    except Exception:
        pass


def lib():
    """Load libxscatgpu.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise I.XscatError(f"CUDA library missing: {LIB_PATH} (run `make` or "
                               "__graft_entry__.build())")
        _preload_nccl()
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("XSCAT_LIB") and not hasattr(L, name):
                continue  # an older A/B build: bind what it has
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, ctx=None) -> None:
    if status != 0:
        msg = lib().xs_last_error(ctx)
        raise _STATUS_EXC.get(status, I.XscatError)(
            (msg or b"").decode(errors="replace") or f"xscat status {status}")
