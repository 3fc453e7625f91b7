"""The projector API, mirroring REF include/xscat/transport.hpp:69-116 and
include/xscat/postprocess.hpp:13-41, executed by libxscatgpu.so on a B200.

Free functions keep REF's signatures (``workers`` is accepted and ignored:
results are worker- and GPU-count independent by construction).  They take
the phantom on every call like REF does and therefore upload it every call;
use :class:`Projector` to upload a scene once and run many projections.

There is no CPU fallback: without the CUDA library or a CUDA device every
call raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _capi as A
from . import inputs as I


@dataclasses.dataclass
class WeightLedger:
    """REF WeightLedger (transport.hpp:38-56)."""

    initial: float = 0.0
    escaped: float = 0.0
    absorbed: float = 0.0
    culled: float = 0.0
    roulette_killed: float = 0.0
    roulette_boost: float = 0.0


@dataclasses.dataclass
class SimResult:
    """REF SimResult (transport.hpp:58-64); image is (nv, nu) fp64."""

    image: np.ndarray
    variance: Optional[np.ndarray]
    ledger: WeightLedger
    histories: int
    total: float
    total_std_error: float
    stats: Optional[Dict[str, float]] = None


@dataclasses.dataclass
class ProjectionStack:
    """REF ProjectionStack (detector_image.hpp:28-34): images (n, nv, nu)."""

    angle_values: np.ndarray
    images: np.ndarray

    @property
    def n_angles(self):
        return int(self.images.shape[0])


@dataclasses.dataclass
class ScanResult:
    """REF ScanResult (transport.hpp:104-110)."""

    primary: Optional[ProjectionStack]
    scatter: Optional[ProjectionStack]
    seconds_per_angle: List[float]


PRIMARY, SCATTER, BOTH = 0, 1, 2  # REF ScanQuantity


def device_count() -> int:
    n = C.c_int32()
    A.check(A.lib().xs_device_count(C.byref(n)))
    return n.value


class Context:
    """One CUDA device + stream + uploaded scene (an ``xs_context``)."""

    def __init__(self, device: int = 0):
        L = A.lib()
        h = C.c_void_p()
        A.check(L.xs_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            A.lib().xs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st):
        A.check(st, self.h)

    def set_option(self, key: str, value: int):
        """xs_ctx_set_option: "exact_walk", "smem_kb", "max_slots", "grab"."""
        self.check(A.lib().xs_ctx_set_option(self.h, key.encode(), int(value)))

    def set_stream(self, cuda_stream_ptr: int):
        self.check(A.lib().xs_ctx_set_stream(self.h, C.c_void_p(cuda_stream_ptr)))

    def upload(self, ph: I.VoxelPhantom, resp: I.DetectorResponse):
        pk = A.Packed()
        self.check(A.lib().xs_upload_phantom(self.h, C.byref(pk.phantom(ph))))
        self.check(A.lib().xs_upload_response(self.h, C.byref(pk.response(resp))))

    # multi-process (one process per GPU): an NCCL communicator in the library
    @staticmethod
    def comm_unique_id() -> bytes:
        """xs_comm_unique_id on the rank that creates the communicator; send
        the 128 bytes to every rank (e.g. torch.distributed.broadcast)."""
        cid = A.XsCommId()
        A.check(A.lib().xs_comm_unique_id(C.byref(cid)))
        return C.string_at(C.addressof(cid), 128)

    def comm_init(self, n_ranks: int, rank: int, unique_id: bytes):
        cid = A.XsCommId()
        C.memmove(C.addressof(cid), bytes(unique_id), min(len(unique_id), 128))
        self.check(A.lib().xs_ctx_comm_init(self.h, int(n_ranks), int(rank), C.byref(cid)))

    def comm_size(self):
        n, r = C.c_int32(), C.c_int32()
        self.check(A.lib().xs_ctx_comm_size(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def launch_stats(self) -> Dict[str, float]:
        s = A.XsLaunchStats()
        self.check(A.lib().xs_last_launch_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in A.XsLaunchStats._fields_}


_contexts: Dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


def _result(img, var, res, g, stats=None) -> SimResult:
    return SimResult(img.reshape(g.nv, g.nu), None if var is None else var.reshape(g.nv, g.nu),
                     WeightLedger(*[getattr(res.ledger, k) for k, _ in A.XsLedger._fields_]),
                     int(res.histories), float(res.total), float(res.total_std_error), stats)


class Projector:
    """A scene (phantom + detector response) resident on one GPU."""

    def __init__(self, phantom: I.VoxelPhantom, response: I.DetectorResponse,
                 ctx: Optional[Context] = None, device: int = 0):
        self.ctx = ctx or default_context(device)
        self.phantom = phantom
        self.response = response
        self.ctx.upload(phantom, response)

    # REF simulate_scatter_stats (transport.cpp:246-324)
    def scatter_stats(self, g: I.ScanGeometry, angle_idx: int, spec: I.Spectrum,
                      cfg: I.SimConfig) -> SimResult:
        pk = A.Packed()
        img = np.empty(g.nu * g.nv)
        var = np.empty(g.nu * g.nv) if cfg.track_variance else None
        res = A.XsScatterResult()
        res.image = A.dptr(img)
        res.variance = A.dptr(var) if var is not None else None
        self.ctx.check(A.lib().xs_simulate_scatter_stats(
            self.ctx.h, C.byref(pk.geometry(g)), angle_idx, C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), C.byref(res)))
        return _result(img, var, res, g, self.ctx.launch_stats())

    # REF simulate_primary (transport.cpp:333-377)
    def primary(self, g: I.ScanGeometry, angle_idx: int, spec: I.Spectrum,
                cfg: Optional[I.SimConfig] = None) -> np.ndarray:
        pk = A.Packed()
        img = np.empty(g.nu * g.nv)
        self.ctx.check(A.lib().xs_simulate_primary(
            self.ctx.h, C.byref(pk.geometry(g)), angle_idx, C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg or I.SimConfig())), A.dptr(img)))
        return img.reshape(g.nv, g.nu)

    # REF run_scan (transport.cpp:379-422)
    def run_scan(self, g: I.ScanGeometry, spec: I.Spectrum, cfg: I.SimConfig,
                 angle_subset: Sequence[int], what: int = BOTH) -> ScanResult:
        pk = A.Packed()
        sub = np.ascontiguousarray(np.asarray(angle_subset, dtype=np.int32))
        n = int(sub.size)
        np_ = g.nu * g.nv
        prim = np.empty((max(n, 1), g.nv, g.nu)) if what != SCATTER else None
        scat = np.empty((max(n, 1), g.nv, g.nu)) if what != PRIMARY else None
        secs = np.zeros(max(n, 1))
        self.ctx.check(A.lib().xs_run_scan(
            self.ctx.h, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), sub.ctypes.data_as(C.POINTER(C.c_int32)), n, what,
            A.dptr(prim) if prim is not None else None,
            A.dptr(scat) if scat is not None else None, A.dptr(secs)))
        angles = g.angles[sub] if n else np.zeros(0)
        return ScanResult(None if prim is None else ProjectionStack(angles, prim[:n]),
                          None if scat is None else ProjectionStack(angles, scat[:n]),
                          list(secs[:n]))

    # photon batches / angle ranges over the context's NCCL communicator
    def scatter_stats_mgpu(self, g: I.ScanGeometry, angle_idx: int, spec: I.Spectrum,
                           cfg: I.SimConfig, root: int = 0, d_image_ptr: int = 0,
                           host_image: bool = True, image_out: Optional[np.ndarray] = None) -> SimResult:
        """xs_simulate_scatter_stats_mgpu: every rank calls it; the root's
        result holds the whole projection, the others only `histories`.
        image_out: a caller-owned float64 host buffer of nu*nv pixels to fill
        (reused across calls), else one is allocated."""
        pk = A.Packed()
        if image_out is not None:
            assert image_out.dtype == np.float64 and image_out.flags.c_contiguous and image_out.size == g.nu * g.nv
        img = (image_out.reshape(-1) if image_out is not None else np.empty(g.nu * g.nv)) if host_image else None
        var = np.empty(g.nu * g.nv) if cfg.track_variance and host_image else None
        res = A.XsScatterResult()
        res.image = A.dptr(img) if img is not None else None
        res.variance = A.dptr(var) if var is not None else None
        self.ctx.check(A.lib().xs_simulate_scatter_stats_mgpu(
            self.ctx.h, C.byref(pk.geometry(g)), angle_idx, C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), int(root), C.byref(res),
            C.c_void_p(d_image_ptr) if d_image_ptr else None))
        if img is None:
            img = np.zeros(g.nu * g.nv)
        return _result(img, var, res, g, self.ctx.launch_stats())

    def run_scan_mgpu(self, g: I.ScanGeometry, spec: I.Spectrum, cfg: I.SimConfig,
                      angle_subset: Sequence[int], what: int = BOTH, gather: bool = True,
                      root: int = 0, primary_out: Optional[np.ndarray] = None,
                      scatter_out: Optional[np.ndarray] = None) -> ScanResult:
        """xs_run_scan_mgpu: this rank's angle range (all of them on the root
        with gather).  primary_out / scatter_out: caller-owned (n, nv, nu)
        float64 arrays to fill (reused across calls), else allocated here."""
        pk = A.Packed()
        sub = np.ascontiguousarray(np.asarray(angle_subset, dtype=np.int32))
        n = int(sub.size)
        prim = scat = None
        if what != SCATTER:
            prim = primary_out if primary_out is not None else np.zeros((max(n, 1), g.nv, g.nu))
        if what != PRIMARY:
            scat = scatter_out if scatter_out is not None else np.zeros((max(n, 1), g.nv, g.nu))
        for a in (prim, scat):
            assert a is None or (a.dtype == np.float64 and a.flags.c_contiguous and a.size >= n * g.nu * g.nv)
        secs = np.zeros(max(n, 1))
        self.ctx.check(A.lib().xs_run_scan_mgpu(
            self.ctx.h, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), sub.ctypes.data_as(C.POINTER(C.c_int32)), n, what,
            1 if gather else 0, int(root),
            A.dptr(prim) if prim is not None else None,
            A.dptr(scat) if scat is not None else None, A.dptr(secs)))
        angles = g.angles[sub] if n else np.zeros(0)
        return ScanResult(None if prim is None else ProjectionStack(angles, prim[:n]),
                          None if scat is None else ProjectionStack(angles, scat[:n]),
                          list(secs[:n]))

    # device-level split (photon batches across GPUs)
    def accumulate(self, g, angle_idx, spec, cfg, hist_begin, hist_end, d_accum_ptr: int):
        pk = A.Packed()
        self.ctx.check(A.lib().xs_scatter_accumulate_device(
            self.ctx.h, C.byref(pk.geometry(g)), angle_idx, C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), hist_begin, hist_end, C.c_void_p(d_accum_ptr)))

    def finalize(self, g, spec, cfg, d_accum_ptr: int, hist_begin, hist_end) -> SimResult:
        pk = A.Packed()
        img = np.empty(g.nu * g.nv)
        var = np.empty(g.nu * g.nv) if cfg.track_variance else None
        res = A.XsScatterResult()
        res.image = A.dptr(img)
        res.variance = A.dptr(var) if var is not None else None
        self.ctx.check(A.lib().xs_scatter_finalize_device(
            self.ctx.h, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), C.c_void_p(d_accum_ptr), hist_begin, hist_end,
            C.byref(res), None))
        return _result(img, var, res, g, self.ctx.launch_stats())


class Group:
    """One process, several GPUs (an ``xs_group``): a scene replicated on every
    member; scatter projections split into photon batches over the members
    (their accumulators summed by the root's finalize kernel over NVLink peer
    memory), scans and the correction loop's scans split by angle.  A device
    may be listed more than once."""

    def __init__(self, devices: Sequence[int], phantom: Optional[I.VoxelPhantom] = None,
                 response: Optional[I.DetectorResponse] = None):
        L = A.lib()
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        A.check(L.xs_group_create(devs, len(devices), C.byref(h)))
        self.h = h
        self.devices = list(devices)
        if phantom is not None:
            self.upload(phantom, response)

    def close(self):
        if self.h:
            A.lib().xs_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st):
        if st != 0:
            msg = A.lib().xs_group_last_error(self.h)
            raise A._STATUS_EXC.get(st, I.XscatError)((msg or b"").decode(errors="replace"))

    def __len__(self):
        return int(A.lib().xs_group_size(self.h))

    def set_option(self, key: str, value: int):
        self.check(A.lib().xs_group_set_option(self.h, key.encode(), int(value)))

    def upload(self, ph: I.VoxelPhantom, resp: Optional[I.DetectorResponse]):
        pk = A.Packed()
        if resp is not None:
            self.check(A.lib().xs_group_upload_response(self.h, C.byref(pk.response(resp))))
        self.check(A.lib().xs_group_upload_phantom(self.h, C.byref(pk.phantom(ph))))

    def launch_stats(self, member: int = 0) -> Dict[str, float]:
        s = A.XsLaunchStats()
        A.check(A.lib().xs_last_launch_stats(A.lib().xs_group_context(self.h, member), C.byref(s)))
        return {k: getattr(s, k) for k, _ in A.XsLaunchStats._fields_}

    def scatter_stats(self, g: I.ScanGeometry, angle_idx: int, spec: I.Spectrum,
                      cfg: I.SimConfig) -> SimResult:
        pk = A.Packed()
        img = np.empty(g.nu * g.nv)
        var = np.empty(g.nu * g.nv) if cfg.track_variance else None
        res = A.XsScatterResult()
        res.image = A.dptr(img)
        res.variance = A.dptr(var) if var is not None else None
        self.check(A.lib().xs_group_simulate_scatter_stats(
            self.h, C.byref(pk.geometry(g)), angle_idx, C.byref(pk.spectrum(spec)),
            C.byref(pk.config(cfg)), C.byref(res)))
        return _result(img, var, res, g, self.launch_stats())

    def run_scan(self, g: I.ScanGeometry, spec: I.Spectrum, cfg: I.SimConfig,
                 angle_subset: Sequence[int], what: int = BOTH) -> ScanResult:
        pk = A.Packed()
        sub = np.ascontiguousarray(np.asarray(angle_subset, dtype=np.int32))
        n = int(sub.size)
        prim = np.empty((max(n, 1), g.nv, g.nu)) if what != SCATTER else None
        scat = np.empty((max(n, 1), g.nv, g.nu)) if what != PRIMARY else None
        secs = np.zeros(max(n, 1))
        self.check(A.lib().xs_group_run_scan(
            self.h, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)), C.byref(pk.config(cfg)),
            sub.ctypes.data_as(C.POINTER(C.c_int32)), n, what,
            A.dptr(prim) if prim is not None else None,
            A.dptr(scat) if scat is not None else None, A.dptr(secs)))
        angles = g.angles[sub] if n else np.zeros(0)
        return ScanResult(None if prim is None else ProjectionStack(angles, prim[:n]),
                          None if scat is None else ProjectionStack(angles, scat[:n]),
                          list(secs[:n]))


# ------------------------------------------------ REF-signature free functions
def simulate_scatter_stats(ph, g, angle_idx, spec, resp, cfg, workers: int = 1,
                           device: int = 0) -> SimResult:
    return Projector(ph, resp, device=device).scatter_stats(g, angle_idx, spec, cfg)


def simulate_scatter(ph, g, angle_idx, spec, resp, cfg, workers: int = 1, device: int = 0):
    return simulate_scatter_stats(ph, g, angle_idx, spec, resp, cfg, workers, device).image


def simulate_primary(ph, g, angle_idx, spec, resp, cfg=None, workers: int = 1, device: int = 0):
    return Projector(ph, resp, device=device).primary(g, angle_idx, spec, cfg)


def run_scan(ph, g, spec, resp, cfg, angle_subset, what=BOTH, workers: int = 1,
             device: int = 0) -> ScanResult:
    return Projector(ph, resp, device=device).run_scan(g, spec, cfg, angle_subset, what)


def apportion_photons(spec: I.Spectrum, photons_total: int) -> np.ndarray:
    """REF apportion_photons (transport.cpp:42-64)."""
    pk = A.Packed()
    out = np.zeros(spec.n_bins, np.uint64)
    A.check(A.lib().xs_apportion_photons(C.byref(pk.spectrum(spec)), int(photons_total),
                                         out.ctypes.data_as(A.c_u64_p)))
    return out


def history_count(spec: I.Spectrum, photons_total: int) -> int:
    pk = A.Packed()
    n = C.c_uint64()
    A.check(A.lib().xs_history_count(C.byref(pk.spectrum(spec)), int(photons_total),
                                     C.byref(n)))
    return int(n.value)


def point_detector_score(response_factor, p_dir, weight, n_pixels, d2, tau) -> float:
    """REF point_detector_score (transport.cpp:66-71)."""
    return A.lib().xs_point_detector_score(response_factor, p_dir, weight, n_pixels, d2, tau)


def finalize_host(g, spec, cfg, accum: np.ndarray, hist_begin: int, hist_end: int) -> SimResult:
    """Finalize a (reduced) fixed-point accumulator on the host (no GPU)."""
    pk = A.Packed()
    accum = np.ascontiguousarray(accum, dtype=np.uint64)
    img = np.empty(g.nu * g.nv)
    var = np.empty(g.nu * g.nv) if cfg.track_variance else None
    res = A.XsScatterResult()
    res.image = A.dptr(img)
    res.variance = A.dptr(var) if var is not None else None
    A.check(A.lib().xs_scatter_finalize_host(
        C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)), C.byref(pk.config(cfg)),
        accum.ctypes.data_as(A.c_u64_p), hist_begin, hist_end, C.byref(res)))
    return _result(img, var, res, g)


# ------------------------------------------------------------ post-processing
@dataclasses.dataclass
class SgFilterSpec:
    """REF SgFilterSpec (postprocess.hpp:8-11)."""

    window: int = 15
    polyorder: int = 3


def validate_sg_spec(f: SgFilterSpec) -> None:
    A.check(A.lib().xs_validate_sg_spec(f.window, f.polyorder))


def default_sg_spec(nu: int, nv: int) -> SgFilterSpec:
    w, p = C.c_int32(), C.c_int32()
    A.check(A.lib().xs_default_sg_spec(nu, nv, C.byref(w), C.byref(p)))
    return SgFilterSpec(w.value, p.value)


def sg_kernel(left: int, right: int, polyorder: int) -> np.ndarray:
    out = np.empty(left + right + 1)
    A.check(A.lib().xs_sg_kernel(left, right, polyorder, A.dptr(out)))
    return out


def _as_stack(x):
    a = np.ascontiguousarray(x, dtype=np.float64)
    return (a[None], True) if a.ndim == 2 else (a, False)


def sg_smooth(img, f: SgFilterSpec, ctx: Optional[Context] = None) -> np.ndarray:
    """REF sg_smooth (postprocess.cpp:124-145); img (nv, nu) or a stack (n, nv, nu)."""
    ctx = ctx or default_context()
    a, single = _as_stack(img)
    out = np.empty_like(a)
    ctx.check(A.lib().xs_sg_smooth(ctx.h, a.ctypes.data, out.ctypes.data, a.shape[2], a.shape[1],
                                   a.shape[0], f.window, f.polyorder, 0))
    return out[0] if single else out


def interpolate_angles(stack: ProjectionStack, target_angles,
                       ctx: Optional[Context] = None) -> ProjectionStack:
    """REF interpolate_angles (postprocess.cpp:147-196)."""
    ctx = ctx or default_context()
    imgs = np.ascontiguousarray(stack.images, dtype=np.float64)
    src = np.ascontiguousarray(stack.angle_values, dtype=np.float64)
    tgt = np.ascontiguousarray(target_angles, dtype=np.float64)
    n, nv, nu = imgs.shape
    out = np.empty((tgt.size, nv, nu))
    ctx.check(A.lib().xs_interpolate_angles(ctx.h, imgs.ctypes.data, A.dptr(src), n,
                                            out.ctypes.data, A.dptr(tgt), tgt.size, nu, nv, 0))
    return ProjectionStack(tgt.copy(), out)


def upsample_image(img, nu_out: int, nv_out: int, ctx: Optional[Context] = None) -> np.ndarray:
    """REF upsample_image (postprocess.cpp:235-252)."""
    ctx = ctx or default_context()
    a, single = _as_stack(img)
    out = np.empty((a.shape[0], nv_out, nu_out))
    ctx.check(A.lib().xs_upsample_image(ctx.h, a.ctypes.data, a.shape[2], a.shape[1], a.shape[0],
                                        out.ctypes.data, nu_out, nv_out, 0))
    return out[0] if single else out


def downsample_average(img, nu_out: int, nv_out: int, ctx: Optional[Context] = None) -> np.ndarray:
    """REF downsample_average (postprocess.cpp:254-271)."""
    ctx = ctx or default_context()
    a, single = _as_stack(img)
    out = np.empty((a.shape[0], nv_out, nu_out))
    ctx.check(A.lib().xs_downsample_average(ctx.h, a.ctypes.data, a.shape[2], a.shape[1],
                                            a.shape[0], out.ctypes.data, nu_out, nv_out, 0))
    return out[0] if single else out


# ------------------------------------------------------ correction-loop stages
def intensity_to_attenuation(intensity, flatfield, ctx: Optional[Context] = None) -> np.ndarray:
    """REF intensity_to_attenuation (recon.cpp:324-348): a = ln(flat / I) per pixel.
    ``intensity``: (n, nv, nu) stack (or one image); ``flatfield``: (nv, nu)."""
    ctx = ctx or default_context()
    a, single = _as_stack(intensity)
    flat = np.ascontiguousarray(flatfield, dtype=np.float64)
    if flat.shape != a.shape[1:]:
        raise I.XscatError("intensity_to_attenuation: flatfield dims mismatch")
    out = np.empty_like(a)
    ctx.check(A.lib().xs_intensity_to_attenuation(ctx.h, a.ctypes.data, flat.ctypes.data, a.shape[2],
                                                  a.shape[1], a.shape[0], out.ctypes.data, 0))
    return out[0] if single else out


def correct_projections(a, primary, scatter, ctx: Optional[Context] = None):
    """REF correct_projections (correction.cpp:58-86), Eq. 8:
    c = a - ln(Ip / (Ip + max(Is, 0))).  Returns (corrected, clamped_count)."""
    ctx = ctx or default_context()
    sa, single = _as_stack(a)
    sp, _ = _as_stack(primary)
    ss, _ = _as_stack(scatter)
    if sa.shape != sp.shape or sa.shape != ss.shape:
        raise I.XscatError("correct_projections: stack dims mismatch")
    out = np.empty_like(sa)
    clamped = C.c_uint64(0)
    ctx.check(A.lib().xs_correct_projections(ctx.h, sa.ctypes.data, sp.ctypes.data, ss.ctypes.data,
                                             sa.shape[2], sa.shape[1], sa.shape[0], out.ctypes.data,
                                             C.byref(clamped), 0))
    return (out[0] if single else out), int(clamped.value)


def correction_tail(scatter_sub, sub_angles, primary_mc, full_angles, f: SgFilterSpec, a,
                    ctx: Optional[Context] = None):
    """The correction loop's tail after the Monte Carlo runs (REF
    correction.cpp:199-246), fused on the device: SG on the scatter images,
    angle interpolation, Catmull-Rom up-sampling of scatter and primary to the
    size of ``a``, primary floor at 1e-12 of each view's peak, Eq. 8.
    Returns (corrected stack, mean scatter fraction, clamped count)."""
    ctx = ctx or default_context()
    s = np.ascontiguousarray(scatter_sub, dtype=np.float64)
    p = np.ascontiguousarray(primary_mc, dtype=np.float64)
    aa = np.ascontiguousarray(a, dtype=np.float64)
    sa = np.ascontiguousarray(sub_angles, dtype=np.float64)
    fa = np.ascontiguousarray(full_angles, dtype=np.float64)
    n_sub, nv, nu = s.shape
    n_full, nv_out, nu_out = aa.shape
    if p.shape != (n_full, nv, nu) or sa.size != n_sub or fa.size != n_full:
        raise I.XscatError("correction_tail: stack dims mismatch")
    out = np.empty_like(aa)
    frac = C.c_double(0.0)
    clamped = C.c_uint64(0)
    ctx.check(A.lib().xs_correction_tail(ctx.h, s.ctypes.data, sa.ctypes.data, n_sub, p.ctypes.data,
                                         fa.ctypes.data, n_full, nu, nv, f.window, f.polyorder,
                                         aa.ctypes.data, nu_out, nv_out, out.ctypes.data,
                                         C.byref(frac), C.byref(clamped), 0))
    return out, float(frac.value), int(clamped.value)


# -------------------------------------------------------------------- FDK
RAMLAK, HANN = 0, 1


def default_voxel_size(g: I.ScanGeometry, dims) -> np.ndarray:
    """REF default_voxel_size (recon.cpp:13-18)."""
    pk = A.Packed()
    d = (C.c_int32 * 3)(*dims)
    out = np.zeros(3)
    A.lib().xs_default_voxel_size(C.byref(pk.geometry(g)), d, A.dptr(out))
    return out


def fbp_reconstruct(stack: ProjectionStack, g: I.ScanGeometry, dims, voxel_size=None, window: int = HANN,
                    ctx: Optional[Context] = None) -> np.ndarray:
    """REF fbp_reconstruct (recon.cpp:58-157): FDK of an attenuation stack;
    returns the float32 volume (dims[2], dims[1], dims[0]) in 1/m."""
    ctx = ctx or default_context()
    imgs = np.ascontiguousarray(stack.images, dtype=np.float64)
    ang = np.ascontiguousarray(stack.angle_values, dtype=np.float64)
    n, nv, nu = imgs.shape
    vx = np.ascontiguousarray(default_voxel_size(g, dims) if voxel_size is None else voxel_size,
                              dtype=np.float64)
    out = np.empty((dims[2], dims[1], dims[0]), np.float32)
    pk = A.Packed()
    d = (C.c_int32 * 3)(*dims)
    ctx.check(A.lib().xs_fbp_reconstruct(ctx.h, imgs.ctypes.data, A.dptr(ang), n, nu, nv,
                                         C.byref(pk.geometry(g)), d, A.dptr(vx), int(window),
                                         out.ctypes.data, 0))
    return out



# ----------------------------------------------------------- segmentation
# REF recon.hpp:27-53 / recon.cpp:159-322 on the device.
@dataclasses.dataclass
class ClassSpec:
    """REF ClassSpec (recon.hpp:32-35)."""
    material_id: int = 0
    density: float = 0.0


@dataclasses.dataclass
class SegmentationResult:
    """REF SegmentationResult (recon.hpp:37-41); labels shaped like the volume."""
    thresholds: List[float]
    labels: np.ndarray
    class_map: List[ClassSpec]


def _volume(vol) -> np.ndarray:
    v = np.ascontiguousarray(vol, dtype=np.float32)
    if v.ndim != 3:
        raise I.XscatError("volume: expected a (nz, ny, nx) array")
    return v


def otsu_thresholds(vol, n_classes: int, histogram_bins: int = 1024,
                    ctx: Optional[Context] = None) -> List[float]:
    """REF otsu_thresholds (recon.cpp:159-240) of a (nz, ny, nx) float volume."""
    ctx = ctx or default_context()
    v = _volume(vol)
    d = (C.c_int32 * 3)(v.shape[2], v.shape[1], v.shape[0])
    out = np.zeros(max(0, min(int(n_classes), 4) - 1) + 1)
    ctx.check(A.lib().xs_otsu_thresholds(ctx.h, v.ctypes.data, d, int(n_classes), int(histogram_bins),
                                         out.ctypes.data, 0))
    return [float(x) for x in out[:int(n_classes) - 1]]


def segment_volume(vol, thresholds, class_map, ctx: Optional[Context] = None) -> SegmentationResult:
    """REF segment_volume (recon.cpp:242-262)."""
    ctx = ctx or default_context()
    v = _volume(vol)
    thr = np.ascontiguousarray(thresholds, dtype=np.float64).reshape(-1)
    labels = np.empty(v.shape, np.uint8)
    ctx.check(A.lib().xs_segment_volume(ctx.h, v.ctypes.data, v.size, A.dptr(thr), thr.size,
                                        len(class_map), labels.ctypes.data, 0))
    return SegmentationResult([float(x) for x in thr], labels, list(class_map))


def to_density_phantom(vol, voxel_size, seg: SegmentationResult, target_dims, materials,
                       ctx: Optional[Context] = None) -> I.VoxelPhantom:
    """REF to_density_phantom (recon.cpp:264-322): `vol` gives the source
    dims (nz, ny, nx) and `voxel_size` its voxel size (REF Volume); `materials`
    is REF's list without the vacuum entry, which is prepended like REF
    make_empty_phantom does."""
    ctx = ctx or default_context()
    shape = np.shape(vol)
    src = (C.c_int32 * 3)(shape[2], shape[1], shape[0])
    tgt = (C.c_int32 * 3)(*target_dims)
    mats = [None] + [m for m in materials if m is not None]
    pk = A.Packed()
    labels = np.ascontiguousarray(seg.labels, dtype=np.uint8)
    n_out = int(target_dims[0]) * int(target_dims[1]) * int(target_dims[2])
    ids = np.empty(n_out, np.uint8)
    dens = np.empty(n_out, np.float32)
    ctx.check(A.lib().xs_to_density_phantom(ctx.h, labels.ctypes.data, src, pk.class_map(seg.class_map),
                                            len(seg.class_map), tgt, len(mats), pk.materials(mats),
                                            ids.ctypes.data, dens.ctypes.data, 0))
    vs = [float(voxel_size[a]) * shape[2 - a] / int(target_dims[a]) for a in range(3)]
    origin = [(-int(target_dims[a]) * vs[a]) * 0.5 for a in range(3)]
    return I.VoxelPhantom(tuple(target_dims), tuple(vs), tuple(origin), ids, dens, mats)


def segment_to_scene(vol, voxel_size, n_classes: int, class_map, target_dims, materials,
                     response: Optional[I.DetectorResponse] = None, histogram_bins: int = 1024,
                     ctx: Optional[Context] = None) -> List[float]:
    """The loop's segmentation stage (REF correction.cpp:168-171) fused on the
    device: Otsu -> labels -> density phantom, which becomes ctx's scene.
    Returns the thresholds."""
    ctx = ctx or default_context()
    v = _volume(vol)
    d = (C.c_int32 * 3)(v.shape[2], v.shape[1], v.shape[0])
    vs = np.ascontiguousarray(voxel_size, dtype=np.float64)
    tgt = (C.c_int32 * 3)(*target_dims)
    mats = [None] + [m for m in materials if m is not None]
    pk = A.Packed()
    thr = np.zeros(5)
    ctx.check(A.lib().xs_segment_to_scene(ctx.h, v.ctypes.data, d, A.dptr(vs), int(n_classes),
                                          int(histogram_bins), pk.class_map(class_map), tgt, len(mats),
                                          pk.materials(mats), thr.ctypes.data, 0))
    if response is not None:
        ctx.check(A.lib().xs_upload_response(ctx.h, C.byref(pk.response(response))))
    return [float(x) for x in thr[:int(n_classes) - 1]]


# --------------------------------------------------- iterative correction
@dataclasses.dataclass
class CorrectionConfig:
    """REF CorrectionConfig (correction.hpp:13-24), same defaults."""
    n_iterations: int = 3
    simulate_every_kth_angle: int = 2
    mc_nu: int = 0
    mc_nv: int = 0
    recon_dims: tuple = (64, 64, 64)
    n_classes: int = 3
    class_map: list = dataclasses.field(default_factory=list)
    sim: I.SimConfig = dataclasses.field(default_factory=I.SimConfig)
    sg: SgFilterSpec = dataclasses.field(default_factory=lambda: SgFilterSpec(15, 3))
    sg_auto_window: bool = True
    workers: int = 1


@dataclasses.dataclass
class IterationReport:
    """REF IterationReport (correction.hpp:26-39); seconds_postprocess holds
    the fused post-processing + correction pass (seconds_correction = 0)."""
    iteration: int
    seconds_fbp: float
    seconds_segmentation: float
    seconds_mc_scatter: float
    seconds_mc_primary: float
    seconds_postprocess: float
    seconds_correction: float
    seconds_total: float
    mc_seconds_per_projection: float
    mean_scatter_fraction: float
    ncc_to_previous: float
    negative_scatter_clamped: int


@dataclasses.dataclass
class CorrectionResult:
    """REF CorrectionResult (correction.hpp:53-57)."""
    corrected_volume: np.ndarray
    corrected_stack: ProjectionStack
    reports: List[IterationReport]


def reports_from(arr, n) -> List[IterationReport]:
    names = [k for k, _ in A.XsIterationReport._fields_ if k != "pad_"]
    return [IterationReport(**{k: getattr(arr[i], k) for k in names}) for i in range(n)]


def run_iterative_correction(raw_intensity: ProjectionStack, flatfield, g: I.ScanGeometry, spec: I.Spectrum,
                             resp: I.DetectorResponse, cfg: CorrectionConfig, materials,
                             ctx: Optional[Context] = None, group: Optional["Group"] = None) -> CorrectionResult:
    """REF run_iterative_correction (correction.cpp:137-266) with every stage
    on the device; `materials` is REF's list (vacuum prepended here)."""
    raw = np.ascontiguousarray(raw_intensity.images, dtype=np.float64)
    cmap = list(cfg.class_map or [])
    if 2 <= int(cfg.n_classes) <= 4 and len(cmap) != int(cfg.n_classes):
        raise I.XscatError("correction config: class_map must have n_classes entries")
    flat = np.ascontiguousarray(flatfield, dtype=np.float64)
    # the C call reads g.nu * g.nv per image: check the caller's dims first, with
    # REF's messages (recon.cpp:327-328; correction.cpp:60-63 inside stage())
    if flat.shape[-2:] != raw.shape[-2:] or flat.size != raw.shape[-1] * raw.shape[-2]:
        raise I.XscatError("intensity_to_attenuation: flatfield dims mismatch")
    if raw.shape[0] != g.n_angles:
        raise I.XscatError("run_iterative_correction: stack angle count mismatch")
    if raw.shape[1:] != (g.nv, g.nu):
        raise I.XscatError("iteration 1, stage correction: correct_projections: stack dims mismatch")
    mats = [None] + [m for m in materials if m is not None]
    pk = A.Packed()
    vol = np.empty(tuple(int(d) for d in cfg.recon_dims[::-1]), np.float32)
    stack = np.empty_like(raw)
    reps = (A.XsIterationReport * max(1, int(cfg.n_iterations)))()
    args = (raw.ctypes.data, flat.ctypes.data, C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
            C.byref(pk.correction_config(cfg)), len(mats), pk.materials(mats), vol.ctypes.data,
            stack.ctypes.data, reps, 0)
    if group is not None:  # the loop's scans sharded by angle over the group's GPUs
        group.check(A.lib().xs_group_upload_response(group.h, C.byref(pk.response(resp))))
        group.check(A.lib().xs_group_run_iterative_correction(group.h, *args))
    else:
        ctx = ctx or default_context()
        ctx.check(A.lib().xs_upload_response(ctx.h, C.byref(pk.response(resp))))
        ctx.check(A.lib().xs_run_iterative_correction(ctx.h, *args))
    return CorrectionResult(vol, ProjectionStack(list(raw_intensity.angle_values), stack),
                            reports_from(reps, int(cfg.n_iterations)))
