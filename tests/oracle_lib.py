"""ctypes bindings of the TEST-ONLY oracles.

- ``oracle()``: oracle/liboracle.so, the plain-C restatement (always built).
- ``ref()``: oracle/_ref/libxscat_ref.so, the unmodified reference library
  compiled from /root/reference (present when built in the build container;
  the prebuilt .so travels to GPU boxes).  ``None`` when absent.

Both take the xs_* structs of include/xscat_gpu.h, packed by
paper_2201_13191_b200._capi.Packed.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

from paper_2201_13191_b200 import _capi as A
from paper_2201_13191_b200 import inputs as I

ROOT = pathlib.Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libxscat_ref.so"

_P = C.c_void_p
_dp = A.c_double_p
_ph = C.POINTER(A.XsPhantom)
_g = C.POINTER(A.XsGeometry)
_s = C.POINTER(A.XsSpectrum)
_r = C.POINTER(A.XsResponse)
_c = C.POINTER(A.XsSimConfig)
_res = C.POINTER(A.XsScatterResult)
_m = C.POINTER(A.XsMaterial)


def _sig(L, prefix):
    p = prefix
    sigs = {
        f"{p}_simulate_scatter_stats": (C.c_int, [_ph, _g, C.c_int32, _s, _r, _c, C.c_int32, _res]),
        f"{p}_simulate_primary": (C.c_int, [_ph, _g, C.c_int32, _s, _r, _c, C.c_int32, _dp]),
        f"{p}_apportion_photons": (C.c_int, [_s, C.c_uint64, A.c_u64_p]),
        f"{p}_trace_attenuation": (C.c_int, [_ph, _dp, _dp, C.c_double, C.c_int32, _dp]),
        f"{p}_trace_rho_lengths": (C.c_int, [_ph, _dp, _dp, _dp]),
        f"{p}_sample_free_path": (C.c_int, [_ph, _dp, _dp, C.c_double, C.c_double,
                                            C.POINTER(C.c_int32), _dp, C.POINTER(C.c_int32)]),
        f"{p}_p_lambda": (C.c_int, [_m, C.c_int32, C.c_double, C.c_double, _dp]),
        f"{p}_sample_compton": (C.c_int, [_m, C.c_double, C.c_uint64, C.c_int64, _dp, _dp, _dp]),
        f"{p}_sample_rayleigh": (C.c_int, [_m, C.c_double, C.c_uint64, C.c_int64, _dp, _dp]),
        f"{p}_f2_q2_cdf": (C.c_int, [_m, _dp]),
        f"{p}_rng_uniform": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int64, _dp]),
        f"{p}_sg_kernel": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _dp]),
        f"{p}_default_sg_spec": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32)]),
        f"{p}_sg_smooth": (C.c_int, [_dp, _dp, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
        f"{p}_interpolate_angles": (C.c_int, [_dp, _dp, C.c_int32, _dp, _dp, C.c_int32,
                                              C.c_int32, C.c_int32]),
        f"{p}_upsample_image": (C.c_int, [_dp, C.c_int32, C.c_int32, _dp, C.c_int32, C.c_int32]),
        f"{p}_downsample_average": (C.c_int, [_dp, C.c_int32, C.c_int32, _dp, C.c_int32,
                                              C.c_int32]),
        f"{p}_intensity_to_attenuation": (C.c_int, [_dp, _dp, C.c_int32, C.c_int32, C.c_int32, _dp]),
        f"{p}_correct_projections": (C.c_int, [_dp, _dp, _dp, C.c_int32, C.c_int32, C.c_int32, _dp,
                                               A.c_u64_p]),
        f"{p}_correction_tail": (C.c_int, [_dp, _dp, C.c_int32, _dp, _dp, C.c_int32, C.c_int32,
                                           C.c_int32, C.c_int32, C.c_int32, _dp, C.c_int32,
                                           C.c_int32, _dp, _dp, A.c_u64_p]),
        f"{p}_fbp_reconstruct": (C.c_int, [_dp, _dp, C.c_int32, C.c_int32, C.c_int32, _g,
                                           C.POINTER(C.c_int32), _dp, C.c_int32, C.c_void_p]),
        f"{p}_otsu_thresholds": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                           _dp]),
        f"{p}_segment_volume": (C.c_int, [C.c_void_p, C.c_uint64, _dp, C.c_int32, C.c_int32,
                                          C.c_void_p]),
        f"{p}_to_density_phantom": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32),
                                              C.POINTER(A.XsClassSpec), C.c_int32,
                                              C.POINTER(C.c_int32), C.c_int32, _m, C.c_void_p,
                                              C.c_void_p]),
        f"{p}_last_error": (C.c_char_p, []),
    }
    if prefix == "xo":
        sigs["xo_scatter_accumulate_range"] = (C.c_int, [_ph, _g, C.c_int32, _s, _r, _c,
                                                         C.c_uint64, C.c_uint64, A.c_u64_p])
    else:
        sigs.update({
            "xr_analog_scatter": (C.c_int, [_ph, _g, C.c_int32, _s, _r, C.c_uint64, C.c_uint64,
                                            _dp, _dp, _dp]),
            "xr_trace_sorted_crossings": (C.c_int, [_ph, _dp, _dp, C.c_double, _dp]),
            "xr_run_iterative_correction": (C.c_int, [_dp, _dp, _g, _s, _r,
                                                      C.POINTER(A.XsCorrectionConfig), C.c_int32, _m,
                                                      C.c_void_p, C.c_void_p,
                                                      C.POINTER(A.XsIterationReport), C.c_int32]),
            "xr_make_phantom": (C.c_int, [C.c_int32, C.c_int32, C.c_double, _dp, C.c_double,
                                          C.POINTER(C.c_int32), _dp, _dp,
                                          C.POINTER(C.c_uint8), C.POINTER(C.c_float)]),
            "xr_scene_create": (_P, [_ph, _r]),
            "xr_scene_destroy": (None, [_P]),
            "xr_scene_simulate_scatter": (C.c_int, [_P, _g, C.c_int32, _s, _c, C.c_int32, _res]),
            "xr_scene_simulate_primary": (C.c_int, [_P, _g, C.c_int32, _s, _c, C.c_int32, _dp]),
        })
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


class Oracle:
    """Uniform Python face over either library (prefix xo_ or xr_)."""

    def __init__(self, path, prefix):
        self.L = C.CDLL(str(path))
        self.p = prefix
        _sig(self.L, prefix)

    def fn(self, name):
        return getattr(self.L, f"{self.p}_{name}")

    def check(self, st):
        if st != 0:
            msg = self.fn("last_error")().decode(errors="replace")
            raise {2: I.XscatOutOfRange, 3: I.XscatInvalidArgument,
                   4: I.XscatDomainError}.get(st, I.XscatError)(msg)

    # ---------------------------------------------------------- transport
    def simulate_scatter_stats(self, ph, g, angle, spec, resp, cfg, workers=8):
        pk = A.Packed()
        img = np.zeros(g.nu * g.nv)
        var = np.zeros(g.nu * g.nv) if cfg.track_variance else None
        res = A.XsScatterResult()
        res.image = A.dptr(img)
        res.variance = A.dptr(var) if var is not None else None
        self.check(self.fn("simulate_scatter_stats")(
            pk.phantom(ph), pk.geometry(g), angle, pk.spectrum(spec), pk.response(resp),
            pk.config(cfg), workers, C.byref(res)))
        return dict(image=img.reshape(g.nv, g.nu),
                    variance=None if var is None else var.reshape(g.nv, g.nu),
                    ledger={k: getattr(res.ledger, k) for k, _ in A.XsLedger._fields_},
                    histories=res.histories, total=res.total,
                    total_std_error=res.total_std_error)

    def simulate_primary(self, ph, g, angle, spec, resp, cfg=None, workers=8):
        pk = A.Packed()
        img = np.zeros(g.nu * g.nv)
        self.check(self.fn("simulate_primary")(pk.phantom(ph), pk.geometry(g), angle,
                                               pk.spectrum(spec), pk.response(resp),
                                               pk.config(cfg or I.SimConfig()), workers,
                                               A.dptr(img)))
        return img.reshape(g.nv, g.nu)

    def accumulate_range(self, ph, g, angle, spec, resp, cfg, h0, h1, accum):
        pk = A.Packed()
        self.check(self.L.xo_scatter_accumulate_range(
            pk.phantom(ph), pk.geometry(g), angle, pk.spectrum(spec), pk.response(resp),
            pk.config(cfg), h0, h1, accum.ctypes.data_as(A.c_u64_p)))

    def apportion(self, spec, n):
        pk = A.Packed()
        out = np.zeros(spec.n_bins, np.uint64)
        self.check(self.fn("apportion_photons")(pk.spectrum(spec), n,
                                                out.ctypes.data_as(A.c_u64_p)))
        return out

    # ------------------------------------------------------------ tracing
    def trace_attenuation(self, ph, o, d, e, step=1):
        pk = A.Packed()
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        tau = C.c_double()
        self.check(self.fn("trace_attenuation")(pk.phantom(ph), A.dptr(o), A.dptr(d), e, step,
                                                C.byref(tau)))
        return tau.value

    def sample_free_path(self, ph, o, d, e, u):
        pk = A.Packed()
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        esc = C.c_int32()
        pt = np.zeros(3)
        vox = (C.c_int32 * 3)()
        self.check(self.fn("sample_free_path")(pk.phantom(ph), A.dptr(o), A.dptr(d), e, u,
                                               C.byref(esc), A.dptr(pt), vox))
        return bool(esc.value), pt, tuple(vox)

    # ----------------------------------------------------------- samplers
    def sample_compton(self, m, e, seed, n):
        pk = A.Packed()
        mm = A.XsMaterial()
        pk.material(m, mm)
        th, ph_, ap = np.zeros(n), np.zeros(n), np.zeros(n)
        self.check(self.fn("sample_compton")(C.byref(mm), e, seed, n, A.dptr(th), A.dptr(ph_),
                                             A.dptr(ap)))
        return th, ph_, ap

    def sample_rayleigh(self, m, e, seed, n):
        pk = A.Packed()
        mm = A.XsMaterial()
        pk.material(m, mm)
        th, ph_ = np.zeros(n), np.zeros(n)
        self.check(self.fn("sample_rayleigh")(C.byref(mm), e, seed, n, A.dptr(th), A.dptr(ph_)))
        return th, ph_

    def p_lambda(self, m, compton, e, theta):
        pk = A.Packed()
        mm = A.XsMaterial()
        pk.material(m, mm)
        p = C.c_double()
        self.check(self.fn("p_lambda")(C.byref(mm), int(compton), e, theta, C.byref(p)))
        return p.value

    def f2_q2_cdf(self, m):
        pk = A.Packed()
        mm = A.XsMaterial()
        pk.material(m, mm)
        out = np.zeros(len(m.f_factor))
        self.check(self.fn("f2_q2_cdf")(C.byref(mm), A.dptr(out)))
        return out

    def rng_uniform(self, seed, angle, b, photon, n):
        out = np.zeros(n)
        self.fn("rng_uniform")(seed, angle, b, photon, n, A.dptr(out))
        return out

    # -------------------------------------------------------- postprocess
    def sg_kernel(self, left, right, order):
        out = np.zeros(left + right + 1)
        self.check(self.fn("sg_kernel")(left, right, order, A.dptr(out)))
        return out

    def default_sg_spec(self, nu, nv):
        w, p = C.c_int32(), C.c_int32()
        self.fn("default_sg_spec")(nu, nv, C.byref(w), C.byref(p))
        return w.value, p.value

    def sg_smooth(self, img, window, order):
        img = np.ascontiguousarray(img, np.float64)
        out = np.zeros_like(img)
        nv, nu = img.shape
        self.check(self.fn("sg_smooth")(A.dptr(img), A.dptr(out), nu, nv, window, order))
        return out

    def interpolate_angles(self, stack, src, tgt):
        stack = np.ascontiguousarray(stack, np.float64)
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        n, nv, nu = stack.shape
        out = np.zeros((tgt.size, nv, nu))
        self.check(self.fn("interpolate_angles")(A.dptr(stack), A.dptr(src), n, A.dptr(out),
                                                 A.dptr(tgt), tgt.size, nu, nv))
        return out

    def upsample_image(self, img, nu_out, nv_out):
        img = np.ascontiguousarray(img, np.float64)
        nv, nu = img.shape
        out = np.zeros((nv_out, nu_out))
        self.check(self.fn("upsample_image")(A.dptr(img), nu, nv, A.dptr(out), nu_out, nv_out))
        return out

    def downsample_average(self, img, nu_out, nv_out):
        img = np.ascontiguousarray(img, np.float64)
        nv, nu = img.shape
        out = np.zeros((nv_out, nu_out))
        self.check(self.fn("downsample_average")(A.dptr(img), nu, nv, A.dptr(out), nu_out,
                                                 nv_out))
        return out


    # correction-loop stages (REF recon.cpp:324-348, correction.cpp:58-86, :199-246)
    def intensity_to_attenuation(self, intensity, flat):
        x = np.ascontiguousarray(intensity, np.float64)
        f = np.ascontiguousarray(flat, np.float64)
        n, nv, nu = x.shape
        out = np.zeros_like(x)
        self.check(self.fn("intensity_to_attenuation")(A.dptr(x), A.dptr(f), nu, nv, n, A.dptr(out)))
        return out

    def correct_projections(self, a, primary, scatter):
        a = np.ascontiguousarray(a, np.float64)
        p = np.ascontiguousarray(primary, np.float64)
        s = np.ascontiguousarray(scatter, np.float64)
        n, nv, nu = a.shape
        out = np.zeros_like(a)
        cl = C.c_uint64(0)
        self.check(self.fn("correct_projections")(A.dptr(a), A.dptr(p), A.dptr(s), nu, nv, n, A.dptr(out),
                                                  C.byref(cl)))
        return out, int(cl.value)

    def correction_tail(self, scatter_sub, sub_angles, primary_mc, full_angles, window, order, a):
        s = np.ascontiguousarray(scatter_sub, np.float64)
        p = np.ascontiguousarray(primary_mc, np.float64)
        a = np.ascontiguousarray(a, np.float64)
        sa = np.ascontiguousarray(sub_angles, np.float64)
        fa = np.ascontiguousarray(full_angles, np.float64)
        n_sub, nv, nu = s.shape
        n_full, nv_out, nu_out = a.shape
        out = np.zeros_like(a)
        frac = C.c_double(0.0)
        cl = C.c_uint64(0)
        self.check(self.fn("correction_tail")(A.dptr(s), A.dptr(sa), n_sub, A.dptr(p), A.dptr(fa), n_full, nu,
                                              nv, window, order, A.dptr(a), nu_out, nv_out, A.dptr(out),
                                              C.byref(frac), C.byref(cl)))
        return out, float(frac.value), int(cl.value)


    def fbp_reconstruct(self, stack, angles, g, dims, voxel, hann=True):
        from paper_2201_13191_b200 import _capi as A_
        st = np.ascontiguousarray(stack, np.float64)
        an = np.ascontiguousarray(angles, np.float64)
        n, nv, nu = st.shape
        d = (C.c_int32 * 3)(*dims)
        vx = np.ascontiguousarray(voxel, np.float64)
        out = np.zeros((dims[2], dims[1], dims[0]), np.float32)
        pk = A_.Packed()
        self.check(self.fn("fbp_reconstruct")(A.dptr(st), A.dptr(an), n, nu, nv, C.byref(pk.geometry(g)), d,
                                              A.dptr(vx), 1 if hann else 0, out.ctypes.data))
        return out


    # ------------------------------------------------------- segmentation
    def otsu_thresholds(self, vol, n_classes, bins=1024):
        v = np.ascontiguousarray(vol, np.float32)
        d = (C.c_int32 * 3)(v.shape[2], v.shape[1], v.shape[0])
        out = np.zeros(4)
        self.check(self.fn("otsu_thresholds")(v.ctypes.data, d, n_classes, bins, A.dptr(out)))
        return [float(x) for x in out[:n_classes - 1]]

    def segment_volume(self, vol, thresholds, n_class_map):
        v = np.ascontiguousarray(vol, np.float32)
        thr = np.ascontiguousarray(thresholds, np.float64).reshape(-1)
        labels = np.empty(v.shape, np.uint8)
        self.check(self.fn("segment_volume")(v.ctypes.data, v.size, A.dptr(thr), thr.size, n_class_map,
                                             labels.ctypes.data))
        return labels

    def to_density_phantom(self, labels, class_map, target_dims, materials):
        """materials: REF list without vacuum (None entries dropped)."""
        lab = np.ascontiguousarray(labels, np.uint8)
        src = (C.c_int32 * 3)(lab.shape[2], lab.shape[1], lab.shape[0])
        tgt = (C.c_int32 * 3)(*target_dims)
        mats = [None] + [m for m in materials if m is not None]
        pk = A.Packed()
        n = int(np.prod(target_dims))
        ids = np.empty(n, np.uint8)
        dens = np.empty(n, np.float32)
        self.check(self.fn("to_density_phantom")(lab.ctypes.data, src, pk.class_map(class_map),
                                                 len(class_map), tgt, len(mats), pk.materials(mats),
                                                 ids.ctypes.data, dens.ctypes.data))
        return ids, dens


    def run_iterative_correction(self, raw, flat, g, spec, resp, cfg, materials, workers=8):
        """REF run_iterative_correction (xr_ only); returns (volume, stack, reports)."""
        from paper_2201_13191_b200 import projector as P
        raw = np.ascontiguousarray(raw, np.float64)
        flat = np.ascontiguousarray(flat, np.float64)
        mats = [None] + [m for m in materials if m is not None]
        pk = A.Packed()
        vol = np.empty(tuple(int(d) for d in cfg.recon_dims[::-1]), np.float32)
        stack = np.empty_like(raw)
        reps = (A.XsIterationReport * cfg.n_iterations)()
        self.check(self.fn("run_iterative_correction")(
            A.dptr(raw), A.dptr(flat), C.byref(pk.geometry(g)), C.byref(pk.spectrum(spec)),
            C.byref(pk.response(resp)), C.byref(pk.correction_config(cfg)), len(mats),
            pk.materials(mats), vol.ctypes.data, stack.ctypes.data, reps, workers))
        return vol, stack, P.reports_from(reps, cfg.n_iterations)


_oracle = None
_ref = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle(ORACLE_SO, "xo")
    return _oracle


def ref():
    """The compiled reference, or None when oracle/_ref was not built."""
    global _ref
    if _ref is None and REF_SO.exists():
        _ref = Oracle(REF_SO, "xr")
    return _ref
