"""The C-ABI library on a machine without a GPU: it loads, exports every
symbol include/xscat_gpu.h declares, and its host-only functions (photon
apportioning, SG weights, tally finalize, validation) agree with the oracle.
No compute call needs a device here."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A
from paper_2201_13191_b200 import inputs as I
import cases

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "xscat_gpu.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int32_t|void|double|const char\*|xs_context\*|const xs_\w+\*)\s+(xs_\w+)\(",
                              header, re.M))
    assert len(declared) >= 80
    L = A.lib()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert set(A.SIGNATURES) <= declared | set()  # every binding is a declared symbol


def test_version_and_defaults():
    L = A.lib()
    assert L.xs_abi_version() == 1
    assert b"sm_100a" in L.xs_version()
    c = A.XsSimConfig()
    L.xs_sim_config_default(C.byref(c))
    d = I.SimConfig()
    assert (c.photons_total, c.splitting, c.roulette_survival, c.roulette_wmin_rel,
            c.step_voxels, c.max_interactions, c.seed) == (
        d.photons_total, d.splitting, d.roulette_survival, d.roulette_wmin_rel,
        d.step_voxels, d.max_interactions, d.seed)


def test_apportion_matches_oracle(orc):
    for spec, n in ((I.kramers_spectrum(150.0), 10**8), (cases.mixed_spectrum(), 1000),
                    (I.spectrum("w200kv_2mmal"), 12345), (I.monochromatic_spectrum(60.0), 7)):
        assert np.array_equal(X.apportion_photons(spec, n), orc.apportion(spec, n))
        assert X.history_count(spec, n) == int(orc.apportion(spec, n).sum())


def test_sg_kernel_bit_exact_vs_oracle(orc):
    for left in range(8):
        for right in range(8):
            for order in (2, 3):
                assert np.array_equal(X.sg_kernel(left, right, order), orc.sg_kernel(left, right, order))
    assert X.default_sg_spec(576, 800).window == 15
    assert X.default_sg_spec(16, 16).window == 5
    with pytest.raises(X.XscatError, match="window must be odd"):
        X.projector.validate_sg_spec(X.SgFilterSpec(6, 3))


def test_point_detector_score_properties():
    """REF test_transport.cpp:69-81."""
    x = X.point_detector_score(0.8, 0.2, 1.5, 64.0, 100.0, 0.7)
    assert X.point_detector_score(0.8, 0.2, 0.0, 64.0, 100.0, 0.7) == 0.0
    assert X.point_detector_score(0.8, 0.2, 3.0, 64.0, 100.0, 0.7) == pytest.approx(2 * x, rel=1e-15)
    assert X.point_detector_score(0.8, 0.2, 1.5, 64.0, 400.0, 0.7) == pytest.approx(0.25 * x, rel=1e-15)
    assert X.point_detector_score(0.8, 0.2, 1.5, 64.0, 100.0, 1.7) == pytest.approx(x * np.exp(-1.0), rel=1e-14)


def test_config_validation_maps_to_reference_errors():
    L = A.lib()
    for kw, msg in (({"photons_total": 0}, "photons_total must be >= 1"),
                    ({"splitting": 0}, "splitting must be >= 1"),
                    ({"roulette_survival": 0.0}, "roulette_survival must lie in (0,1]"),
                    ({"step_voxels": 0}, "step_voxels must be >= 1")):
        pk = A.Packed()
        st = L.xs_validate_sim_config(C.byref(pk.config(I.SimConfig(**kw))))
        assert st == 1  # XS_E_RUNTIME <-> std::runtime_error
        assert msg in L.xs_last_error(None).decode()


def test_finalize_host_matches_reference_mode(orc):
    """Fixed-point tallies of the oracle finalized by the product's host code
    agree with the reference's fp64 chunked reduction."""
    for name in ("crit2", "poly1"):
        ph, g, angle, spec, resp, cfg = cases.SCATTER_CASES[name]()
        L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
        n = X.history_count(spec, cfg.photons_total)
        acc = np.zeros(L["words"], np.uint64)
        orc.accumulate_range(ph, g, angle, spec, resp, cfg, 0, n, acc)
        got = X.finalize_host(g, spec, cfg, acc, 0, n)
        want = orc.simulate_scatter_stats(ph, g, angle, spec, resp, cfg)
        assert got.histories == want["histories"] == n
        nz = want["image"] > 0
        assert np.max(np.abs(got.image[nz] - want["image"][nz]) / want["image"][nz]) < 1e-12
        assert np.all(got.image[~nz] == 0)
        assert got.total == pytest.approx(want["total"], rel=1e-12)
        assert got.total_std_error == pytest.approx(want["total_std_error"], rel=1e-9)
        for k in ("initial", "escaped", "absorbed", "culled", "roulette_killed", "roulette_boost"):
            assert getattr(got.ledger, k) == pytest.approx(want["ledger"][k], rel=1e-12, abs=1e-300)
        if cfg.track_variance:
            nzv = want["variance"] > 0
            assert np.max(np.abs(got.variance[nzv] - want["variance"][nzv]) / want["variance"][nzv]) < 1e-9


def test_history_range_splits_are_bit_identical(orc):
    """The multi-GPU contract: integer limb sums over any split of the
    history range equal the single-range accumulator exactly."""
    ph, g, angle, spec, resp, cfg = cases.poly(1)
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
    n = X.history_count(spec, cfg.photons_total)
    full = np.zeros(L["words"], np.uint64)
    orc.accumulate_range(ph, g, angle, spec, resp, cfg, 0, n, full)
    for parts in (2, 3, 8):
        acc = np.zeros(L["words"], np.uint64)
        for r in range(parts):
            part = np.zeros(L["words"], np.uint64)
            orc.accumulate_range(ph, g, angle, spec, resp, cfg, n * r // parts, n * (r + 1) // parts, part)
            acc += part
        assert np.array_equal(acc, full)


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(X.XscatError):
        X.Context(0)


def test_correction_loop_rejects_mismatched_dims_before_the_device():
    """The C loop reads g.nu*g.nv per image: the Python mirror checks the
    caller's stack / flat-field / class_map sizes first with REF's messages
    (recon.cpp:327-328, correction.cpp:40-42, :60-63, :133-134)."""
    g = I.make_circular_geometry(60.0, 40.0, 8, 6, 0.5, 4)
    spec, resp = I.monochromatic_spectrum(60.0), I.detector_response()
    ok = X.CorrectionConfig(n_classes=2, class_map=[X.ClassSpec(0, 0.0), X.ClassSpec(1, 1.0)])
    good = X.ProjectionStack(list(g.angles), np.ones((4, 6, 8)))
    with pytest.raises(X.XscatError, match="flatfield dims mismatch"):
        X.run_iterative_correction(good, np.ones((6, 7)), g, spec, resp, ok, [I.material("water")])
    with pytest.raises(X.XscatError, match="stack angle count mismatch"):
        X.run_iterative_correction(X.ProjectionStack(list(g.angles[:3]), np.ones((3, 6, 8))), np.ones((6, 8)),
                                   g, spec, resp, ok, [I.material("water")])
    with pytest.raises(X.XscatError, match="stack dims mismatch"):
        X.run_iterative_correction(X.ProjectionStack(list(g.angles), np.ones((4, 5, 8))), np.ones((5, 8)),
                                   g, spec, resp, ok, [I.material("water")])
    short = X.CorrectionConfig(n_classes=3, class_map=[X.ClassSpec(0, 0.0)])
    with pytest.raises(X.XscatError, match="class_map must have n_classes entries"):
        X.run_iterative_correction(good, np.ones((6, 8)), g, spec, resp, short, [I.material("water")])
