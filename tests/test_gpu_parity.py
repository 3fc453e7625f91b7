"""GPU parity: libxscatgpu.so (through the C ABI) vs the CPU oracle.

The oracle (oracle/liboracle.so) is the plain-C restatement of the reference,
pinned bit-exact to the compiled reference in tests/test_oracle.py.

Tolerances
- primary: |gpu - cpu| / cpu <= 1e-12 per pixel (north_star bar: 1e-5); the
  device walk is the reference's fp64 arithmetic, only exp() differs in ulps.
- scatter, same seed ("replay"): the device runs each history with the
  reference's arithmetic and RNG stream, so per-pixel values agree to
  rounding (<= 1e-9 relative, image total <= 1e-11) unless a last-ulp libm
  difference flips a branch; we allow at most 1e-3 of the pixels to differ
  by more than 1e-9 relative.
- scatter, independent seeds: MC-statistical: total within
  3 combined standard errors, fraction(|z| > 3) <= 2 * 0.27 %, squared L2
  difference <= 1.2 * sum of variances.
"""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["exact-wave", "macro-wave", "exact-mega", "macro-mega"])
def walk_mode(request):
    """exact: voxel-by-voxel Siddon (strict REF replay); macro: uniform
    blocks crossed in one step (fp64-rounding-level change; the default
    walk_mode 2 picks one of the two per phantom).  wave: the wavefront engine (default); mega: the persistent
    megakernel."""
    mode, engine = request.param.split("-")
    ctx = X.projector.default_context(0)
    ctx.set_option("exact_walk", 1 if mode == "exact" else 0)
    ctx.set_option("engine", 1 if engine == "wave" else 0)
    yield request.param
    ctx.set_option("walk_mode", 2)
    ctx.set_option("engine", 1)


def _crit2():
    w = I.material("water")
    ph = S.make_cube_phantom(32, 0.2, 6.4, w, 1.0)
    g = I.make_circular_geometry(60.0, 40.0, 24, 24, 0.55, 1)
    return ph, g


def _rods(n=48):
    return S.make_rods_phantom(n, 10.0 / n, 4.5, 8.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                               I.material("iron"), 7.874)


def test_primary_matches_oracle_c1(orc):
    w = X.configs.c1(photons=1000)
    proj = X.Projector(w.phantom, w.response)
    gpu = proj.primary(w.geometry, 0, w.spectrum, w.config)
    cpu = orc.simulate_primary(w.phantom, w.geometry, 0, w.spectrum, w.response, w.config)
    assert np.all(cpu > 0)
    rel = np.abs(gpu - cpu) / cpu
    assert rel.max() <= 1e-12, rel.max()


def test_primary_polyenergetic_two_materials(orc):
    ph = _rods()
    g = I.make_circular_geometry(128.2, 86.2, 64, 48, 0.3, 8)
    spec = I.kramers_spectrum(150.0)
    resp = I.detector_response()
    proj = X.Projector(ph, resp)
    for a in (0, 3, 5):
        gpu = proj.primary(g, a, spec)
        cpu = orc.simulate_primary(ph, g, a, spec, resp)
        assert np.max(np.abs(gpu - cpu) / cpu) <= 1e-12


def test_primary_beer_lambert_criterion3():
    """REF acceptance criterion 3 (acceptance_main.cpp:162-211): rel err < 1e-6."""
    resp = I.detector_response()
    worst = 0.0
    for m, rho, thick, e in ((I.material("water"), 1.0, 4.0, 100.0),
                             (I.material("aluminum"), 2.699, 2.0, 60.0)):
        n = 32
        ph = I.make_empty_phantom(n, n, n, (thick / 16.0, 0.6, 0.6), [m])
        ids = ph.material_id.reshape(n, n, n)
        ids[:, :, 8:24] = 1
        ph.density.reshape(n, n, n)[:, :, 8:24] = np.float32(rho)
        g = I.make_circular_geometry(60.0, 40.0, 32, 32, 0.45, 1)
        img = X.simulate_primary(ph, g, 0, I.monochromatic_spectrum(e), resp)
        mu = I.mu_at(m, e, rho)
        src = g.source_position(0)
        for iv in range(g.nv):
            for iu in range(g.nu):
                d = g.pixel_position(0, iu, iv) - src
                d2 = float(d @ d)
                cos_x = abs(d[0]) / np.sqrt(d2)
                expect = resp.response_factor(e) / d2 * np.exp(-mu * thick / cos_x)
                worst = max(worst, abs(img[iv, iu] - expect) / expect)
    assert worst < 1e-6, worst


def tally_quantum(g, spec):
    """Resolution of the device's fixed-point image tallies: 2^-64 U_img,
    U_img = 2^floor(log2(sum_b w_b / sdd^2)) (include/xscat_gpu.h
    xs_accum_units_make); each score rounds to it (limb0 round-half-even)."""
    import math
    return math.ldexp(1.0, math.frexp(float(np.sum(spec.weight)) / g.sdd ** 2)[1] - 1 - 64)


def _replay_compare(gpu, cpu, frac_tol=1e-3, quantum=0.0):
    """Same-seed replay: per pixel |gpu - cpu| <= 1e-9 |cpu| + atol, where
    atol = 1024 tally quanta (2^-64 U_img, ~5e-17 of the flat field per
    pixel; pass `quantum` = tally_quantum(g, spec)).  Scores far below the
    quantum (rays through centimetres of iron, exp(-tau) < 1e-20) cannot be
    represented by the fixed-point tally, so such pixels are compared in
    absolute terms.  At most frac_tol of the pixels may exceed the bound (a
    last-ulp libm difference can flip a branch of one history)."""
    a, b = gpu.image, cpu["image"]
    assert gpu.histories == cpu["histories"]
    assert abs(gpu.total - cpu["total"]) <= 1e-11 * abs(cpu["total"]) + 1e-300 or \
        abs(gpu.total - cpu["total"]) <= 1e-6 * abs(cpu["total"])
    atol = 1024.0 * quantum
    nz = b > 0
    bad = np.abs(a[nz] - b[nz]) > 1e-9 * b[nz] + atol
    assert np.mean(bad) <= frac_tol, (np.mean(bad), (np.abs(a[nz] - b[nz]) / b[nz]).max())
    assert np.all(np.abs(a[~nz]) <= atol)
    for k in ("initial", "escaped", "absorbed", "culled", "roulette_killed", "roulette_boost"):
        x, y = getattr(gpu.ledger, k), cpu["ledger"][k]
        assert abs(x - y) <= 1e-9 * max(abs(y), 1e-300) or abs(x - y) <= 1e-6 * abs(y), (k, x, y)


def test_scatter_replay_criterion2(orc, walk_mode):
    """Acceptance criterion 2 inputs (acceptance_main.cpp:128-158), same seed:
    total 0.000496451 (proj/test_output.txt:31)."""
    ph, g = _crit2()
    spec, resp = I.monochromatic_spectrum(100.0), I.detector_response()
    cfg = I.SimConfig(photons_total=100000, splitting=10, seed=424242)
    gpu = X.simulate_scatter_stats(ph, g, 0, spec, resp, cfg)
    cpu = orc.simulate_scatter_stats(ph, g, 0, spec, resp, cfg)
    _replay_compare(gpu, cpu)
    assert abs(gpu.total - 0.000496451) < 1e-9
    assert abs(gpu.total_std_error - cpu["total_std_error"]) <= 1e-9 * cpu["total_std_error"]


@pytest.mark.parametrize("step", [1, 3])
def test_scatter_replay_polyenergetic_roulette_variance(orc, step, walk_mode):
    ph = _rods(32)
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=30000, splitting=5, seed=777, step_voxels=step,
                      roulette_wmin_rel=2.0, roulette_survival=0.6, track_variance=True)
    proj = X.Projector(ph, resp)
    gpu = proj.scatter_stats(g, 2, spec, cfg)
    cpu = orc.simulate_scatter_stats(ph, g, 2, spec, resp, cfg)
    _replay_compare(gpu, cpu)
    nz = cpu["variance"] > 0
    rel = np.abs(gpu.variance[nz] - cpu["variance"][nz]) / cpu["variance"][nz]
    assert np.mean(rel > 1e-6) <= 1e-3


def test_scatter_bit_identical_runs_and_splits(walk_mode):
    """Fixed-point tallies: identical bits for repeated runs and any split of
    the history range (the multi-GPU photon-batch contract)."""
    import torch
    ph, g = _crit2()
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=4, seed=99, track_variance=True)
    proj = X.Projector(ph, resp)
    a = proj.scatter_stats(g, 0, spec, cfg)
    b = proj.scatter_stats(g, 0, spec, cfg)
    assert np.array_equal(a.image, b.image) and a.total == b.total
    from paper_2201_13191_b200 import _capi as A
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, True)
    n = X.history_count(spec, cfg.photons_total)
    for parts in (2, 3, 8):
        bufs = []
        for r in range(parts):
            buf = torch.zeros(L["words"], dtype=torch.int64, device="cuda")
            proj.accumulate(g, 0, spec, cfg, n * r // parts, n * (r + 1) // parts, buf.data_ptr())
            bufs.append(buf)
        total = torch.stack(bufs).sum(0)
        torch.cuda.synchronize()
        c = proj.finalize(g, spec, cfg, total.data_ptr(), 0, n)
        assert np.array_equal(a.image, c.image), parts
        assert np.array_equal(a.variance, c.variance)
        assert a.total == c.total and a.total_std_error == c.total_std_error
        assert a.ledger == c.ledger


def test_scatter_statistical_independent_seeds(orc):
    """SURVEY.md §8(d) parity checks (i)-(iii) at matched photon counts."""
    ph = _rods(32)
    g = I.make_circular_geometry(100.0, 60.0, 16, 16, 1.6, 1)
    spec, resp = I.monochromatic_spectrum(100.0), I.detector_response()
    cfg_g = I.SimConfig(photons_total=200000, splitting=10, seed=1234, track_variance=True)
    cfg_c = I.SimConfig(photons_total=200000, splitting=10, seed=98765, track_variance=True)
    gpu = X.simulate_scatter_stats(ph, g, 0, spec, resp, cfg_g)
    cpu = orc.simulate_scatter_stats(ph, g, 0, spec, resp, cfg_c)
    se = np.hypot(gpu.total_std_error, cpu["total_std_error"])
    assert abs(gpu.total - cpu["total"]) < 3 * se
    # REF variance (transport.cpp:317-322) is the variance of the pixel sum itself
    var = gpu.variance + cpu["variance"]
    ok = var > 0
    z = (gpu.image - cpu["image"])[ok] / np.sqrt(var[ok])
    assert np.mean(np.abs(z) > 3) <= 2 * 0.0027 + 3 * np.sqrt(0.0027 / z.size)
    assert abs(np.mean(z)) < 3 / np.sqrt(z.size) + 0.05
    d2 = np.sum((gpu.image - cpu["image"]) ** 2)
    assert d2 <= 1.2 * np.sum(var) + 3 * np.sqrt(2 * np.sum(var ** 2))


def test_vacuum_phantom_scatter_is_zero():
    """REF test_transport.cpp:43-51."""
    ph = I.make_empty_phantom(8, 8, 8, (0.5, 0.5, 0.5), [I.material("water")])
    g = I.make_circular_geometry(60.0, 40.0, 16, 16, 0.6, 4)
    r = X.simulate_scatter_stats(ph, g, 0, I.monochromatic_spectrum(100.0),
                                 I.detector_response(), I.SimConfig(photons_total=2000, seed=20240915))
    assert np.all(r.image == 0.0) and r.total == 0.0


def test_errors_map_to_reference_exceptions():
    ph, g = _crit2()
    spec, resp = I.monochromatic_spectrum(100.0), I.detector_response()
    with pytest.raises(X.XscatOutOfRange, match="angle index out of range"):
        X.simulate_scatter_stats(ph, g, 3, spec, resp, I.SimConfig())
    with pytest.raises(X.XscatError, match="splitting must be >= 1"):
        X.simulate_scatter_stats(ph, g, 0, spec, resp, I.SimConfig(splitting=0))
    proj = X.Projector(ph, resp)
    with pytest.raises(X.XscatError, match="empty angle subset"):
        proj.run_scan(g, spec, I.SimConfig(), [])
    with pytest.raises(X.XscatOutOfRange, match="angle index"):
        proj.run_scan(g, spec, I.SimConfig(), [7])


def test_run_scan_matches_single_calls():
    ph, _ = _crit2()
    g = I.make_circular_geometry(60.0, 40.0, 24, 24, 0.55, 3)
    spec, resp = I.monochromatic_spectrum(100.0), I.detector_response()
    cfg = I.SimConfig(photons_total=6000, splitting=5, seed=20240915)
    proj = X.Projector(ph, resp)
    scan = proj.run_scan(g, spec, cfg, [0, 1, 2], X.BOTH)
    for i in range(3):
        assert np.array_equal(scan.scatter.images[i], proj.scatter_stats(g, i, spec, cfg).image)
        assert np.array_equal(scan.primary.images[i], proj.primary(g, i, spec, cfg))
