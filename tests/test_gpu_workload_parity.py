"""Scatter parity at the BASELINE.json workloads (SURVEY.md §8(d) "Parity
checks"), against the CPU oracle (oracle/liboracle.so, pinned bit-exact to
the compiled reference in tests/test_oracle.py).

Two kinds of check:

* Replay (same seed).  The device runs every history on the reference's
  Philox stream with the reference's fp64 arithmetic, so the images agree
  pixel by pixel up to rounding (`_replay_compare`: at most 1e-3 of the
  pixels off by more than 1e-9 relative + 1024 tally quanta, totals and
  ledger to 1e-6).
  - C3 scene (512^3 Al/Fe cylinder head, 2048^2, 150 kVp / 65 bins,
    splitting 20) at 1e6 photons, in the default walk (uniform blocks
    crossed in one step, 7 levels up to 128 voxels, 8-bit palette, the default
    slots in flight) and the strict voxel walk;
  - C2 at its full 1e7 photons;
  - C3 history ranges against the oracle's per-range accumulator: the
    fixed-point integer tallies themselves (limbs), to a few quanta.

* Statistics (independent seeds), the north_star scatter criterion and
  SURVEY.md §8(d) (i)-(iii), with the reference's own per-pixel variance
  (REF transport.cpp:317-322, track_variance):
  (i)   |T_gpu - T_cpu| < 3 sqrt(se_gpu^2 + se_cpu^2);
  (ii)  z = (I_gpu - I_cpu) / sqrt(var_gpu + var_cpu) per (super-)pixel:
        fraction(|z| > 3) <= 2 x 0.27 % (+ 3 binomial sigma); |mean z| only
        gets a loose sanity bound (see the statistical test's docstring);
  (iii) ||I_gpu - I_cpu||^2 <= 1.2 sum(var_gpu + var_cpu) (+ 3 sigma of
        that sum).
  Matched photon counts on both sides, as SURVEY.md §8(d) asks: the
  estimators' skew then cancels in the difference.
  Super-pixels: 8x8 at 2048^2 and 2x2 at 512^2, so every cell holds enough
  scores for the Gaussian z; the super-pixel variance is the sum of its
  pixels' variances (two rays of one history share a 8x8 cell with
  probability ~ 20*19/2 / 65536 = 0.3 %, negligible covariance).
"""
import os

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import configs

from test_gpu_parity import _replay_compare, tally_quantum

pytestmark = pytest.mark.gpu
CORES = os.cpu_count() or 4


def _ledger_close(gpu, cpu):
    for k, v in cpu["ledger"].items():
        assert getattr(gpu.ledger, k) == pytest.approx(v, rel=1e-6, abs=1e-300), k


@pytest.fixture(scope="module")
def c3_scene():
    return configs.c3(photons=1_000_000)


@pytest.mark.parametrize("walk", ["default", "voxel"])
def test_c3_scene_replay_1e6(orc, c3_scene, walk):
    """C3 scene at 1e6 photons, same seed: GPU vs oracle per history."""
    w = c3_scene
    ctx = X.projector.Context(0)
    if walk == "voxel":
        ctx.set_option("walk_mode", 0)
    proj = X.Projector(w.phantom, w.response, ctx=ctx)
    gpu = proj.scatter_stats(w.geometry, 0, w.spectrum, w.config)
    if walk == "default":
        assert gpu.stats["block_walk"] == 1 and gpu.stats["voxel_format"] == 1  # 8-bit palette + levels
        assert gpu.stats["live_histories"] >= 1_000_000  # every history in flight at once
    cpu = orc.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, w.config, CORES)
    assert gpu.histories == cpu["histories"] == 1_000_000
    _replay_compare(gpu, cpu, quantum=tally_quantum(w.geometry, w.spectrum))
    _ledger_close(gpu, cpu)


@pytest.mark.parametrize("step", [2, 3])
def test_c3_scene_march_mode_replay(orc, c3_scene, step):
    """REF's march mode (step_voxels > 1, trace.cpp:116-134) on the C3 scene:
    the block march (midpoint samples summed inside uniform blocks) replayed
    against the oracle's midpoint samples at 2e5 photons."""
    w = configs.c3(photons=200_000, phantom=c3_scene.phantom)
    cfg = w.config
    cfg.step_voxels = step
    proj = X.Projector(w.phantom, w.response, ctx=X.projector.Context(0))
    gpu = proj.scatter_stats(w.geometry, 0, w.spectrum, cfg)
    cpu = orc.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, cfg, CORES)
    assert gpu.histories == cpu["histories"]
    _replay_compare(gpu, cpu, quantum=tally_quantum(w.geometry, w.spectrum))
    _ledger_close(gpu, cpu)


def test_c4_scan_angle_sharded_replay_vs_oracle(orc):
    """C4 (BASELINE configs[3]: the 360-angle scan of the C3 scene),
    angle-sharded over a device group, at four angles spread over the circle
    -- the walk's run field then takes each travel direction (-x, -y, +x,
    +y) -- and 2e5 photons each: every scan image replays the oracle's
    projection at that angle (same criterion as _replay_compare)."""
    w = configs.c4(photons=200_000)
    subset = [0, 100, 190, 280]
    grp = X.Group([0, 0], w.phantom, w.response)
    scan = grp.run_scan(w.geometry, w.spectrum, w.config, subset, X.SCATTER)
    atol = 1024.0 * tally_quantum(w.geometry, w.spectrum)
    for k, a in enumerate(subset):
        cpu = orc.simulate_scatter_stats(w.phantom, w.geometry, a, w.spectrum, w.response, w.config, CORES)
        img, ref = scan.scatter.images[k].ravel(), np.asarray(cpu["image"]).ravel()
        nz = ref > 0
        bad = np.abs(img[nz] - ref[nz]) > 1e-9 * ref[nz] + atol
        assert np.mean(bad) <= 1e-3, (a, np.mean(bad))
        assert np.all(np.abs(img[~nz]) <= atol), a
        assert abs(img.sum() - ref.sum()) <= 1e-6 * ref.sum(), a


@pytest.mark.parametrize("walk", [0, 1])
def test_c3_history_ranges_bitwise_vs_oracle(orc, c3_scene, walk):
    """C3 scene, three ranges of 2000 histories (low, middle and high
    spectrum bins): the device's fixed-point accumulator against the
    oracle's (xo_scatter_accumulate_range, the same limb arithmetic).  The
    strict voxel walk (walk_mode 0) reproduces the reference's arithmetic, so
    every pixel agrees to 1e-9 (+ 1024 tally quanta of 2^-64 U_img: only the
    device's exp / log / acos may differ from glibc in the last ulp, which
    moves about 12 % of the scores by an ulp); the block walk (1) changes
    depths at rounding level, so its images agree to 1e-9."""
    import torch
    from paper_2201_13191_b200 import _capi as A
    w = c3_scene
    g, spec, cfg = w.geometry, w.spectrum, w.config
    ctx = X.projector.Context(0)
    ctx.set_option("walk_mode", walk)
    proj = X.Projector(w.phantom, w.response, ctx=ctx)
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, False)
    n = X.history_count(spec, cfg.photons_total)
    for h0 in (1000, n // 2, n - 2000):
        h1 = h0 + 2000
        acc = torch.zeros(L["words"], dtype=torch.int64, device="cuda")
        proj.accumulate(g, 0, spec, cfg, h0, h1, acc.data_ptr())
        dev = acc.cpu().numpy().view(np.uint64)
        cpu = np.zeros(L["words"], np.uint64)
        orc.accumulate_range(w.phantom, g, 0, spec, w.response, cfg, h0, h1, cpu)
        a = X.projector.finalize_host(g, spec, cfg, dev, h0, h1)
        b = X.projector.finalize_host(g, spec, cfg, cpu, h0, h1)
        assert a.histories == b.histories == 2000
        nz = b.image > 0
        if walk == 0:  # only libm last-ulp differences: every pixel to 1e-9
            q = tally_quantum(g, spec)
            assert np.all(np.abs(a.image - b.image) <= 1e-9 * b.image + 1024 * q), \
                np.max(np.abs(a.image - b.image) / (b.image + q))
        assert np.count_nonzero(a.image) == np.count_nonzero(b.image)
        rel = np.abs(a.image[nz] - b.image[nz]) / b.image[nz]
        assert np.mean(rel > 1e-9) <= 1e-3, (h0, np.mean(rel > 1e-9))
        for k in ("initial", "escaped", "absorbed", "culled", "roulette_killed", "roulette_boost"):
            assert getattr(a.ledger, k) == pytest.approx(getattr(b.ledger, k), rel=1e-9, abs=1e-300), k


def test_c2_full_photon_count_replay(orc):
    """C2 at its full 1e7 photons (BASELINE configs[1]), same seed."""
    w = configs.c2()
    gpu = X.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, w.config)
    cpu = orc.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, w.config, CORES)
    assert gpu.histories == cpu["histories"] == 10_000_000
    _replay_compare(gpu, cpu, quantum=tally_quantum(w.geometry, w.spectrum))
    _ledger_close(gpu, cpu)


def _bin(img, k):
    if k == 1:
        return img.ravel()
    nv, nu = img.shape
    return img.reshape(nv // k, k, nu // k, k).sum(axis=(1, 3)).ravel()


def z_stats(a_img, a_var, b_img, b_var, k):
    a, b = _bin(a_img, k), _bin(b_img, k)
    var = _bin(a_var, k) + _bin(b_var, k)
    ok = var > 0
    z = (a - b)[ok] / np.sqrt(var[ok])
    return dict(n=int(z.size), frac_z3=float(np.mean(np.abs(z) > 3)), mean_z=float(np.mean(z)),
                l2_ratio=float(np.sum((a - b) ** 2) / np.sum(var)),
                l2_bound=float(1.2 + 3 * np.sqrt(2 * np.sum(var ** 2)) / np.sum(var)))


def statistical_checks(gpu, cpu, k):
    """SURVEY.md §8(d) (i)-(iii); returns the measured quantities."""
    se = np.hypot(gpu.total_std_error, cpu["total_std_error"])
    out = z_stats(gpu.image, gpu.variance, cpu["image"], cpu["variance"], k)
    out["total_z"] = float((gpu.total - cpu["total"]) / se)
    n = out["n"]
    assert abs(out["total_z"]) < 3, out                                        # (i)
    assert out["frac_z3"] <= 2 * 0.0027 + 3 * np.sqrt(0.0027 / n), out         # (ii)
    assert abs(out["mean_z"]) <= 0.05, out
    assert out["l2_ratio"] <= out["l2_bound"], out                              # (iii)
    return out


@pytest.mark.parametrize("name,photons,k", [
    ("c1", 1_000_000, 1),   # 256^2 pixels, ~60 scores each
    ("c2", 2_000_000, 2),   # 512^2 -> 256^2 cells
    ("c3", 1_000_000, 8),   # 2048^2 -> 256^2 cells of 8x8 pixels
])
def test_statistical_parity_independent_seeds(orc, name, photons, k):
    """The north_star scatter criterion at each workload: independent seeds,
    matched photon counts, per-(super-)pixel z-scores and the relative L2
    against the expected statistical error.

    Why no "|mean z| <= 3/sqrt(n)": the cells are not independent.  One
    history scores `splitting` pixels with one weight, so a heavy history
    lifts many cells together and mean(z) fluctuates by more than 1/sqrt(n)
    (a GPU-vs-GPU control with independent seeds shows |mean z| up to 4/sqrt(n)
    at C3).  The global bias that mean(z) would catch is tested on the image
    total instead, criterion (i), which accounts for the correlation; mean(z)
    keeps a loose sanity bound.  The same control is asserted below for C3:
    the GPU-vs-oracle statistics must pass the same bounds as GPU-vs-GPU."""
    make = getattr(configs, name)
    kw = {}
    if name == "c3":
        kw["phantom"] = configs.c3_phantom()
    wg = make(photons=photons, seed=1_000_003, **kw)
    wc = make(photons=photons, seed=2_000_029, **kw)
    wg.config.track_variance = True
    wc.config.track_variance = True
    proj = X.Projector(wg.phantom, wg.response)
    gpu = proj.scatter_stats(wg.geometry, 0, wg.spectrum, wg.config)
    cpu = orc.simulate_scatter_stats(wc.phantom, wc.geometry, 0, wc.spectrum, wc.response, wc.config, CORES)
    out = statistical_checks(gpu, cpu, k)
    print(name, "gpu/oracle", out)
    if name == "c3":  # control: GPU vs GPU, a third independent seed
        wc.config.seed = 3_000_017
        g2 = proj.scatter_stats(wc.geometry, 0, wc.spectrum, wc.config)
        ctl = statistical_checks(gpu, {"image": g2.image, "variance": g2.variance, "total": g2.total,
                                       "total_std_error": g2.total_std_error}, k)
        print(name, "gpu/gpu control", ctl)
