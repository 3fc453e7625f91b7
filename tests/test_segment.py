"""Segmentation stage: the C oracle against the
compiled reference, bit for bit (CPU), on REF's own test cases
(tests/test_recon.cpp:158-290, acceptance criterion 9 at
acceptance_main.cpp:539-580) and on fresh volumes."""
import numpy as np
import pytest

from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200.projector import ClassSpec


def mixture(rng, shape, nan=False):
    """Three-class mixture (REF test_recon.cpp:170-190 style)."""
    pick = rng.uniform(size=shape)
    v = np.where(pick < 0.3, rng.normal(10.0, 1.5, shape),
                 np.where(pick < 0.7, rng.normal(25.0, 2.0, shape), rng.normal(45.0, 2.5, shape)))
    v = v.astype(np.float32)
    if nan:
        v.reshape(-1)[rng.integers(0, v.size, 7)] = np.nan
    return v


def brute_force_cuts(count, n_classes):
    """REF tests/support/oracles.hpp:231-273 (exhaustive search, long double)."""
    import itertools
    bins = len(count)
    c = np.asarray(count, np.longdouble)
    pc = np.concatenate([[0], np.cumsum(c)])
    ps = np.concatenate([[0], np.cumsum(c * (np.arange(bins) + np.longdouble(0.5)))])

    def score(b0, b1):
        n = pc[b1] - pc[b0]
        return np.longdouble(-1e38) if n <= 0 else (ps[b1] - ps[b0]) ** 2 / n

    best, best_s = None, np.longdouble(-1e38)
    for idx in itertools.combinations(range(1, bins), n_classes - 1):
        edges = (0,) + idx + (bins,)
        s = sum(score(edges[i], edges[i + 1]) for i in range(n_classes))
        if s > best_s:
            best_s, best = s, idx
    return list(best)


def interior_hist(vol, bins):
    nz, ny, nx = vol.shape
    m = [max(0, n // 20) for n in (nx, ny, nz)]
    inner = vol[m[2]:nz - m[2], m[1]:ny - m[1], m[0]:nx - m[0]].astype(np.float64)
    lo, hi = inner.min(), inner.max()
    b = np.clip(((inner - lo) / (hi - lo) * bins).astype(np.int64), 0, bins - 1)
    return np.bincount(b.ravel(), minlength=bins).astype(np.float64), lo, hi


@pytest.mark.parametrize("n_classes", [2, 3, 4])
@pytest.mark.parametrize("bins", [64, 1024])
def test_otsu_oracle_bitwise(orc, ref, n_classes, bins):
    rng = np.random.default_rng(100 * n_classes + bins)
    vol = mixture(rng, (20, 21, 22))
    a = orc.otsu_thresholds(vol, n_classes, bins)
    b = ref.otsu_thresholds(vol, n_classes, bins)
    assert np.array_equal(np.array(a).view(np.uint64), np.array(b).view(np.uint64))
    assert all(x < y for x, y in zip(a, a[1:]))


def test_otsu_nan_voxels(orc, ref):
    vol = mixture(np.random.default_rng(5), (16, 16, 16), nan=True)
    assert orc.otsu_thresholds(vol, 3, 256) == ref.otsu_thresholds(vol, 3, 256)


@pytest.mark.parametrize("n_classes", [2, 3])
def test_otsu_matches_brute_force(orc, n_classes):
    # REF test_recon.cpp:170-219 / acceptance criterion 9: 64-bin histograms
    vol = mixture(np.random.default_rng(29 + n_classes), (20, 20, 20))
    th = orc.otsu_thresholds(vol, n_classes, 64)
    count, lo, hi = interior_hist(vol, 64)
    cuts = brute_force_cuts(count, n_classes)
    for t, c in zip(th, cuts):
        assert t == pytest.approx(lo + c * (hi - lo) / 64, rel=1e-12)


def test_otsu_bimodal_and_scaling(orc):
    # REF test_recon.cpp:158-168 and :221-232
    rng = np.random.default_rng(17)
    vol = np.where(rng.uniform(size=(24, 24, 24)) < 0.4, 10.0, 50.0).astype(np.float32)
    th = orc.otsu_thresholds(vol, 2, 256)
    assert len(th) == 1 and 10.0 < th[0] < 50.0
    vol = (5.0 + 40.0 * rng.uniform(size=(16, 16, 16)) + 60.0 * (rng.uniform(size=(16, 16, 16)) < 0.5))
    vol = vol.astype(np.float32)
    t1 = orc.otsu_thresholds(vol, 2, 128)[0]
    t3 = orc.otsu_thresholds(vol * np.float32(3.0), 2, 128)[0]
    assert t3 == pytest.approx(3.0 * t1, rel=1e-6)


def test_otsu_errors(orc, ref):
    vol = np.full((16, 16, 16), 4.0, np.float32)
    for o in (orc, ref):
        with pytest.raises(I.XscatError, match="degenerate histogram"):
            o.otsu_thresholds(vol, 2)
        with pytest.raises(I.XscatInvalidArgument, match="n_classes must be in"):
            o.otsu_thresholds(vol, 5)
        with pytest.raises(I.XscatInvalidArgument, match="too few histogram bins"):
            o.otsu_thresholds(vol, 3, 2)


def test_segment_volume_bitwise(orc, ref):
    rng = np.random.default_rng(3)
    vol = mixture(rng, (9, 10, 11), nan=True)
    thr = [17.5, 35.25]
    a = orc.segment_volume(vol, thr, 3)
    assert np.array_equal(a, ref.segment_volume(vol, thr, 3))
    assert set(np.unique(a)) == {0, 1, 2}
    for o in (orc, ref):
        with pytest.raises(I.XscatError, match="strictly increasing"):
            o.segment_volume(vol, [3.0, 3.0], 3)
        with pytest.raises(I.XscatError, match="class_map must cover all 3 classes"):
            o.segment_volume(vol, thr, 2)


WATER = None


def water():
    global WATER
    if WATER is None:
        WATER = I.material("water")
    return WATER


@pytest.mark.parametrize("src,tgt", [((8, 8, 8), (4, 4, 4)), ((13, 11, 9), (5, 4, 3)),
                                     ((4, 5, 6), (6, 5, 9)), ((12, 12, 12), (12, 12, 12))])
def test_density_phantom_bitwise(orc, ref, src, tgt):
    rng = np.random.default_rng(sum(src) + sum(tgt))
    labels = rng.integers(0, 3, size=src[::-1]).astype(np.uint8)
    cmap = [ClassSpec(0, 0.0), ClassSpec(1, 0.9), ClassSpec(2, 2.699)]
    mats = [water(), I.material("aluminum")]
    if any(t > s_ for s_, t in zip(src, tgt)):
        # up-sampling leaves empty blocks: 0/0 density, rejected by validate_phantom
        for o in (orc, ref):
            with pytest.raises(I.XscatError, match="negative density"):
                o.to_density_phantom(labels, cmap, tgt, mats)
        return
    a = orc.to_density_phantom(labels, cmap, tgt, mats)
    b = ref.to_density_phantom(labels, cmap, tgt, mats)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


def test_density_phantom_reference_cases(orc, ref):
    # REF test_recon.cpp:243-290
    for o in (orc, ref):
        lab = np.zeros((8, 8, 8), np.uint8)
        ids, dens = o.to_density_phantom(lab, [ClassSpec(1, 1.0)], (4, 4, 4), [water()])
        assert (ids == 1).all() and (dens == 1.0).all()
        ids, dens = o.to_density_phantom(lab, [ClassSpec(0, 0.0)], (4, 4, 4), [water()])
        assert (ids == 0).all() and (dens == 0.0).all()
        z, y, x = np.mgrid[0:8, 0:8, 0:8]
        board = ((x + y + z) % 2).astype(np.uint8)
        ids, dens = o.to_density_phantom(board, [ClassSpec(0, 0.0), ClassSpec(1, 2.0)], (4, 4, 4), [water()])
        assert (ids == 1).all() and np.allclose(dens, 1.0)
        bad = board.copy()
        bad.reshape(-1)[0] = 7
        with pytest.raises(I.XscatError, match="unmapped label 7"):
            o.to_density_phantom(bad, [ClassSpec(0, 0.0), ClassSpec(1, 2.0)], (4, 4, 4), [water()])
        with pytest.raises(I.XscatError, match="material id 3 has no loaded material"):
            o.to_density_phantom(board, [ClassSpec(0, 0.0), ClassSpec(3, 2.0)], (4, 4, 4), [water()])
