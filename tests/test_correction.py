"""Correction-loop stages: the C oracle against the
compiled reference, bit for bit (CPU)."""
import numpy as np
import pytest

from paper_2201_13191_b200 import inputs as I


def _stacks(rng, n=3, nv=12, nu=16):
    a = rng.uniform(0.1, 3.0, (n, nv, nu))
    p = rng.uniform(0.05, 2.0, (n, nv, nu))
    s = rng.normal(0.05, 0.05, (n, nv, nu))  # some negative scatter (clamped)
    return a, p, s


def test_intensity_to_attenuation_bitwise(orc, ref):
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(1)
    inten = rng.uniform(0.01, 1.0, (4, 10, 14))
    flat = rng.uniform(1.0, 2.0, (10, 14))
    assert np.array_equal(orc.intensity_to_attenuation(inten, flat), ref.intensity_to_attenuation(inten, flat))
    inten[1, 3, 4] = 0.0
    inten[2, 0, 0] = -1.0
    flat[5, 5] = 0.0
    for o in (orc, ref):
        with pytest.raises(I.XscatError, match="intensity_to_attenuation: 3 non-positive pixels"):
            o.intensity_to_attenuation(inten, flat)


def test_correct_projections_bitwise(orc, ref):
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(2)
    a, p, s = _stacks(rng)
    co, clo = orc.correct_projections(a, p, s)
    cr, clr = ref.correct_projections(a, p, s)
    assert np.array_equal(co, cr) and clo == clr and clo == int((s < 0).sum())
    p[0, 2, 3] = 0.0
    for o in (orc, ref):
        with pytest.raises(I.XscatError, match="non-positive primary pixel"):
            o.correct_projections(a, p, s)


def test_correction_tail_bitwise(orc, ref):
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(3)
    nu, nv, nu_out, nv_out = 20, 16, 40, 32
    full = np.linspace(0.0, 2 * np.pi, 8, endpoint=False)
    sub = full[::2]
    yy, xx = np.mgrid[0:nv, 0:nu]
    base = np.exp(-((xx - nu / 2) ** 2 + (yy - nv / 2) ** 2) / 40.0)
    scat = np.stack([0.2 * base + 0.01 * rng.standard_normal((nv, nu)) for _ in sub])
    prim = np.stack([1.0 - 0.9 * base + 0.001 * k for k in range(full.size)])
    a = rng.uniform(0.0, 2.0, (full.size, nv_out, nu_out))
    co, fo, clo = orc.correction_tail(scat, sub, prim, full, 5, 2, a)
    cr, fr, clr = ref.correction_tail(scat, sub, prim, full, 5, 2, a)
    assert np.array_equal(co, cr)
    assert fo == fr and clo == clr
