"""Correction-loop stages on the device against the oracle / compiled
reference.

Tolerances: the stages are REF's fp64 arithmetic (-fmad=false); only the
device `log` may differ from glibc's in the last ulp, so corrected values
agree to 1e-14 absolute (values are O(1)), counts exactly, and the mean
scatter fraction to 1e-12 relative (the device sums it in fixed point,
REF in sequential fp64)."""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I

pytestmark = pytest.mark.gpu


def test_intensity_to_attenuation(orc):
    rng = np.random.default_rng(11)
    inten = rng.uniform(0.01, 1.0, (5, 33, 47))
    flat = rng.uniform(1.0, 2.0, (33, 47))
    g = X.intensity_to_attenuation(inten, flat)
    c = orc.intensity_to_attenuation(inten, flat)
    assert np.max(np.abs(g - c)) <= 1e-14
    inten[2, 3, 4] = 0.0
    flat[1, 1] = -1.0
    with pytest.raises(I.XscatError, match="intensity_to_attenuation: 2 non-positive pixels"):
        X.intensity_to_attenuation(inten, flat)


def test_correct_projections(orc):
    rng = np.random.default_rng(12)
    a = rng.uniform(0.1, 3.0, (4, 40, 50))
    p = rng.uniform(0.05, 2.0, a.shape)
    s = rng.normal(0.05, 0.05, a.shape)
    g, gc = X.correct_projections(a, p, s)
    c, cc = orc.correct_projections(a, p, s)
    assert gc == cc == int((s < 0).sum())
    assert np.max(np.abs(g - c)) <= 1e-14
    p[1, 5, 5] = 0.0
    with pytest.raises(I.XscatError, match="correct_projections: non-positive primary pixel"):
        X.correct_projections(a, p, s)


@pytest.mark.parametrize("shape", [(20, 16, 40, 32), (64, 48, 256, 192)])
def test_correction_tail(orc, shape):
    nu, nv, nu_out, nv_out = shape
    rng = np.random.default_rng(13)
    full = np.linspace(0.0, 2 * np.pi, 12, endpoint=False)
    sub = full[::2]
    yy, xx = np.mgrid[0:nv, 0:nu]
    base = np.exp(-((xx - nu / 2) ** 2 + (yy - nv / 2) ** 2) / (0.05 * nu * nv))
    scat = np.stack([0.2 * base + 0.01 * rng.standard_normal((nv, nu)) for _ in sub])
    prim = np.stack([1.0 - 0.999 * base + 1e-4 * k for k in range(full.size)])
    a = rng.uniform(0.0, 2.0, (full.size, nv_out, nu_out))
    f = X.SgFilterSpec(5, 2)
    g, gf, gc = X.correction_tail(scat, sub, prim, full, f, a)
    c, cf, cc = orc.correction_tail(scat, sub, prim, full, 5, 2, a)
    assert gc == cc
    assert abs(gf - cf) <= 1e-12 * cf
    assert np.max(np.abs(g - c)) <= 1e-13


def test_correction_tail_matches_separate_stages(orc):
    """The fused tail equals the unfused device stages composed by hand
    (sg_smooth, interpolate_angles, upsample_image, floor, correct_projections)."""
    rng = np.random.default_rng(14)
    nu, nv, nu_out, nv_out = 24, 20, 48, 40
    full = np.linspace(0.0, 2 * np.pi, 6, endpoint=False)
    sub = full[::3]
    scat = rng.uniform(-0.01, 0.3, (sub.size, nv, nu))
    prim = rng.uniform(0.2, 1.0, (full.size, nv, nu))
    a = rng.uniform(0.0, 2.0, (full.size, nv_out, nu_out))
    f = X.SgFilterSpec(5, 3)
    fused, frac, cl = X.correction_tail(scat, sub, prim, full, f, a)
    sm = X.sg_smooth(scat, f)
    s_full = X.interpolate_angles(X.ProjectionStack(np.asarray(sub), sm), full)
    s_hi = X.upsample_image(s_full.images, nu_out, nv_out)
    p_hi = X.upsample_image(prim, nu_out, nv_out)
    p_hi = np.maximum(p_hi, 1e-12 * np.maximum(p_hi.reshape(full.size, -1).max(1), 0.0)[:, None, None])
    sep, cl2 = X.correct_projections(a, p_hi, s_hi)
    assert cl == cl2
    assert np.max(np.abs(fused - sep)) <= 1e-13
