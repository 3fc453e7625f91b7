"""GPU post-processing kernels vs the oracle restatement of REF postprocess.cpp:
same fp64 operations in the same order -> bit-identical outputs."""
import numpy as np
import pytest

import paper_2201_13191_b200 as X

pytestmark = pytest.mark.gpu


def _imgs(n, nv, nu, seed=3):
    return np.random.default_rng(seed).random((n, nv, nu))


@pytest.mark.parametrize("window,order,nu,nv", [(5, 3, 16, 12), (7, 2, 40, 33), (15, 3, 64, 48)])
def test_sg_smooth_bit_exact(orc, window, order, nu, nv):
    st = _imgs(3, nv, nu)
    gpu = X.sg_smooth(st, X.SgFilterSpec(window, order))
    for i in range(3):
        assert np.array_equal(gpu[i], orc.sg_smooth(st[i], window, order))


def test_interpolate_angles_bit_exact(orc):
    src = np.array([0.0, 1.0, 2.0, 3.0, 4.0, 5.0])
    tgt = np.array([0.0, 0.5, 1.0, 2.25, 5.0, 5.9, 6.2])
    st = _imgs(6, 9, 11)
    gpu = X.interpolate_angles(X.ProjectionStack(src, st), tgt)
    cpu = orc.interpolate_angles(st, src, tgt)
    assert np.array_equal(gpu.images, cpu)
    tgt2 = np.array([-0.5 + 0.6, 5.5])  # wrap below the first / above the last
    assert np.array_equal(X.interpolate_angles(X.ProjectionStack(src[1:], st[1:]), tgt2).images,
                          orc.interpolate_angles(st[1:], src[1:], tgt2))


@pytest.mark.parametrize("nu,nv,nuo,nvo", [(16, 12, 64, 48), (7, 5, 7, 13), (1, 4, 3, 9)])
def test_upsample_bit_exact(orc, nu, nv, nuo, nvo):
    st = _imgs(2, nv, nu)
    gpu = X.upsample_image(st, nuo, nvo)
    for i in range(2):
        assert np.array_equal(gpu[i], orc.upsample_image(st[i], nuo, nvo))


def test_downsample_bit_exact(orc):
    st = _imgs(2, 48, 64)
    gpu = X.downsample_average(st, 16, 12)
    for i in range(2):
        assert np.array_equal(gpu[i], orc.downsample_average(st[i], 16, 12))


def test_postprocess_errors():
    with pytest.raises(X.XscatError, match="window must be odd"):
        X.sg_smooth(_imgs(1, 16, 16)[0], X.SgFilterSpec(4, 3))
    with pytest.raises(X.XscatError, match="smaller than filter window"):
        X.sg_smooth(_imgs(1, 4, 4)[0], X.SgFilterSpec(5, 3))
    with pytest.raises(X.XscatError, match="target dims"):
        X.upsample_image(_imgs(1, 8, 8)[0], 4, 4)
