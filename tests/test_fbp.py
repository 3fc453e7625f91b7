"""FDK: the C oracle against the compiled reference,
bit for bit (CPU), on a small cone-beam scan of a synthetic phantom's
line integrals."""
import numpy as np
import pytest

from paper_2201_13191_b200 import inputs as I


def scan(n_views=48, nu=24, nv=16, seed=3):
    g = I.make_circular_geometry(60.0, 40.0, nu, nv, 0.5, n_views)
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:nv, 0:nu]
    base = np.exp(-((xx - nu / 2) ** 2 / 30.0 + (yy - nv / 2) ** 2 / 20.0))
    stack = np.stack([base * (1.0 + 0.1 * np.sin(k)) + 0.01 * rng.standard_normal((nv, nu))
                      for k in range(n_views)])
    return g, np.asarray(g.angles, dtype=np.float64), stack


@pytest.mark.parametrize("hann", [True, False])
def test_fbp_oracle_bitwise(orc, ref, hann):
    g, ang, stack = scan()
    dims, voxel = (12, 10, 8), (0.35, 0.35, 0.4)
    a = orc.fbp_reconstruct(stack, ang, g, dims, voxel, hann)
    b = ref.fbp_reconstruct(stack, ang, g, dims, voxel, hann)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.count_nonzero(a) > a.size // 2


def test_fbp_errors(orc, ref):
    g, ang, stack = scan(n_views=8)
    for o in (orc, ref):
        with pytest.raises(I.XscatError, match="insufficient angular coverage"):
            o.fbp_reconstruct(stack[:2], ang[:2], g, (4, 4, 4), (0.5, 0.5, 0.5))
