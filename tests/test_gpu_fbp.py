"""FDK on the device against the C oracle (pinned bit-exact to REF in
tests/test_fbp.py): the same arithmetic in the same order, so the float
volumes are compared bit for bit."""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I

from test_fbp import scan

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("hann", [True, False])
@pytest.mark.parametrize("shape", [(48, 24, 16, (12, 10, 8)), (90, 37, 21, (20, 18, 9))])
def test_fbp_bitwise(orc, hann, shape):
    n_views, nu, nv, dims = shape
    g, ang, stack = scan(n_views, nu, nv)
    voxel = X.default_voxel_size(g, dims)
    gpu = X.fbp_reconstruct(X.ProjectionStack(ang, stack), g, dims, voxel, X.HANN if hann else X.RAMLAK)
    cpu = orc.fbp_reconstruct(stack, ang, g, dims, voxel, hann)
    assert np.array_equal(gpu.view(np.uint32), cpu.view(np.uint32))


def test_fbp_errors():
    g, ang, stack = scan(n_views=8)
    with pytest.raises(I.XscatError, match="insufficient angular coverage"):
        X.fbp_reconstruct(X.ProjectionStack(ang[:2], stack[:2]), g, (4, 4, 4))
