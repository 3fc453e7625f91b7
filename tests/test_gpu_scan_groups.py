"""Device scans with several angles per wavefront run (capi.cu scan_group,
wavefront.cu wave_run_jobs): each pipeline transports one angle at a time
and takes the next angle as soon as its current one has drained.  Histories
are pure functions of (seed, angle, bin, photon) and the tallies are
integers, so every grouping must reproduce the angle-by-angle scan bit for
bit (REF run_scan, transport.cpp:379-422)."""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _scene(n_angles=24):
    ph = S.make_rods_phantom(48, 10.0 / 48, 4.5, 8.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                             I.material("iron"), 7.874)
    g = I.make_circular_geometry(100.0, 60.0, 40, 32, 0.7, n_angles)
    return ph, g, I.kramers_spectrum(150.0), I.detector_response()


def _projector(ph, resp):
    ctx = X.Context(0)
    ctx.comm_init(1, 0, X.Context.comm_unique_id())
    return ctx, X.Projector(ph, resp, ctx=ctx)


# every angle of the circle (the run field's key changes four times), a
# descending run, repeats, and a single angle
SUBSETS = [list(range(24)), [23, 22, 21, 20, 19, 2, 1], [5, 5, 6, 5], [9]]


@pytest.mark.parametrize("subset", SUBSETS)
def test_grouped_device_scan_is_bit_identical(subset):
    ph, g, spec, resp = _scene()
    cfg = I.SimConfig(photons_total=40000, splitting=5, seed=77)
    ctx, proj = _projector(ph, resp)
    ref = proj.run_scan(g, spec, cfg, subset, X.BOTH)  # host-output scan: angle by angle
    for jobs, pipes in ((1, 2), (3, 2), (8, 2), (8, 3), (8, 1)):
        ctx.set_option("scan_jobs", jobs)
        ctx.set_option("wave_pipes", pipes)
        got = proj.run_scan_mgpu(g, spec, cfg, subset, X.BOTH)
        assert np.array_equal(got.scatter.images, ref.scatter.images), (jobs, pipes)
        assert np.array_equal(got.primary.images, ref.primary.images), (jobs, pipes)


def test_grouped_scan_few_histories_and_slots():
    """Fewer histories than pipelines and a slot count far below the history
    count (many refills per angle)."""
    ph, g, spec, resp = _scene(8)
    ctx, proj = _projector(ph, resp)
    for photons, slots in ((3, 1 << 22), (30000, 4096)):
        cfg = I.SimConfig(photons_total=photons, splitting=4, seed=5)
        ctx.set_option("wave_slots", slots)
        ctx.set_option("scan_jobs", 1)
        a = proj.run_scan_mgpu(g, spec, cfg, list(range(8)), X.SCATTER)
        ctx.set_option("scan_jobs", 8)
        b = proj.run_scan_mgpu(g, spec, cfg, list(range(8)), X.SCATTER)
        assert np.array_equal(a.scatter.images, b.scatter.images), photons


def test_grouped_scan_reports_refs_errors():
    ph, g, spec, resp = _scene(8)
    ctx, proj = _projector(ph, resp)
    cfg = I.SimConfig(photons_total=1000, splitting=4, seed=5)
    with pytest.raises(X.XscatOutOfRange, match="angle index 9 out of range"):
        proj.run_scan_mgpu(g, spec, cfg, [0, 1, 9], X.SCATTER)
    with pytest.raises(X.XscatError, match="empty angle subset"):
        proj.run_scan_mgpu(g, spec, cfg, [], X.SCATTER)
