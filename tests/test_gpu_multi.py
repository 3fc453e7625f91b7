"""Multi-GPU paths of the library (include/xscat_gpu.h "multi-GPU";
multi.cu), on the one GPU of the test box.

* Groups (one process, N contexts): a device may be listed several times, so
  a group of [0, 0] or [0, 0, 0] runs the real code path (member threads,
  photon-batch shares, scene replication by xs_ctx_copy_scene, the root's
  fused reduce + finalize kernel over the members' accumulators, angle
  sharding, the sharded correction loop) on one device.  Results must be
  bit-identical to one context: the tallies are integers.
* NCCL communicator (multi-process API) with one rank: the communicator,
  ncclReduce and the status agreement run; NCCL rejects two ranks on one GPU,
  so the N > 1 exchange is covered by the gloo test (tests/test_multirank.py)
  and by bench.py under torchrun on a multi-GPU node.
"""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _scene():
    ph = S.make_rods_phantom(48, 10.0 / 48, 4.5, 8.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                             I.material("iron"), 7.874)
    g = I.make_circular_geometry(100.0, 60.0, 40, 32, 0.7, 6)
    return ph, g, I.kramers_spectrum(150.0), I.detector_response()


def _same(a, b):
    assert np.array_equal(a.image, b.image)
    if a.variance is not None:
        assert np.array_equal(a.variance, b.variance)
    assert a.total == b.total and a.total_std_error == b.total_std_error
    assert a.ledger == b.ledger and a.histories == b.histories


@pytest.mark.parametrize("members", [[0, 0], [0, 0, 0]])
def test_group_photon_batches_bit_identical(members):
    ph, g, spec, resp = _scene()
    cfg = I.SimConfig(photons_total=60001, splitting=7, seed=55, track_variance=True,
                      roulette_wmin_rel=2.0, roulette_survival=0.6)
    one = X.Projector(ph, resp, ctx=X.Context(0)).scatter_stats(g, 2, spec, cfg)
    grp = X.Group(members, ph, resp)
    assert len(grp) == len(members)
    many = grp.scatter_stats(g, 2, spec, cfg)
    _same(one, many)
    # each member ran its share only (every history of a share is in flight at once)
    per = [grp.launch_stats(i)["live_histories"] for i in range(len(members))]
    share = -(-one.histories // len(members))
    assert all(share - 1 <= p <= share + 1 for p in per), per  # (+1: two pipelines round up)


def test_group_run_scan_matches_one_context():
    ph, g, spec, resp = _scene()
    cfg = I.SimConfig(photons_total=8000, splitting=5, seed=7)
    one = X.Projector(ph, resp, ctx=X.Context(0)).run_scan(g, spec, cfg, [5, 0, 3, 1, 2], X.BOTH)
    grp = X.Group([0, 0], ph, resp)
    two = grp.run_scan(g, spec, cfg, [5, 0, 3, 1, 2], X.BOTH)
    assert np.array_equal(one.scatter.images, two.scatter.images)
    assert np.array_equal(one.primary.images, two.primary.images)
    assert len(two.seconds_per_angle) == 5 and all(s > 0 for s in two.seconds_per_angle)
    # REF's error (transport.cpp:390-392, :414-417) from the member that met it
    with pytest.raises(X.XscatOutOfRange, match="angle index 9"):
        grp.run_scan(g, spec, cfg, [0, 1, 9], X.SCATTER)
    with pytest.raises(X.XscatError, match="empty angle subset"):
        grp.run_scan(g, spec, cfg, [], X.SCATTER)


def test_group_errors_are_reference_errors():
    ph, g, spec, resp = _scene()
    grp = X.Group([0, 0], ph, resp)
    with pytest.raises(X.XscatOutOfRange, match="angle index out of range"):
        grp.scatter_stats(g, 99, spec, I.SimConfig(photons_total=100))
    with pytest.raises(X.XscatError, match="splitting must be >= 1"):
        grp.scatter_stats(g, 0, spec, I.SimConfig(splitting=0))


def test_copy_scene_gives_the_same_projector():
    ph, g, spec, resp = _scene()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=8)
    a = X.Context(0)
    pa = X.Projector(ph, resp, ctx=a)
    b = X.Context(0)
    X._capi.check(X._capi.lib().xs_ctx_copy_scene(b.h, a.h), b.h)
    pb = X.Projector.__new__(X.Projector)
    pb.ctx, pb.phantom, pb.response = b, ph, resp
    _same(pa.scatter_stats(g, 1, spec, cfg), pb.scatter_stats(g, 1, spec, cfg))
    assert np.array_equal(pa.primary(g, 1, spec), pb.primary(g, 1, spec))


def test_nccl_communicator_single_rank():
    ph, g, spec, resp = _scene()
    cfg = I.SimConfig(photons_total=30000, splitting=5, seed=21, track_variance=True)
    ctx = X.Context(0)
    proj = X.Projector(ph, resp, ctx=ctx)
    uid = X.Context.comm_unique_id()
    assert len(uid) == 128
    ctx.comm_init(1, 0, uid)
    assert ctx.comm_size() == (1, 0)
    _same(proj.scatter_stats(g, 3, spec, cfg), proj.scatter_stats_mgpu(g, 3, spec, cfg))
    a = proj.run_scan(g, spec, cfg, [4, 2, 0], X.BOTH)
    b = proj.run_scan_mgpu(g, spec, cfg, [4, 2, 0], X.BOTH)
    assert np.array_equal(a.scatter.images, b.scatter.images)
    assert np.array_equal(a.primary.images, b.primary.images)
    with pytest.raises(X.XscatOutOfRange, match="angle index out of range"):
        proj.scatter_stats_mgpu(g, 17, spec, cfg)


def test_context_without_communicator_fails():
    ph, g, spec, resp = _scene()
    proj = X.Projector(ph, resp, ctx=X.Context(0))
    with pytest.raises(X.XscatError, match="no communicator"):
        proj.scatter_stats_mgpu(g, 0, spec, I.SimConfig(photons_total=10))


def test_group_correction_loop_matches_one_context():
    """The loop with its scans sharded by angle over a group (the segmented
    phantom replicated to the members every iteration): same reports and
    corrected stack as one context (REF test_correction.cpp:118-160 shape)."""
    from test_gpu_loop import measurement
    w = I.material("water")
    n = 24
    ph = S.make_cylinder_phantom(n, 0.3, 2.2, 5.0, w, 1.0)
    g = I.make_circular_geometry(60.0, 40.0, 24, 24, 0.5, 36)
    spec, resp = I.monochromatic_spectrum(100.0), I.detector_response()
    sim = I.SimConfig(photons_total=2000, splitting=4, seed=99)
    raw, flat = measurement(ph, g, spec, resp, sim, True)
    cfg = X.CorrectionConfig(n_iterations=2, simulate_every_kth_angle=2, mc_nu=12, mc_nv=12,
                             recon_dims=(n, n, n), n_classes=2,
                             class_map=[X.ClassSpec(0, 0.0), X.ClassSpec(1, 1.0)], sim=sim)
    stack = X.ProjectionStack(g.angles, raw)
    one = X.run_iterative_correction(stack, flat, g, spec, resp, cfg, [w], ctx=X.Context(0))
    grp = X.Group([0, 0, 0])
    many = X.run_iterative_correction(stack, flat, g, spec, resp, cfg, [w], group=grp)
    assert np.array_equal(one.corrected_stack.images, many.corrected_stack.images)
    assert np.array_equal(one.corrected_volume, many.corrected_volume)
    for a, b in zip(one.reports, many.reports):
        assert a.mean_scatter_fraction == b.mean_scatter_fraction
        assert a.negative_scatter_clamped == b.negative_scatter_clamped
        assert a.ncc_to_previous == b.ncc_to_previous
