"""The two transport engines against each other and against the oracle on
every device voxel format.

The wavefront pipeline (wavefront.cu) and the persistent megakernel
(transport.cu) run the same per-history arithmetic and the same fixed-point
tallies, so their outputs must be bit-identical (image, variance, totals,
ledger).  The phantoms cover the four encodings the upload chooses (4-bit
palette with register mu table, 4-bit palette, 8-bit palette, raw id +
density) plus both walk modes; each is also replayed against the oracle.
(With the voxel walk, palettes of <= 16 pairs are stored as 4-bit codes.)
"""
import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200 import synthetic as S

from test_gpu_parity import _replay_compare

pytestmark = pytest.mark.gpu


def _phantom(kind):
    water, iron = I.material("water"), I.material("iron")
    if kind == "p4reg":  # water cube in vacuum: 2 palette entries
        return S.make_cube_phantom(32, 0.2, 6.4, water, 1.0)
    if kind == "p4":  # 5..8 (material, density) pairs
        ph = S.make_rods_phantom(32, 10.0 / 32, 4.5, 8.0, water, 1.0, 4, 0.6, 3.0, iron, 7.874)
        ph.density[(ph.material_id == 1) & (np.arange(ph.density.size) % 7 == 0)] = 1.05
        ph.density[(ph.material_id == 1) & (np.arange(ph.density.size) % 11 == 0)] = 0.95
        ph.density[(ph.material_id == 2) & (np.arange(ph.density.size) % 5 == 0)] = 7.5
        return ph
    if kind == "p4wide":  # 9..16 pairs: 4-bit codes on the voxel walk, mu table in shared memory
        ph = S.make_rods_phantom(32, 10.0 / 32, 4.5, 8.0, water, 1.0, 4, 0.6, 3.0, iron, 7.874)
        idx = np.arange(ph.density.size)
        for k, d in enumerate((1.05, 0.95, 1.1, 0.9, 1.15, 0.85, 1.2, 0.8, 1.25, 0.75)):
            ph.density[(ph.material_id == 1) & (idx % (13 + k) == 0)] = d
        ph.density[(ph.material_id == 2) & (idx % 5 == 0)] = 7.5
        return ph
    rng = np.random.default_rng(5)
    ph = S.make_rods_phantom(32, 10.0 / 32, 4.5, 8.0, water, 1.0, 4, 0.6, 3.0, iron, 7.874)
    body = ph.material_id == 1
    levels = 40 if kind == "p8" else 400  # distinct densities -> 8-bit palette / raw
    ph.density[body] = 0.9 + 0.2 * rng.integers(0, levels, body.sum()) / levels
    return ph


def _format_of(stats):
    return {0: "p4", 1: "p8", 2: "raw"}.get(stats["voxel_format"], stats["voxel_format"])


@pytest.mark.parametrize("kind", ["p4reg", "p4", "p8reg", "p8", "raw"])
@pytest.mark.parametrize("exact", [0, 1])
def test_wavefront_equals_megakernel_bitwise(orc, kind, exact):
    ph = _phantom(kind.replace("p8reg", "p4reg"))
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=31337, roulette_wmin_rel=2.0,
                      roulette_survival=0.6, track_variance=True)
    ctx = X.projector.Context(0)
    ctx.set_option("exact_walk", exact)
    ctx.set_option("compact_palette", 1 if kind.startswith("p4") else 0)
    proj = X.Projector(ph, resp, ctx=ctx)
    out = {}
    for engine in (0, 1):
        ctx.set_option("engine", engine)
        out[engine] = proj.scatter_stats(g, 1, spec, cfg)
        assert out[engine].stats["engine"] == engine
    a, b = out[0], out[1]
    fmt = _format_of(b.stats)
    want = {"p4reg": "p4", "p4": "p4", "p8reg": "p8", "p8": "p8", "raw": "raw"}[kind]
    if exact and kind == "p8reg":  # the voxel walk re-encodes <= 16 pairs as 4-bit codes
        want = "p4"
    assert fmt == want, (kind, b.stats["voxel_format"], b.stats["palette_size"])
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.variance, b.variance)
    assert a.total == b.total and a.total_std_error == b.total_std_error
    assert a.ledger == b.ledger and a.histories == b.histories
    for k in ("free_path_steps", "scoring_steps", "histories", "scoring_rays", "interactions"):
        assert a.stats[k] == b.stats[k], k
    cpu = orc.simulate_scatter_stats(ph, g, 1, spec, resp, cfg)
    _replay_compare(b, cpu)


@pytest.mark.parametrize("pipes", [1, 2])
def test_wavefront_slot_count_does_not_change_results(pipes):
    """Fewer histories in flight -> more waves; one or two concurrent
    pipelines sharing the history counter; identical bits."""
    ph = _phantom("p4")
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=4, track_variance=True)
    ctx = X.projector.Context(0)
    ctx.set_option("engine", 0)
    proj = X.Projector(ph, resp, ctx=ctx)
    ref = proj.scatter_stats(g, 0, spec, cfg)  # megakernel
    ctx.set_option("engine", 1)
    ctx.set_option("wave_pipes", pipes)
    for slots in (3, 64, 1000):
        ctx.set_option("wave_slots", slots)
        r = proj.scatter_stats(g, 0, spec, cfg)
        assert np.array_equal(ref.image, r.image), slots
        assert np.array_equal(ref.variance, r.variance), slots
        assert ref.total == r.total and ref.ledger == r.ledger, slots
        assert slots <= r.stats["live_histories"] <= slots + 1


def test_wide_four_bit_palette_on_the_voxel_walk(orc):
    """9..16 (material, density) pairs on the voxel walk are stored as 4-bit
    codes; the wavefront engine's per-lane mu table must hold all 16 entries
    (it was sized for 8).  Both engines, bitwise, and the oracle."""
    ph = _phantom("p4wide")
    n_pairs = len({(int(i), float(d)) for i, d in zip(ph.material_id, ph.density)})
    assert 9 <= n_pairs <= 16, n_pairs
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=4242, track_variance=True)
    ctx = X.projector.Context(0)
    ctx.set_option("walk_mode", 0)
    proj = X.Projector(ph, resp, ctx=ctx)
    out = {}
    for engine in (0, 1):
        ctx.set_option("engine", engine)
        out[engine] = proj.scatter_stats(g, 1, spec, cfg)
    assert _format_of(out[1].stats) == "p4" and out[1].stats["palette_size"] == n_pairs
    assert np.array_equal(out[0].image, out[1].image)
    assert np.array_equal(out[0].variance, out[1].variance)
    assert out[0].ledger == out[1].ledger
    _replay_compare(out[1], orc.simulate_scatter_stats(ph, g, 1, spec, resp, cfg))


@pytest.mark.parametrize("kind", ["p4reg", "p8", "raw"])
@pytest.mark.parametrize("step", [2, 3])
def test_march_mode_on_the_wavefront_engine(orc, kind, step):
    """REF's march mode (step_voxels > 1, trace.cpp:116-134: the scoring rays
    are midpoint samples, free paths stay exact Siddon walks) on the
    wavefront engine: bit-identical to the megakernel, replayed against the
    oracle."""
    ph = _phantom(kind)
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=606 + step, step_voxels=step,
                      roulette_wmin_rel=2.0, roulette_survival=0.6, track_variance=True)
    ctx = X.projector.Context(0)
    proj = X.Projector(ph, resp, ctx=ctx)
    out = {}
    for engine in (0, 1):
        ctx.set_option("engine", engine)
        out[engine] = proj.scatter_stats(g, 2, spec, cfg)
        assert out[engine].stats["engine"] == engine
    a, b = out[0], out[1]
    assert np.array_equal(a.image, b.image) and np.array_equal(a.variance, b.variance)
    assert a.total == b.total and a.ledger == b.ledger
    for k in ("free_path_steps", "scoring_steps", "scoring_rays", "interactions"):
        assert a.stats[k] == b.stats[k], k
    _replay_compare(b, orc.simulate_scatter_stats(ph, g, 2, spec, resp, cfg))


@pytest.mark.parametrize("angle", [0, 1, 2, 4, 6])
def test_run_field_every_travel_direction(orc, angle):
    """The run field (Grid::run_*: same-code run lengths along the dominant
    travel axis of the projection, in the spare 8-bit-palette bits) for the
    four axis directions and the diagonal tie: fewer walk iterations than
    the block walk without runs, both engines bitwise, replayed against the
    oracle."""
    ph = S.make_rods_phantom(32, 10.0 / 32, 4.5, 8.0, I.material("water"), 1.0, 4, 0.6, 3.0,
                             I.material("iron"), 7.874)  # 3 palette entries: 3 run bits
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 8)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=77 + angle, track_variance=True)
    out = {}
    for runs in (0, 1):
        ctx = X.projector.Context(0)
        ctx.set_option("walk_mode", 1)
        ctx.set_option("runs", runs)
        proj = X.Projector(ph, resp, ctx=ctx)
        for engine in (0, 1):
            ctx.set_option("engine", engine)
            out[runs, engine] = proj.scatter_stats(g, angle, spec, cfg)
        assert _format_of(out[runs, 1].stats) == "p8"
    a, b = out[1, 0], out[1, 1]
    assert np.array_equal(a.image, b.image) and np.array_equal(a.variance, b.variance)
    assert a.total == b.total and a.ledger == b.ledger
    assert b.stats["walk_iterations"] < 0.95 * out[0, 1].stats["walk_iterations"]
    _replay_compare(b, orc.simulate_scatter_stats(ph, g, angle, spec, resp, cfg))


@pytest.mark.parametrize("angle", [2, 5])
def test_run_field_two_bits_shared_mu_table(orc, angle):
    """5..8 palette entries on the 8-bit palette: two run bits (runs capped at
    3) and the per-material mu table in shared memory (not the register
    one): both engines bitwise, replayed against the oracle."""
    ph = _phantom("p4")  # 5..8 (material, density) pairs
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 8)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=99 + angle, track_variance=True)
    ctx = X.projector.Context(0)
    ctx.set_option("walk_mode", 1)
    proj = X.Projector(ph, resp, ctx=ctx)
    out = {}
    for engine in (0, 1):
        ctx.set_option("engine", engine)
        out[engine] = proj.scatter_stats(g, angle, spec, cfg)
    a, b = out[0], out[1]
    assert _format_of(b.stats) == "p8" and 5 <= b.stats["palette_size"] <= 8
    assert np.array_equal(a.image, b.image) and np.array_equal(a.variance, b.variance)
    assert a.total == b.total and a.ledger == b.ledger
    off = X.projector.Context(0)  # the same walk without the run field
    off.set_option("walk_mode", 1)
    off.set_option("runs", 0)
    c = X.Projector(ph, resp, ctx=off).scatter_stats(g, angle, spec, cfg)
    assert b.stats["walk_iterations"] < c.stats["walk_iterations"]
    _replay_compare(b, orc.simulate_scatter_stats(ph, g, angle, spec, resp, cfg))


def test_large_splitting_clamps_live_histories_and_stays_exact():
    """Splitting 500 with 2e6 histories: the walker state of every history in
    flight would need ~150 GB, so the wavefront engine lowers its live-history
    count to the memory it has and remembers the decision per
    request; the image equals a run with a small fixed slot count bit for
    bit (the slot count never changes results), and a following
    small-splitting call takes the full count again."""
    ph = _phantom("p4reg")
    g = I.make_circular_geometry(100.0, 60.0, 32, 24, 0.8, 4)
    spec, resp = I.kramers_spectrum(150.0), I.detector_response()
    cfg = I.SimConfig(photons_total=2_000_000, splitting=500, seed=8)
    n = X.history_count(spec, cfg.photons_total)
    ctx = X.projector.Context(0)
    proj = X.Projector(ph, resp, ctx=ctx)
    big = proj.scatter_stats(g, 1, spec, cfg)
    assert big.stats["live_histories"] < n  # clamped
    small_cfg = I.SimConfig(photons_total=20000, splitting=5, seed=8)
    assert proj.scatter_stats(g, 1, spec, small_cfg).stats["live_histories"] >= X.history_count(spec, 20000)
    again = proj.scatter_stats(g, 1, spec, cfg)
    assert again.stats["live_histories"] == big.stats["live_histories"]
    ctx.set_option("wave_slots", 65536)
    fixed = proj.scatter_stats(g, 1, spec, cfg)
    assert fixed.stats["live_histories"] <= 65536 + 2
    for r in (again, fixed):
        assert np.array_equal(big.image, r.image) and big.total == r.total and big.ledger == r.ledger
