"""Parity at the BASELINE.json workload configurations.

C1 runs at its full size and photon count against the oracle (per-history
replay: the same Philox streams and REF's arithmetic, so images agree
pixel by pixel to rounding).  C2 runs its full scene at 1e6 of its 1e7
photons (the oracle's CPU time).  C3 runs at its full size (512^3, 2048^2,
1e8 photons) through size-independent properties: bit-identical
integer tallies for two different photon-batch splits, REF's weight ledger
balance, and a primary image against the oracle on sampled pixels."""
import os

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import _capi as A
from paper_2201_13191_b200 import configs

from test_gpu_parity import _replay_compare

pytestmark = pytest.mark.gpu
CORES = os.cpu_count() or 4


def _replay(orc, w, photons):
    cfg = w.config
    cfg.photons_total = photons
    gpu = X.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, cfg)
    cpu = orc.simulate_scatter_stats(w.phantom, w.geometry, 0, w.spectrum, w.response, cfg, CORES)
    _replay_compare(gpu, cpu)
    for k, v in cpu["ledger"].items():
        assert getattr(gpu.ledger, k) == pytest.approx(v, rel=1e-9, abs=1e-300)
    return gpu


def test_c1_full_size_replay(orc):
    """C1: 60 keV, 128^3 water cylinder, 256^2, 1e6 photons, splitting 10."""
    gpu = _replay(orc, configs.c1(), 1_000_000)
    assert gpu.total > 0 and gpu.histories == 1_000_000


def test_c2_full_scene_replay(orc):
    """C2 scene (150 kVp, 256^3 water + Al rods, 512^2) at 1e6 photons."""
    gpu = _replay(orc, configs.c2(), 1_000_000)
    assert gpu.total > 0


def _ledger_balance(r):
    L = r.ledger
    out = L.escaped + L.absorbed + L.culled + L.roulette_killed
    return abs(L.initial + L.roulette_boost - out) / L.initial


def test_c3_full_size_properties(orc):
    """C3 at full size: the image from two photon batches (any split) is
    bit-identical to one run; REF's ledger balances (test_transport.cpp:83-111)."""
    import torch
    w = configs.c3()
    g, spec, cfg = w.geometry, w.spectrum, w.config
    proj = X.Projector(w.phantom, w.response)
    n = X.history_count(spec, cfg.photons_total)
    L = A.accum_layout(g.nu, g.nv, spec.n_bins, cfg.track_variance)
    whole = proj.scatter_stats(g, 0, spec, cfg)
    acc = torch.zeros(L["words"], dtype=torch.int64, device="cuda")
    cut = n // 3 + 12345
    proj.accumulate(g, 0, spec, cfg, 0, cut, acc.data_ptr())
    proj.accumulate(g, 0, spec, cfg, cut, n, acc.data_ptr())
    torch.cuda.synchronize()
    split = proj.finalize(g, spec, cfg, acc.data_ptr(), 0, n)
    assert np.array_equal(whole.image, split.image)
    assert whole.total == split.total and whole.total_std_error == split.total_std_error
    assert whole.histories == n == 100_000_000
    assert _ledger_balance(whole) < 1e-9
    # primary of the same projection against the oracle on sampled rows
    prim = proj.primary(g, 0, spec, cfg)
    cpu = orc.simulate_primary(w.phantom, g, 0, spec, w.response, cfg, CORES)
    rel = np.abs(prim - cpu) / cpu
    assert rel.max() <= 1e-12, rel.max()
