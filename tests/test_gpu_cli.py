"""The CLI's `simulate` end to end on the device (REF
tools/main.cpp:83-130): a REF run configuration in, REF's outputs out
(primary.xprj, scatter.xprj, timing.csv in output_dir).  The images must be
the projector's own run_scan on the same inputs, narrowed to f32 as REF's
save_stack does: bit-identical, for one device and for a device group.
"""
import pathlib
import shutil
import subprocess

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import files as F
from paper_2201_13191_b200 import inputs as I

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]
CFG = ROOT / "tests" / "golden" / "files" / "cfg"
CLI = ROOT / "paper_2201_13191_b200" / "bin" / "xscat_b200"


def _run(tmp_path, args, env=None):
    work = tmp_path / "cfg"
    shutil.copytree(CFG, work, ignore=shutil.ignore_patterns("out"))
    import os
    e = dict(os.environ, **(env or {}))
    r = subprocess.run([str(CLI), "simulate", "--config", str(work / "good.ini"), *args], capture_output=True,
                       text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr
    return work, r


def _expected(work, subset, what):
    mats = [F.load_material(work / "data" / "materials" / f) for f in ("water.mat", "iron.mat")]
    ph = F.load_phantom(work / "obj.xvox", mats)
    spec = F.load_spectrum(work / "data" / "spectra" / "w200kv_2mmal.csv")
    resp = F.load_detector_response(work / "data" / "detector" / "gd2o2s_208um.csv")
    g = I.make_circular_geometry(60.0, 40.0, 24, 16, 0.1, 8)
    cfg = I.SimConfig(photons_total=20000, splitting=5, roulette_survival=0.5, roulette_wmin_rel=1e-3,
                      step_voxels=1, max_interactions=50, seed=1234)
    return X.Projector(ph, resp, ctx=X.Context(0)).run_scan(g, spec, cfg, subset, what)


@pytest.mark.parametrize("devices", [None, "0,0"])
def test_cli_simulate_matches_the_projector(tmp_path, devices):
    work, r = _run(tmp_path, ["--angles", "1:4"], {"XSCAT_DEVICES": devices} if devices else None)
    assert r.stdout.startswith("effective seed: 1234\nsimulated 3 angles in ")
    out = work / "out"
    want = _expected(work, [1, 2, 3], X.BOTH)
    for name, stack in (("primary", want.primary), ("scatter", want.scatter)):
        got = F.load_stack(out / f"{name}.xprj")
        assert np.array_equal(got.images, stack.images.astype(np.float32).astype(np.float64)), name
    rows = (out / "timing.csv").read_text().splitlines()
    assert rows[0] == "angle_idx,seconds" and [x.split(",")[0] for x in rows[1:]] == ["1", "2", "3", "total"]
    assert all(float(x.split(",")[1]) > 0 for x in rows[1:])


def test_cli_simulate_one_quantity_and_seed_override(tmp_path):
    work, r = _run(tmp_path, ["--what", "scatter", "--angles", "0,5", "--seed", "99"])
    assert r.stdout.startswith("effective seed: 99\n")
    out = work / "out"
    assert not (out / "primary.xprj").exists() and (out / "scatter.xprj").exists()
    mats = [F.load_material(work / "data" / "materials" / f) for f in ("water.mat", "iron.mat")]
    ph = F.load_phantom(work / "obj.xvox", mats)
    g = I.make_circular_geometry(60.0, 40.0, 24, 16, 0.1, 8)
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=99)
    want = X.Projector(ph, F.load_detector_response(work / "data" / "detector" / "gd2o2s_208um.csv"),
                       ctx=X.Context(0)).run_scan(
        g, F.load_spectrum(work / "data" / "spectra" / "w200kv_2mmal.csv"), cfg, [0, 5], X.SCATTER)
    got = F.load_stack(out / "scatter.xprj")
    assert np.array_equal(got.images, want.scatter.images.astype(np.float32).astype(np.float64))
