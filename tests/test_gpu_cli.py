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


def _measurement(work):
    """An 8-angle raw intensity stack (primary + smoothed scatter) and flat
    field of the fixture phantom, through REF's XPRJ1 files (f32)."""
    from test_gpu_loop import measurement
    mats = [F.load_material(work / "data" / "materials" / f) for f in ("water.mat", "iron.mat")]
    ph = F.load_phantom(work / "obj.xvox", mats)
    spec = F.load_spectrum(work / "data" / "spectra" / "w200kv_2mmal.csv")
    resp = F.load_detector_response(work / "data" / "detector" / "gd2o2s_208um.csv")
    g = I.make_circular_geometry(60.0, 40.0, 24, 16, 0.1, 8)
    raw, flat = measurement(ph, g, spec, resp, I.SimConfig(photons_total=20000, splitting=5, seed=5), True)
    F.save_stack(X.ProjectionStack(g.angles, raw), work / "raw.xprj")
    F.save_stack(X.ProjectionStack(np.zeros(1), flat[None]), work / "flat.xprj")
    return mats, spec, resp, g, F.load_stack(work / "raw.xprj", g.angles), F.load_stack(work / "flat.xprj")


def test_cli_reconstruct_matches_the_library(tmp_path):
    work = tmp_path / "cfg"
    shutil.copytree(CFG, work, ignore=shutil.ignore_patterns("out"))
    mats, spec, resp, g, raw, flat = _measurement(work)
    r = subprocess.run([str(CLI), "reconstruct", "--config", str(work / "good.ini"), "--stack",
                        str(work / "raw.xprj"), "--flat", str(work / "flat.xprj"), "--out", str(work / "v.xvol"),
                        "--dim", "16"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"wrote {work / 'v.xvol'} (16x16x16)\n"
    a = X.intensity_to_attenuation(raw.images, flat.images[0])
    want = X.fbp_reconstruct(X.ProjectionStack(g.angles, a), g, (16, 16, 16))
    got = F.load_volume(work / "v.xvol")
    assert np.array_equal(got.values, want)
    assert np.array_equal(got.voxel_size, X.default_voxel_size(g, (16, 16, 16)))


def test_cli_correct_matches_the_library(tmp_path):
    work = tmp_path / "cfg"
    shutil.copytree(CFG, work, ignore=shutil.ignore_patterns("out"))
    mats, spec, resp, g, raw, flat = _measurement(work)
    r = subprocess.run([str(CLI), "correct", "--config", str(work / "good.ini"), "--raw", str(work / "raw.xprj"),
                        "--flat", str(work / "flat.xprj")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "effective seed: 1234" and len(lines) == 4 and lines[1].startswith("iteration 1: ")
    cc = X.CorrectionConfig(n_iterations=3, simulate_every_kth_angle=2, mc_nu=12, mc_nv=8, recon_dims=(16, 16, 16),
                            n_classes=3, class_map=[X.ClassSpec(0, 0.0), X.ClassSpec(1, 1.0), X.ClassSpec(2, 7.874)],
                            sim=I.SimConfig(photons_total=20000, splitting=5, roulette_survival=0.5,
                                            roulette_wmin_rel=1e-3, step_voxels=1, max_interactions=50, seed=1234),
                            sg=X.SgFilterSpec(15, 3), sg_auto_window=True)
    want = X.run_iterative_correction(raw, flat.images[0], g, spec, resp, cc, mats, ctx=X.Context(0))
    out = work / "out"
    assert np.array_equal(F.load_volume(out / "corrected.xvol").values, want.corrected_volume)
    assert np.array_equal(F.load_stack(out / "corrected.xprj").images,
                          want.corrected_stack.images.astype(np.float32).astype(np.float64))
    rep = (out / "iterations.txt").read_text().split("\n\n")
    assert rep[0].startswith("iteration=1\nseconds_fbp=") and "negative_scatter_clamped=" in rep[2]
    for k, it in enumerate(want.reports):
        assert f"negative_scatter_clamped={it.negative_scatter_clamped}" in rep[k]
    csv_rows = (out / "summary.csv").read_text().splitlines()
    assert csv_rows[0] == ("iteration,photons,splitting,step_size,mc_time_per_projection_s,"
                           "mc_time_per_iteration_s,correction_time_per_iteration_s")
    assert [x.split(",")[:4] for x in csv_rows[1:]] == [[str(k), "20000", "5", "1"] for k in (1, 2, 3)]
