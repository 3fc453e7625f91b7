"""The reference's file formats, text inputs and CLI front end on the library
(csrc/files.cpp, cli/xscat_b200.cpp), held to what
the compiled reference does with the same files
(tests/golden/files/files_golden.json, written by
tests/golden/make_files_golden.py from oracle/_ref):

* every REF-written XPRJ1 / XVOX1 / XVOL1 file loads to REF's values, and
  the library's savers reproduce REF's files byte for byte;
* every material / spectrum / response / stack / phantom / volume input,
  valid or broken, loads to REF's values or fails with REF's exact message;
* the CLI's run-configuration validation reports REF's problem list, its
  usage errors and exit codes are REF's (tools/main.cpp), and `inspect`
  prints REF's header lines and slice exports.
No GPU: `simulate` up to the device call; tests/test_gpu_cli.py runs it.
"""
import json
import pathlib
import subprocess

import numpy as np
import pytest

from paper_2201_13191_b200 import files as F
from paper_2201_13191_b200 import inputs as I
from paper_2201_13191_b200.projector import ProjectionStack
import paper_2201_13191_b200 as X

ROOT = pathlib.Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden" / "files"
GOLD = json.loads((OUT / "files_golden.json").read_text())
CLI = ROOT / "paper_2201_13191_b200" / "bin" / "xscat_b200"


def unhex(v):
    return np.array([float.fromhex(x) for x in v])


def expect_error(case, fn):
    with pytest.raises(I.XscatError) as e:
        fn()
    assert str(e.value) == case["error"].replace("{out}", str(OUT))


# ----------------------------------------------------------- REF-written files
def test_ref_written_files_load_and_save_byte_identical(tmp_path):
    w = GOLD["stack_written"]
    s = F.load_stack(OUT / "ref_stack.xprj")
    assert s.images.shape == (w["n"], w["nv"], w["nu"])
    # REF narrows to f32 on save and widens on load
    assert np.array_equal(s.images.ravel(), unhex(w["images"]).astype(np.float32).astype(np.float64))
    F.save_stack(ProjectionStack(np.zeros(w["n"]), unhex(w["images"]).reshape(s.images.shape)), tmp_path / "s.xprj")
    assert (tmp_path / "s.xprj").read_bytes() == (OUT / "ref_stack.xprj").read_bytes()

    p = GOLD["phantom_written"]
    ph = F.load_phantom(OUT / "ref_phantom.xvox", [I.material("water"), I.material("iron")])
    assert list(ph.dims) == p["dims"] and ph.material_id.tolist() == p["ids"]
    assert np.array_equal(ph.density, unhex(p["density"]).astype(np.float32))
    assert np.array_equal(ph.voxel_size, unhex(p["voxel_size"])) and np.array_equal(ph.origin, unhex(p["origin"]))
    F.save_phantom(ph, tmp_path / "p.xvox")
    assert (tmp_path / "p.xvox").read_bytes() == (OUT / "ref_phantom.xvox").read_bytes()
    h = F.load_phantom_header(OUT / "ref_phantom.xvox")
    assert h.material_count == p["n_materials"] and list(h.dims) == p["dims"]

    v = GOLD["volume_written"]
    vol = F.load_volume(OUT / "ref_volume.xvol")
    assert list(vol.dims) == v["dims"] and np.array_equal(vol.voxel_size, unhex(v["voxel_size"]))
    assert np.array_equal(vol.values.ravel(), unhex(v["values"]).astype(np.float32))
    F.save_volume(vol, tmp_path / "v.xvol")
    assert (tmp_path / "v.xvol").read_bytes() == (OUT / "ref_volume.xvol").read_bytes()


# ------------------------------------------------------------- binary inputs
@pytest.mark.parametrize("name", sorted(GOLD["stack"]))
def test_stack_inputs(name):
    case, path = GOLD["stack"][name], OUT / "inputs" / name
    if not case["ok"]:
        return expect_error(case, lambda: F.load_stack(path))
    s = F.load_stack(path)
    assert s.images.shape == (case["n"], case["nv"], case["nu"])
    assert np.array_equal(s.images.ravel(), unhex(case["images"]))


@pytest.mark.parametrize("name", sorted(GOLD["phantom"]))
def test_phantom_inputs(name):
    case, path = GOLD["phantom"][name], OUT / "inputs" / name
    mats = [I.material("water")] * case["files"]
    if not case["ok"]:
        return expect_error(case, lambda: F.load_phantom(path, mats))
    ph = F.load_phantom(path, mats)
    assert list(ph.dims) == case["dims"] and ph.material_id.tolist() == case["ids"]
    assert np.array_equal(ph.density, unhex(case["density"]).astype(np.float32))


@pytest.mark.parametrize("name", sorted(GOLD["volume"]))
def test_volume_inputs(name):
    case, path = GOLD["volume"][name], OUT / "inputs" / name
    if not case["ok"]:
        return expect_error(case, lambda: F.load_volume(path))
    v = F.load_volume(path)
    assert list(v.dims) == case["dims"] and np.array_equal(v.voxel_size, unhex(case["voxel_size"]))
    assert np.array_equal(v.values.ravel(), unhex(case["values"]).astype(np.float32))


# --------------------------------------------------------------- text inputs
@pytest.mark.parametrize("name", sorted(GOLD["material"]))
def test_material_inputs(name):
    case, path = GOLD["material"][name], OUT / "inputs" / name
    if not case["ok"]:
        return expect_error(case, lambda: F.load_material(path))
    m = F.load_material(path)
    assert m.z_eff == float.fromhex(case["z_eff"]) and m.density_ref == float.fromhex(case["density"])
    got = []
    for t in (m.mu, m.sigma_incoh, m.sigma_coh, m.sigma_pe, m.s_factor, m.f_factor):
        got += [t.x, t.y]
    assert [t.size for t in got[::2]] == case["counts"]
    assert np.array_equal(np.concatenate(got), unhex(case["xy"]))


@pytest.mark.parametrize("name", sorted(GOLD["spectrum"]))
def test_spectrum_inputs(name):
    case, path = GOLD["spectrum"][name], OUT / "inputs" / f"spec_{name}"
    if not case["ok"]:
        return expect_error(case, lambda: F.load_spectrum(path))
    s = F.load_spectrum(path)
    assert np.array_equal(s.energy_kev, unhex(case["e"])) and np.array_equal(s.weight, unhex(case["w"]))


@pytest.mark.parametrize("name", sorted(GOLD["response"]))
def test_response_inputs(name):
    case, path = GOLD["response"][name], OUT / "inputs" / f"resp_{name}"
    if not case["ok"]:
        return expect_error(case, lambda: F.load_detector_response(path))
    r = F.load_detector_response(path)
    assert np.array_equal(r.dqe.x, unhex(case["e"])) and np.array_equal(r.dqe.y, unhex(case["dqe"]))
    assert np.array_equal(r.deposit.y, unhex(case["deposit"]))


def test_bundled_tables_round_trip_through_the_file_loaders(tmp_path):
    """The bundled reference data written out and read back by the library's
    loaders is the bundle, bit for bit (the CLI's inputs)."""
    root = I.write_reference_data(tmp_path)
    for name in ("water", "aluminum", "iron", "cement", "gd2o2s"):
        a, b = F.load_material(root / "materials" / f"{name}.mat"), I.material(name)
        for f in ("mu", "sigma_incoh", "sigma_coh", "sigma_pe", "s_factor", "f_factor"):
            assert np.array_equal(getattr(a, f).x, getattr(b, f).x)
            assert np.array_equal(getattr(a, f).y, getattr(b, f).y)
        assert (a.name, a.z_eff, a.density_ref) == (b.name, b.z_eff, b.density_ref)


# ----------------------------------------------------------------------- CLI
def cli(*args, cwd=None):
    assert CLI.exists(), f"{CLI} not built (make cli / __graft_entry__.build())"
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=120)


@pytest.mark.parametrize("name", sorted(GOLD["config"]))
def test_cli_config_validation_matches_reference(name):
    case, cfg = GOLD["config"][name], OUT / "cfg"
    # (an invalid --what stops a valid configuration after its inputs load,
    # before any device work or output in the fixture tree)
    r = cli("simulate", "--config", cfg / name, "--what", "nothing")
    if not case["ok"]:  # REF parse_ini throws: a runtime error
        assert r.returncode == 3
        assert r.stderr == "error: " + case["error"].replace("{dir}", str(cfg)) + "\n"
    elif case["problems"]:
        probs = [p.replace("{dir}", str(cfg)) for p in case["problems"]]
        assert r.returncode == 2
        assert r.stderr == f"config validation failed ({len(probs)} problems):\n" + "".join(
            f"  - {p}\n" for p in probs)
    else:  # valid: inputs load and the seed is reported
        assert r.returncode == 2 and r.stdout == "effective seed: 1234\n"
        assert r.stderr == "--what must be primary|scatter|both\n"


def test_cli_usage_errors_and_overrides():
    good = OUT / "cfg" / "good.ini"
    r = cli("simulate", "--config", good, "--seed", 77, "--what", "everything")
    assert r.returncode == 2 and r.stdout == "effective seed: 77\n"
    assert r.stderr == "--what must be primary|scatter|both\n"
    r = cli("simulate", "--config", good, "--angles", "5:5")
    assert r.returncode == 2 and r.stderr == "usage error: empty angle list\n"
    r = cli("simulate", "--config", good, "--angles", "1,9")
    assert r.returncode == 2 and r.stderr == "angle index 9 out of range\n"
    r = cli("simulate", "--config", OUT / "cfg" / "absent.ini")
    assert r.returncode == 3 and r.stderr == f"error: cannot open config file {OUT / 'cfg' / 'absent.ini'}\n"
    assert cli("simulate").returncode == 2
    assert cli("frobnicate").returncode == 2
    r = cli("inspect", "--file", OUT / "cfg" / "good.ini")
    assert r.returncode == 2 and r.stderr == "unknown file type (expected .xvox/.xprj/.xvol)\n"


def test_cli_inspect_prints_reference_headers(tmp_path):
    p = GOLD["phantom_written"]
    vs, o = unhex(p["voxel_size"]), unhex(p["origin"])
    r = cli("inspect", "--file", OUT / "ref_phantom.xvox")
    assert r.returncode == 0
    assert r.stdout == ("XVOX1 phantom: dims %d x %d x %d, voxel %.4f x %.4f x %.4f cm, "
                        "origin (%.3f, %.3f, %.3f), %u materials\n" % (*p["dims"], *vs, *o, p["n_materials"]))
    r = cli("inspect", "--file", OUT / "ref_stack.xprj")
    assert r.stdout == "XPRJ1 stack: 5 x 3 pixels, 2 angles\n"
    r = cli("inspect", "--file", OUT / "inputs" / "short_pixels.xprj")
    assert r.returncode == 3 and r.stderr == f"error: {OUT / 'inputs' / 'short_pixels.xprj'}: truncated pixel data\n"

    v = GOLD["volume_written"]
    vals = unhex(v["values"]).astype(np.float32).reshape(2, 3, 4)
    r = cli("inspect", "--file", OUT / "ref_volume.xvol", "--slice", 1, "--export", tmp_path / "s.csv")
    assert r.stdout == ("XVOL1 volume: dims 4 x 3 x 2, voxel 0.1250 x 0.3000 x 0.7000 cm\n"
                        f"wrote slice 1 to {tmp_path / 's.csv'}\n")
    rows = (tmp_path / "s.csv").read_text().splitlines()
    assert rows == [",".join("%g" % float(x) for x in vals[1, y]) for y in range(3)]  # ostream default: %g
    cli("inspect", "--file", OUT / "ref_volume.xvol", "--export", tmp_path / "m.pgm")  # middle slice
    pgm = (tmp_path / "m.pgm").read_bytes()
    head = b"P5\n4 3\n255\n"
    s = vals[1].astype(np.float64)
    lo, hi = s.min(), s.max()
    want = np.floor(np.clip((s - lo) / (hi - lo), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    assert pgm[:len(head)] == head and np.array_equal(np.frombuffer(pgm[len(head):], np.uint8), want.ravel())
    r = cli("inspect", "--file", OUT / "ref_volume.xvol", "--slice", 5, "--export", tmp_path / "x.csv")
    assert r.returncode == 3 and r.stderr == "error: volume_slice_z: slice index out of range\n"


def test_cli_reconstruct_and_correct_usage_and_input_errors():
    good, stack = OUT / "cfg" / "good.ini", OUT / "ref_stack.xprj"  # a 2-image stack; good.ini has 8 angles
    assert cli("reconstruct", "--config", good, "--stack", stack).returncode == 2  # --out missing
    assert cli("correct", "--config", good, "--raw", stack).returncode == 2  # --flat missing
    r = cli("reconstruct", "--config", good, "--stack", stack, "--out", "/tmp/never.xvol")
    assert r.returncode == 3 and r.stderr == f"error: {stack}: angle list size does not match file (8 vs 2)\n"
    r = cli("correct", "--config", good, "--raw", stack, "--flat", stack)
    assert r.returncode == 3 and r.stdout == "effective seed: 1234\n"
    assert r.stderr == f"error: {stack}: angle list size does not match file (8 vs 2)\n"


@pytest.mark.parametrize("kind", ["empty", "cube", "cylinder", "rods", "cylinder-head-like"])
def test_cli_phantom_matches_the_reference_generators(tmp_path, kind):
    """`phantom` writes the XVOX1 file of REF's generators (synthetic.cpp,
    mirrored by paper_2201_13191_b200.synthetic, which tests/test_inputs.py
    pins to the compiled reference) with REF's materials and defaults."""
    from paper_2201_13191_b200 import synthetic as S
    mdir = I.write_reference_data(tmp_path / "data") / "materials"
    out = tmp_path / "p.xvox"
    r = cli("phantom", "--kind", kind, "--out", out, "--dim", 24, "--voxel-cm", 0.25, "--radius-cm", 2.5,
            "--height-cm", 4.0, "--rods", 5, "--materials-dir", mdir)
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"wrote {out} (24^3 voxels of 0.250 cm)\n"
    m = {k: F.load_material(mdir / f"{k}.mat") for k in ("water", "cement", "iron", "aluminum")}
    if kind == "empty":
        ph = I.make_empty_phantom(24, 24, 24, (0.25,) * 3, [m["water"]])
    elif kind == "cube":
        ph = S.make_cube_phantom(24, 0.25, 5.0, m["water"], 1.0)
    elif kind == "cylinder":
        ph = S.make_cylinder_phantom(24, 0.25, 2.5, 4.0, m["water"], 1.0)
    elif kind == "rods":
        ph = S.make_rods_phantom(24, 0.25, 2.5, 4.0, m["cement"], m["cement"].density_ref, 5, 2.5 * 0.08,
                                 2.5 * 0.6, m["iron"], m["iron"].density_ref)
    else:
        ph = S.make_cylinder_head_phantom(24, 0.25, m["aluminum"], m["aluminum"].density_ref, m["iron"],
                                          m["iron"].density_ref)
    F.save_phantom(ph, tmp_path / "want.xvox")
    assert out.read_bytes() == (tmp_path / "want.xvox").read_bytes()


def test_cli_phantom_errors():
    r = cli("phantom", "--kind", "torus", "--out", "/tmp/never.xvox")
    assert r.returncode == 2 and r.stderr.startswith("unknown phantom kind 'torus'")
    r = cli("phantom", "--kind", "rods", "--out", "/tmp/never.xvox", "--rods", 0,
            "--materials-dir", OUT / "cfg" / "data" / "materials")
    assert r.returncode == 3 and r.stderr == "error: rods phantom: need at least one rod\n"
    r = cli("phantom", "--kind", "cube", "--out", "/tmp/never.xvox", "--materials-dir", "/nonexistent")
    assert r.returncode == 3 and r.stderr == "error: cannot open material file /nonexistent/water.mat\n"


def test_cli_metrics_match_the_reference_formulas(tmp_path):
    """`metrics` (REF metrics.cpp): MSE and NCC of two images, CNR of two
    rectangles (population statistics), a row-band profile."""
    a, b = F.load_stack(OUT / "ref_stack.xprj").images  # two 3 x 5 images
    a = np.round(np.abs(np.log10(a + 1e-300)), 3)
    b = a[::-1].copy() * 0.5 + 1.0
    F.save_stack(X.ProjectionStack(np.zeros(2), np.stack([a, b])), tmp_path / "s.xprj")
    F.save_stack(X.ProjectionStack(np.zeros(1), b[None]), tmp_path / "t.xprj")
    A32 = np.asarray(a, np.float32).astype(np.float64)
    B32 = np.asarray(b, np.float32).astype(np.float64)
    r = cli("metrics", "--a", tmp_path / "s.xprj", "--b", tmp_path / "t.xprj", "--roi", "0,0,1,2,2,2,1,3",
            "--profile", "0,2", "--profile-out", tmp_path / "p.csv")
    assert r.returncode == 0, r.stderr
    vals = dict(line.split(",") for line in r.stdout.splitlines()[1:])
    d = A32 - B32
    assert float(vals["mse"]) == pytest.approx(float("%g" % (np.sum(d * d) / d.size)), rel=1e-12)
    x, y = A32 - A32.mean(), B32 - B32.mean()
    assert float(vals["ncc"]) == pytest.approx(float("%g" % ((x * y).sum() / np.sqrt((x * x).sum() * (y * y).sum()))),
                                               rel=1e-12)
    roi, bg = A32[0:1, 0:2], A32[2:3, 2:5]
    want = abs(roi.mean() - bg.mean()) / np.sqrt(((bg - bg.mean()) ** 2).mean())
    assert float(vals["cnr"]) == pytest.approx(float("%g" % want), rel=1e-12)
    prof = [line.split(",") for line in (tmp_path / "p.csv").read_text().splitlines()[1:]]
    assert [int(c) for c, _ in prof] == list(range(5))
    assert [float(v) for _, v in prof] == pytest.approx([float("%g" % v) for v in A32[0:2].mean(axis=0)], rel=1e-12)
    r = cli("metrics", "--a", tmp_path / "s.xprj", "--roi", "0,0,2,2,1,1,2,2")
    assert r.returncode == 3 and r.stderr == "error: cnr: ROI and background rectangles overlap\n"
    r = cli("metrics", "--a", tmp_path / "s.xprj", "--profile", "1")
    assert r.returncode == 2 and r.stderr == "--profile wants row0,row1[,col0,col1]\n"
