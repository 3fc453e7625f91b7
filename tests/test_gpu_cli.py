"""Integration example (examples/ref_cli_integration.cpp; not a product
component, SURVEY.md §8(f) rank 4 is not claimed): the reference CLI's compute commands on the B200: REF's INI run configuration, input loaders and file
formats (XVOX1 phantom in, XPRJ1 stacks / XVOL1 volume / timing.csv out), with
every computation through the adapter.  The stacks it writes must equal the
Python API's results for the same inputs, rounded to float32 like REF's
save_stack (detector_image.cpp:33-51)."""
import pathlib
import subprocess

import numpy as np
import pytest

import paper_2201_13191_b200 as X
from paper_2201_13191_b200 import inputs as I

ROOT = pathlib.Path(__file__).resolve().parents[1]
CLI = ROOT / "oracle" / "_ref" / "xscat_b200_cli"

pytestmark = pytest.mark.gpu


def read_xprj(path):
    """REF XPRJ1 (detector_image.cpp:33-51): magic, u32 nu, nv, n; f32 images."""
    b = pathlib.Path(path).read_bytes()
    assert b[:5] == b"XPRJ1"
    nu, nv, n = np.frombuffer(b[5:17], np.uint32)
    return np.frombuffer(b[17:], np.float32).reshape(n, nv, nu)


def read_xvox(path, materials):
    """REF XVOX1 (phantom.cpp:74-92)."""
    b = pathlib.Path(path).read_bytes()
    assert b[:5] == b"XVOX1"
    dims = np.frombuffer(b[5:17], np.uint32).astype(int)
    vs = np.frombuffer(b[17:41], np.float64)
    org = np.frombuffer(b[41:65], np.float64)
    n = int(np.prod(dims))
    ids = np.frombuffer(b[69:69 + n], np.uint8)
    dens = np.frombuffer(b[69 + n:69 + 5 * n], np.float32)
    return I.VoxelPhantom(tuple(dims), tuple(vs), tuple(org), ids, dens, [None] + materials)


def test_cli_simulate_matches_api(tmp_path):
    if not CLI.exists():
        pytest.skip("oracle/_ref/xscat_b200_cli not built (needs /root/reference at build time)")
    data = I.write_reference_data(tmp_path / "data")
    xvox = tmp_path / "obj.xvox"
    r = subprocess.run([str(CLI), "synth-phantom", "rods", "32", "0.3", str(data / "materials"), str(xvox)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    ini = tmp_path / "run.ini"
    ini.write_text(f"""[paths]
materials_dir = {data / 'materials'}
materials = water.mat, aluminum.mat
spectrum = {data / 'spectra' / 'w200kv_2mmal.csv'}
detector_response = {data / 'detector' / 'gd2o2s_208um.csv'}
phantom = {xvox}
output_dir = {tmp_path / 'out'}

[geometry]
sdd_cm = 60.0
sod_cm = 40.0
det_nu = 32
det_nv = 24
pixel_pitch_cm = 0.5
n_angles = 8

[sim]
photons_total = 20000
splitting = 5
seed = 77

[run]
threads = 4
""")
    r = subprocess.run([str(CLI), str(ini), "simulate", "--what", "both", "--angles", "0:3"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = tmp_path / "out"
    prim, scat = read_xprj(out / "primary.xprj"), read_xprj(out / "scatter.xprj")
    assert prim.shape == scat.shape == (3, 24, 32)
    timing = (out / "timing.csv").read_text().splitlines()
    assert timing[0] == "angle_idx,seconds" and len(timing) == 5 and timing[-1].startswith("total,")
    mats = [I.load_material(data / "materials" / m) for m in ("water.mat", "aluminum.mat")]
    ph = read_xvox(xvox, mats)
    g = I.make_circular_geometry(60.0, 40.0, 32, 24, 0.5, 8)
    spec = I.load_spectrum(data / "spectra" / "w200kv_2mmal.csv")
    resp = I.load_detector_response(data / "detector" / "gd2o2s_208um.csv")
    cfg = I.SimConfig(photons_total=20000, splitting=5, seed=77)
    scan = X.run_scan(ph, g, spec, resp, cfg, [0, 1, 2], X.BOTH)
    assert np.array_equal(prim, scan.primary.images.astype(np.float32))
    assert np.array_equal(scat, scan.scatter.images.astype(np.float32))
    assert scat.sum() > 0
    # usage errors exit 2 like REF's CLI
    r = subprocess.run([str(CLI), str(ini), "simulate", "--angles", "7:9"], capture_output=True, text=True)
    assert r.returncode == 2 and "out of range" in r.stderr


def write_xprj(path, images):
    """REF XPRJ1 writer (detector_image.cpp:33-51): images rounded to float32."""
    a = np.ascontiguousarray(images, np.float32)
    n, nv, nu = a.shape
    pathlib.Path(path).write_bytes(b"XPRJ1" + np.array([nu, nv, n], np.uint32).tobytes() + a.tobytes())


def read_xvol(path):
    """REF XVOL1 (volume.hpp:33-35): magic, u32 nx, ny, nz, f64 voxel x3, f32 data."""
    b = pathlib.Path(path).read_bytes()
    assert b[:5] == b"XVOL1"
    nx, ny, nz = np.frombuffer(b[5:17], np.uint32)
    return np.frombuffer(b[41:], np.float32).reshape(nz, ny, nx)


def test_cli_reconstruct_and_correct_match_api(tmp_path):
    if not CLI.exists():
        pytest.skip("oracle/_ref/xscat_b200_cli not built (needs /root/reference at build time)")
    data = I.write_reference_data(tmp_path / "data")
    xvox = tmp_path / "obj.xvox"
    assert subprocess.run([str(CLI), "synth-phantom", "cylinder", "24", "0.3", str(data / "materials"), str(xvox)],
                          capture_output=True, timeout=120).returncode == 0
    mats = [I.load_material(data / "materials" / "water.mat")]
    ph = read_xvox(xvox, mats)
    g = I.make_circular_geometry(60.0, 40.0, 24, 24, 0.5, 36)
    spec = I.load_spectrum(data / "spectra" / "mono_100kev.csv")
    resp = I.load_detector_response(data / "detector" / "gd2o2s_208um.csv")
    sim = I.SimConfig(photons_total=2000, splitting=4, seed=99)
    # scatter-free "measurement" (REF test_correction.cpp:118-160) and flat field
    raw = X.run_scan(ph, g, spec, resp, sim, list(range(36)), X.PRIMARY).primary.images
    empty = I.make_empty_phantom(*ph.dims, ph.voxel_size, mats)
    flat = X.simulate_primary(empty, g, 0, spec, resp, sim)
    write_xprj(tmp_path / "raw.xprj", raw)
    write_xprj(tmp_path / "flat.xprj", flat[None])
    ini = tmp_path / "run.ini"
    ini.write_text(f"""[paths]
materials_dir = {data / 'materials'}
materials = water.mat
spectrum = {data / 'spectra' / 'mono_100kev.csv'}
detector_response = {data / 'detector' / 'gd2o2s_208um.csv'}
phantom = {xvox}
output_dir = {tmp_path / 'out'}

[geometry]
sdd_cm = 60.0
sod_cm = 40.0
det_nu = 24
det_nv = 24
pixel_pitch_cm = 0.5
n_angles = 36

[sim]
photons_total = 2000
splitting = 4
seed = 99

[correction]
n_iterations = 1
simulate_every_kth_angle = 2
mc_nu = 12
mc_nv = 12
recon_dim = 24
n_classes = 2
class_map = air:0, water:1.0
""")
    raw32 = raw.astype(np.float32).astype(np.float64)
    flat32 = flat.astype(np.float32).astype(np.float64)
    # reconstruct: ln(flat / raw) then FDK, like REF tools/main.cpp:132-150
    r = subprocess.run([str(CLI), str(ini), "reconstruct", str(tmp_path / "raw.xprj"), "--flat",
                        str(tmp_path / "flat.xprj"), str(tmp_path / "vol.xvol"), "16"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    a = X.intensity_to_attenuation(raw32, flat32)
    want = X.fbp_reconstruct(X.ProjectionStack(g.angles, a), g, (16, 16, 16))
    assert np.array_equal(read_xvol(tmp_path / "vol.xvol"), want)
    # correct: the whole loop (REF tools/main.cpp:152-180)
    r = subprocess.run([str(CLI), str(ini), "correct", str(tmp_path / "raw.xprj"), str(tmp_path / "flat.xprj")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    cfg = X.CorrectionConfig(n_iterations=1, simulate_every_kth_angle=2, mc_nu=12, mc_nv=12, recon_dims=(24, 24, 24),
                             n_classes=2, class_map=[X.ClassSpec(0, 0.0), X.ClassSpec(1, 1.0)], sim=sim)
    res = X.run_iterative_correction(X.ProjectionStack(g.angles, raw32), flat32, g, spec, resp, cfg, mats)
    assert np.array_equal(read_xvol(tmp_path / "out" / "corrected.xvol"), res.corrected_volume)
    rep = (tmp_path / "out" / "reports.txt").read_text()
    assert "iteration=1" in rep and "ncc_to_previous=" in rep
