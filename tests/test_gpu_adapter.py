"""The drop-in adapter: a program written against the reference's API
(tests/cpp/ref_adapter_demo.cpp, compiled with the reference headers) runs the
reference library on the CPU and, through include/xscat_b200_ref_adapter.hpp,
the B200 library, and checks they agree (exit code 0)."""
import pathlib
import subprocess

import pytest

from paper_2201_13191_b200 import inputs as I

ROOT = pathlib.Path(__file__).resolve().parents[1]
DEMO = ROOT / "oracle" / "_ref" / "ref_adapter_demo"


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [None, "0,0"])
def test_reference_api_program_on_b200(tmp_path, devices):
    """devices "0,0": XSCAT_DEVICES makes the adapter run on an xs_group (two
    contexts on the test box's one GPU): the same checks must pass."""
    import os
    if not DEMO.exists():
        pytest.skip("oracle/_ref/ref_adapter_demo not built (needs /root/reference at build time)")
    data = I.write_reference_data(tmp_path / "data")
    env = dict(os.environ)
    if devices:
        env["XSCAT_DEVICES"] = devices
    r = subprocess.run([str(DEMO), str(data)], capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout


def test_reference_data_writer_round_trips(tmp_path):
    data = I.write_reference_data(tmp_path / "data")
    for name in ("water", "aluminum", "iron"):
        m = I.load_material(data / "materials" / f"{name}.mat")
        ref = I.material(name)
        for a, b in zip(m.tables(), ref.tables()):
            assert (a.x == b.x).all() and (a.y == b.y).all()
    s = I.load_spectrum(data / "spectra" / "w200kv_2mmal.csv")
    assert (s.weight == I.spectrum("w200kv_2mmal").weight).all()
    r = I.load_detector_response(data / "detector" / "gd2o2s_208um.csv")
    assert (r.deposit.y == I.detector_response().deposit.y).all()
