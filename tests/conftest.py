import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    # the oracle is test infrastructure: build it on demand (gcc only)
    if not (ROOT / "oracle" / "liboracle.so").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def orc():
    import oracle_lib
    return oracle_lib.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle_lib
    r = oracle_lib.ref()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    return r
