import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def olib():
    import vf_py

    return vf_py.oracle_lib()


@pytest.fixture(scope="session")
def rlib():
    import vf_py

    if not vf_py.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    lib = vf_py.ref_lib()
    lib.lib.vfr_set_threads(1)
    return lib
