import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def built():
    """Builds libktc.so and the oracle once per session (cheap when up to date)."""
    import __graft_entry__ as g

    g.build()
    return True


@pytest.fixture(scope="session")
def backend(built):
    import paper_1703_06503_b200 as pkg

    if pkg.device_count() < 1:
        pytest.fail("GPU test without a CUDA device: " + pkg._ktc.last_error())
    be = pkg.CudaBackend(0)
    yield be
    be.close()


@pytest.fixture(scope="session")
def golden():
    import json

    return json.loads((ROOT / "tests" / "golden" / "oracle_golden.json").read_text())
