import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box with -m gpu)")


def cuda_available() -> bool:
    try:
        import paper_2501_11779_b200 as gh
        return gh.lib().gh_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def need_gpu():
    if not cuda_available():
        pytest.fail("GPU test selected but no CUDA device is visible")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the in-tree extension + oracle once per session if missing (CPU-side build)."""
    so = ROOT / "paper_2501_11779_b200" / "libgh.so"
    orc = ROOT / "oracle" / "liboracle.so"
    if not so.exists() or not orc.exists():
        import __graft_entry__
        __graft_entry__.build()
