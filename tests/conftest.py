import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libspk CUDA library")
    config.addinivalue_line("markers", "slow: longer oracle runs")


@pytest.fixture(scope="session")
def spk():
    """The CUDA binding; GPU tests fail loudly (no fallback) if the library is missing."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected on a host without CUDA")
    from paper_2301_13659_b200 import spk as _spk

    _spk.lib()  # raises if libspk.so is absent
    return _spk


def pytest_sessionfinish(session, exitstatus):
    """Write the parity report (counts of near-threshold / near-tie cases, error percentiles)
    gathered by the GPU parity tests (tests/parity.py ParityReport)."""
    from parity import ParityReport

    path = os.environ.get("SPK_PARITY_REPORT", str(ROOT / "profiles" / "parity_report.json"))
    ParityReport.dump(path)
