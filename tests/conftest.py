import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def ctx():
    if not gpu_available():
        pytest.skip("no CUDA device")
    from paper_2601_17196_b200 import pot
    return pot.Context(0)


@pytest.fixture(scope="session", autouse=True)
def oracle_all_threads():
    """The CPU oracle (test infrastructure) on every host thread: its results
    do not depend on the thread count (fixed per-row / per-column sums,
    oracle/pot_oracle.hpp), only the wall time of the parity tests does."""
    try:
        from oracle import binding
        binding.lib().oracle_set_threads(os.cpu_count() or 1)
    except Exception:  # oracle not built: the tests that need it fail on their own
        pass
    yield
