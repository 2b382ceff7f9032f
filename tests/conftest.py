import os
import sys

import pytest

# The single-GPU tensor-parallel / pipeline emulation runs t <= 8 ranks on t streams (host-ordered:
# no kernel waits on another rank's launch).  One hardware work queue per stream keeps a rank's
# queued launches from serialising behind a peer's (the default is 8 queues, shared with torch's
# own streams).  Must be set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


@pytest.fixture(autouse=True)
def _restore_library_options(request):
    """sm_set_option knobs are process-wide: restore the library defaults after every GPU test
    so a test that flips one (gemm_pair, fused_epilogue, pdl, ...) cannot leak it into the next."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    mod = sys.modules.get("paper_2506_01986_b200")
    if mod is not None and getattr(mod, "_lib", None) is not None:
        mod.reset_options()
