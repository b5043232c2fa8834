import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


# Randomized parity tests scale with DS_FUZZ_SCALE (default 1): a sweep runs
# e.g. DS_FUZZ_SCALE=10 for ten times the trials on fresh seeds.
FUZZ_SCALE = max(1, int(os.environ.get("DS_FUZZ_SCALE", "1")))


def fuzz_seed(base: int) -> int:
    """The test's fixed seed at scale 1, a different stream per larger scale."""
    return base if FUZZ_SCALE == 1 else base * 1000 + FUZZ_SCALE
