import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (still part of the default run)")


@pytest.fixture(scope="session")
def has_gpu():
    import torch
    return torch.cuda.is_available()


@pytest.fixture(scope="module", autouse=True)
def _close_cached_handles(request):
    """GPU test modules cache their library handles in a module-level `_handles` dict (one handle per
    config and flag set); each conv-net handle binds several GB of net scratch, so close them when the
    module is done instead of holding every module's handles until the process exits."""
    yield
    cache = getattr(request.module, "_handles", None)
    if isinstance(cache, dict):
        for h in cache.values():
            try:
                h.close()
            except Exception:
                pass
        cache.clear()
