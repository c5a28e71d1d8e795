import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


import pytest  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _release_device_memory():
    """Give cached device memory back after every module: the full-size goldens (C5: tens of GB
    through torch's caching allocator) would otherwise stay reserved in this process while the
    multi-process tests start their own CUDA contexts on the same GPU."""
    yield
    import sys as _sys
    torch = _sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
