import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def c1_graph():
    import synth
    return synth.build_host_graph(synth.config("C1"))


@pytest.fixture(scope="session")
def c2_graph():
    import synth
    return synth.build_host_graph(synth.config("C2"))


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """After each GPU test: collect reference cycles (contexts <-> blocks) and return the
    freed device memory, so that full-size shards (C4: 36 GB, C5) of earlier tests do not
    accumulate on the 180 GB device."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import gc
    gc.collect()
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    except Exception:
        pass
