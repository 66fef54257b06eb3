import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

try:  # numpy may already be imported by a plugin: pin BLAS threads explicitly
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
except Exception:  # pragma: no cover
    pass

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_kernel(g):
    from oracle import ifmm_oracle as O
    return O.KernelSpec(str(g["kernel"]), a=float(g["a"]), scale=float(g["scale"]), shift=float(g["shift"]))


@pytest.fixture(autouse=True)
def _release_device_memory(request):
    """GPU tests: drop the previous test's stores / factorizations (reference cycles wait
    for the collector otherwise) so the next test starts with the whole device."""
    yield
    if request.node.get_closest_marker("gpu") is not None:
        import gc
        gc.collect()
