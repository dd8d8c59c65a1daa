import os
import sys

# streams blocked on peer-exchange flags must not share a hardware work queue
# with streams that have to progress (paper_2008_11480_b200/peer.py); set
# before CUDA initialises
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture
def rng():
    return np.random.default_rng(20260808)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_fro(x, ref):
    x = np.asarray(x)
    ref = np.asarray(ref)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (den if den > 0 else 1.0))


def release_gpu_memory():
    """Hand cached device memory back before a test starts other GPU processes
    (the caching allocator of this process may still hold tens of GB from the
    full-size tests)."""
    import gc

    gc.collect()
    try:
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            from paper_2008_11480_b200 import _lib

            _lib.call("si_trim", _lib.handle(0))
    except Exception:  # noqa: BLE001 -- best effort
        pass


# Long host-bound oracle runs started as soon as the test session knows it will
# need them, so they overlap the GPU tests (tests/fullsize_c4_worker.py).
BACKGROUND = {}


def pytest_collection_finish(session):
    if session.config.option.collectonly:
        return
    try:
        import torch

        if not torch.cuda.is_available():
            return
    except ImportError:
        return
    if any(item.nodeid.endswith("test_c4_full_size_two_iterations_vs_oracle")
           for item in session.items):
        out = tempfile.mkdtemp(prefix="si_c4_fullsize_")
        proc = subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "fullsize_c4_worker.py"),
                                 out], cwd=ROOT)
        BACKGROUND["c4_fullsize"] = (proc, out)
