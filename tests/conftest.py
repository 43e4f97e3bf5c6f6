import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_sessionstart(session):
    """A fresh checkout has no libtadakv_b200.so (built artefacts are not in git): build it (nvcc cross-compiles
    sm_100a without a GPU) so the ABI / host tests load the real library."""
    import shutil
    import subprocess

    lib = os.path.join(ROOT, "paper_2506_04642_b200", "libtadakv_b200.so")
    if not os.path.exists(lib) and shutil.which("make") and os.path.exists("/usr/local/cuda/bin/nvcc"):
        subprocess.run(["make", "-C", ROOT, "-j8"], check=False, stdout=subprocess.DEVNULL)


def _has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
