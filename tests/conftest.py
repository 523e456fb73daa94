import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # build (no-op when up to date): the .so files are git-ignored
    r = subprocess.run(["make", "-s", "-j8", os.environ.get("DMOE_MAKE_TARGET", "all")], cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        raise pytest.UsageError("make failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
