import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def _gpu_count():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # noqa: BLE001
        return 0


def pytest_collection_modifyitems(config, items):
    n = _gpu_count()
    skip_multi = pytest.mark.skip(reason="needs >= 2 GPUs")
    for item in items:
        if "multigpu" in item.keywords and n < 2:
            item.add_marker(skip_multi)
