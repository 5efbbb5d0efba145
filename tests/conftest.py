import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
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


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, name)))


def reference_fkc():
    """The reference package ``fkc`` (region / field), imported from the
    offline install ``baseline/_ref`` (travels to the GPU box) or, in the
    build container only, from /root/reference/pkg/src.  None if neither is
    present.  Test infrastructure: the product never imports it."""
    import importlib
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "fkc")):
            if path not in sys.path:
                sys.path.append(path)
            try:
                return importlib.import_module("fkc.field"), importlib.import_module("fkc.region")
            except ImportError:  # pragma: no cover
                return None
    return None
