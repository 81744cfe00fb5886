import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    # Build (or confirm up to date) the product library and the CPU checker.
    # _build.py is loaded by path: importing the package needs the library it builds.
    import importlib.util
    spec = importlib.util.spec_from_file_location("_cf_build", ROOT / "paper_1803_02156_b200" / "_build.py")
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)
    _build.build_library()
    _build.build_oracle()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
