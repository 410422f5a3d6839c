import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

try:
    import hypothesis

    hypothesis.settings.register_profile("b200", deadline=None, max_examples=40)
    hypothesis.settings.load_profile("b200")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json
    return json.loads((ROOT / "tests" / "golden" / "reference_frames.json").read_text())


@pytest.fixture(scope="session")
def built_lib():
    from paper_1908_01906_b200 import _build
    _build.build_library()
    _build.build_oracle()
    return True


@pytest.fixture(scope="session")
def built_oracle():
    from paper_1908_01906_b200 import _build
    _build.build_oracle()
    return True


@pytest.fixture(scope="session")
def B(built_lib):
    import paper_1908_01906_b200 as B
    return B
