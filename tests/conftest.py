import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

REFERENCE = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (build container only)")


def pytest_collection_modifyitems(config, items):
    skip_ref = pytest.mark.skip(reason="reference checkout not present (expected on the GPU box)")
    for item in items:
        if "reference" in item.keywords and not REFERENCE.exists():
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "decisions.json").read_text())


@pytest.fixture(scope="session")
def moesim():
    if not REFERENCE.exists():
        pytest.skip("reference checkout not present")
    if str(REFERENCE) not in sys.path:
        sys.path.insert(0, str(REFERENCE))
    import moesim.engine  # noqa: F401
    import moesim.tracegen  # noqa: F401
    return sys.modules["moesim"]
