import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"
REFERENCE_SRC = Path(os.environ.get("MESHDIST_REFERENCE", "/root/reference/pkg/src"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and libgdist.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden.npz")


@pytest.fixture(scope="session")
def golden_meta():
    with open(GOLDEN / "golden.json") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from oracle import meshdist_oracle

    return meshdist_oracle


@pytest.fixture(scope="session")
def reference():
    """The live reference package: /root/reference in the build container, or
    the unmodified copy pip-installed into baseline/_ref (travels to the GPU box)."""
    src = next((s for s in (REFERENCE_SRC, REPO / "baseline" / "_ref") if (s / "meshdist" / "__init__.py").exists()),
               None)
    if src is None:
        pytest.skip("reference package not available here")
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "meshdist_ref", src / "meshdist" / "__init__.py",
        submodule_search_locations=[str(src / "meshdist")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["meshdist_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="session")
def md():
    import paper_2411_11244_b200 as md

    return md


@pytest.fixture(scope="session")
def gpu(md):
    """Skip-free on the GPU box: a gpu test that cannot reach the device fails."""
    from paper_2411_11244_b200 import _lib

    _lib.require_device()
    return True
