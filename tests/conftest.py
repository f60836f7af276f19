import gzip
import os
import shutil
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running statistical test")


@pytest.fixture(scope="session")
def port():
    from pyoracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from pyoracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        try:
            from pyoracle import build_ref
            build_ref()
        except Exception:
            pass
    if not os.path.exists(REF_SO):
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def golden_dir(tmp_path_factory):
    """Decompressed golden PSTR stores."""
    d = tmp_path_factory.mktemp("golden")
    for f in os.listdir(GOLDEN):
        if f.endswith(".pstr.gz"):
            with gzip.open(os.path.join(GOLDEN, f), "rb") as g, open(d / f[:-3], "wb") as o:
                shutil.copyfileobj(g, o)
    return d


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


@pytest.fixture(scope="session")
def ctx():
    from paper_2110_00085_b200.gpu import Context
    c = Context(0)
    yield c
    c.close()
