import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size parity cases")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt .so)")
    return Reference()


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def fixtures():
    z = np.load(os.path.join(GOLDEN, "fixtures.npz"))
    meta = json.loads(bytes(z["__meta__"]).decode())
    out = []
    for m in meta:
        n = m["name"]
        out.append(dict(m, x=z[f"{n}__x"], blob=bytes(z[f"{n}__blob"]), dec0=z[f"{n}__dec0"],
                        dec1=z[f"{n}__dec1"]))
    return out


@pytest.fixture(scope="session")
def gpu_lib():
    """Builds (if stale) and loads the CUDA extension; fails loudly without it."""
    from paper_2011_09017_b200 import build as B
    B.build()
    from paper_2011_09017_b200 import _native
    return _native.load()
