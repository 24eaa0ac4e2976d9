import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def ladder():
    return {e["name"]: e for e in load_golden("jacobi_ladder.json")["entries"]}


@pytest.fixture(scope="session")
def small_arrays():
    with np.load(os.path.join(GOLDEN, "jacobi_small.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o


def kwargs_of(entry):
    kw = dict(entry["kwargs"])
    kw.pop("clock", None)
    if "grid" in kw:
        kw["grid"] = tuple(kw["grid"])
    return kw
