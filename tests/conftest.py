import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


def load_variants():
    """Golden variants written by tests/golden/make_golden.py (reference run_call)."""
    import json
    data = np.load(os.path.join(GOLDEN, "variants.npz"))
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        plans = json.load(f)
    cases = []
    for name in sorted(plans):
        meta = plans[name]
        cases.append(dict(
            name=name, kind=meta["kind"], params=meta["params"], shape=meta["shape"],
            pad=meta["pad"], plan=meta["plan"],
            a=data[name + "__a"], b=data[name + "__b"] if name + "__b" in data else None,
            c=data[name + "__c"], out=data[name + "__out"]))
    return cases
