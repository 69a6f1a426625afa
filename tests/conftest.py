"""Shared fixtures.  `gpu` marks tests that need a CUDA device (B200)."""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
for p in (REPO, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: large problem, minutes")


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_matrix(name):
    from golden.make_golden import SMALL
    build, bs, w, rhs_kind = SMALL[name]
    a = build()
    return a, bs, w, rhs_kind


def rel_err(x, ref):
    ref = np.asarray(ref, dtype=float)
    den = float(np.linalg.norm(ref))
    return float(np.linalg.norm(np.asarray(x) - ref)) / (den if den > 0 else 1.0)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)

# device outputs are NaN-filled before every operator runs (see device.empty)
os.environ.setdefault("TB_POISON", "1")
