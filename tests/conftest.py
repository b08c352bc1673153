import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libbagel.so")
    config.addinivalue_line("markers", "slow: long-running (large oracle instances)")


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line)
    return rows


def spec_examples():
    out = {}
    for row in read_golden("spec_examples.txt"):
        name, value, cite = [c.strip() for c in row.split(" | ", 2)]
        out[name] = value
    return out


def small_gp_data(N=40, d=3, p=2, seed=0):
    """Random standardised-looking inputs and smooth targets for oracle self-tests."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(-2, 2, size=(N, d))
    Y = np.stack([np.sin(X[:, 0] + 0.5 * m) * 0.1 + 0.02 * X[:, -1] for m in range(p)], axis=1)
    ell = np.array([[1.0 + 0.1 * m] * (d - 1) + [0.7 * (1 + 0.1 * m)] for m in range(p)])
    s = Y.var(axis=0) + 1e-3
    noise = 1e-2 * s
    return X, Y, ell, s, noise
