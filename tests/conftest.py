import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small_qcqp")


@pytest.fixture(scope="session")
def golden_analytic():
    return load_golden("analytic")


@pytest.fixture(scope="session")
def golden_c0():
    return load_golden("c0")


@pytest.fixture(scope="session")
def golden_kml():
    return load_golden("kml_small")


ANALYTIC_NAMES = ("ball", "box-lp", "eq-qp", "strongly-convex")


def analytic_arrays(g, name):
    """Arrays of one analytic-suite instance (reference generate.py:195-256)."""
    return dict(Q=g[f"{name}/Q"], q=g[f"{name}/q"], r=g[f"{name}/r"], A=g[f"{name}/A"],
                b=g[f"{name}/b"], lower=g[f"{name}/lower"], upper=g[f"{name}/upper"],
                mu=float(g[f"{name}/mu"]))


@pytest.fixture(scope="session")
def golden_factored():
    return load_golden("factored_small")


# tests/golden/make_golden.py FACTORED_SMALL (kept in sync by test_factored_fixture_instance)
FACTORED_SMALL = dict(n=300, mq=4, rows=30, nnz_row=10, lin_rows=150, lin_nnz=5, seed=5, x0_scale=0.2)
