"""Config-3 (factored Q_i = R_i^T R_i + sparse linear block) oracle pins.

The reference cannot hold a factored operator, so the golden fixture
(tests/golden/factored_small.npz) ran the REAL reference on the densified
instance (FactoredArrays.dense_lists: explicit R_i^T R_i, Q = 0 linear rows).
1. the oracle given the same dense lists reproduces it bit for bit (same
   machine) -- pins the orthant-row encoding and the trace;
2. the oracle's factored restatement (FactoredOp, R^T (R x)) matches it to
   rounding: the accepted step sizes of the first 200 iterations agree to
   1e-9 relative and the iterates to 1e-8.
"""

import numpy as np
import pytest

from conftest import FACTORED_SMALL
from oracle import rapdb_oracle as O
from paper_2605_29291_b200 import instances
from test_oracle_pin import TRACE_TAU, _run, _trace

CASES = {"mono": dict(nm=False, policy=O.Policy(kind="none"), budget=200),
         "nm": dict(nm=True, policy=O.Policy(kind="none"), budget=200)}


@pytest.fixture(scope="module")
def arr():
    return instances.factored_qcqp(**FACTORED_SMALL)


def test_factored_fixture_instance(arr, golden_factored):
    g = golden_factored
    np.testing.assert_array_equal(g["R_checksum"], [arr.R.data.sum(), arr.R.indices.sum()])
    np.testing.assert_array_equal(g["A_checksum"], [arr.A.data.sum(), arr.A.indices.sum(), arr.b.sum()])


def test_factored_probe(arr, golden_factored):
    g = golden_factored
    P = O.factored_problem(arr)
    x, lam = g["probe_x"], g["probe_lam"]
    np.testing.assert_allclose(P.g(x), g["probe_g"], rtol=1e-12, atol=1e-12)
    assert abs(P.f(x) - float(g["probe_f"])) <= 1e-12 * (1 + abs(float(g["probe_f"])))
    np.testing.assert_allclose(P.grad_x(x, np.zeros(0), lam), g["probe_gradx"], rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("key", list(CASES))
def test_oracle_dense_lists_bitwise(arr, golden_factored, key):
    c = CASES[key]
    res, _ = _run(O.factored_problem(arr, dense=True), "yx", c["nm"], c["policy"], c["budget"])
    tr = _trace(res)
    np.testing.assert_array_equal(tr[:, TRACE_TAU], golden_factored[f"{key}/trace"][:, TRACE_TAU])
    np.testing.assert_allclose(res.x, golden_factored[f"{key}/final_x"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("key", list(CASES))
def test_oracle_factored_restatement(arr, golden_factored, key):
    c = CASES[key]
    res, _ = _run(O.factored_problem(arr), "yx", c["nm"], c["policy"], c["budget"])
    tr = _trace(res)
    tg = golden_factored[f"{key}/trace"]
    assert len(tr) == len(tg)
    np.testing.assert_array_equal(tr[:, 5], tg[:, 5])          # backtracks per iteration
    np.testing.assert_allclose(tr[:, 1:5], tg[:, 1:5], rtol=1e-9)
    np.testing.assert_allclose(res.x, golden_factored[f"{key}/final_x"], rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(res.lam, golden_factored[f"{key}/final_lam"], rtol=1e-8, atol=1e-9)


def test_phased_transpose_walks_columns_in_row_order():
    """factored.phased_transpose (the R^T gather layout): concatenating a
    column's entries over the phases gives that column of R^T.tocsr() in
    sorted row order, and the tags decode to (row, block)."""
    from paper_2605_29291_b200.factored import RT_TAG_SHIFT, phased_transpose
    arr = instances.factored_qcqp(n=300, mq=4, rows=30, nnz_row=10, lin_rows=20, lin_nnz=5, seed=5)
    R = arr.R
    nr, n = R.shape
    rmat = np.repeat(np.arange(arr.mq + 1, dtype=np.int32), arr.rows)
    full = R.T.tocsr()
    full.sort_indices()
    for nph, tag in ((1, False), (3, True), (7, True)):
        bounds, mats = phased_transpose(R, rmat, nph, tag)
        assert bounds[0] == 0 and bounds[-1] == nr and len(mats) == nph
        cols = [([], []) for _ in range(n)]
        for S in mats:                      # Sell per phase: slot -> column via map
            assert sorted(int(j) for j in S.map if j >= 0) == list(range(n))
            for s_ in range(S.nslots):
                j = int(S.map[s_])
                pos = int(S.sp[s_ >> 5]) + 32 * np.arange(int(S.len[s_])) + (s_ & 31)
                if j >= 0:
                    cols[j][0].append(S.idx[pos])
                    cols[j][1].append(S.val[pos])
        for j in range(n):
            r = np.concatenate(cols[j][0]).astype(np.int64)
            v = np.concatenate(cols[j][1])
            if tag:
                np.testing.assert_array_equal(r >> RT_TAG_SHIFT, rmat[r & ((1 << RT_TAG_SHIFT) - 1)])
                r = r & ((1 << RT_TAG_SHIFT) - 1)
            np.testing.assert_array_equal(r, full.indices[full.indptr[j]:full.indptr[j + 1]])
            np.testing.assert_array_equal(v, full.data[full.indptr[j]:full.indptr[j + 1]])
