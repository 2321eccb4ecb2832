"""The sliced-ELLPACK layout of the factored path's sparse operands
(paper_2605_29291_b200/factored.py SellMatrix, include/rapdb_b200.h rapdb_sell):
walking the slots the way the device does (lane = slot, entries in stored
order, no FMA) reproduces scipy's csr_matvec bit for bit -- the summation
order the factored restatement (oracle FactoredOp / FactoredProblem) uses."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2605_29291_b200.factored import RT_TAG_SHIFT, SellMatrix, phased_transpose


def walk(S, x, nout, s0=None):
    """Device order: slot s folds its entries t = 0..len-1 from s0[out]."""
    out = np.zeros(nout) if s0 is None else s0.copy()
    seen = np.zeros(nout, dtype=int)
    for s in range(S.nslots):
        j = s if S.map is None else int(S.map[s])
        if j < 0:
            assert S.len[s] == 0
            continue
        if j >= nout:
            assert S.len[s] == 0
            continue
        acc = out[j] if s0 is not None else 0.0
        for t in range(int(S.len[s])):
            pos = int(S.sp[s >> 5]) + 32 * t + (s & 31)
            acc = acc + S.val[pos] * x(int(S.idx[pos]))
        out[j] = acc
        seen[j] += 1
    return out, seen


@pytest.mark.parametrize("shape,density", [((257, 90), 0.08), ((64, 40), 0.3), ((33, 500), 0.01), ((5, 7), 0.0)])
def test_by_row_matches_csr_matvec(shape, density):
    M = sp.random(*shape, density=density, format="csr", random_state=3)
    x = np.random.default_rng(1).normal(size=shape[1])
    S = SellMatrix.by_row(M)
    assert S.nslots % 32 == 0 and S.sp[-1] == S.entries and S.entries % 32 == 0
    got, _ = walk(S, lambda c: x[c], shape[0])
    np.testing.assert_array_equal(got, M @ x)


def test_sorted_length_covers_every_row_once_and_packs_tightly():
    M = sp.random(1000, 300, density=0.03, format="csr", random_state=5)
    x = np.random.default_rng(2).normal(size=300)
    S = SellMatrix.by_sorted_length(M)
    got, seen = walk(S, lambda c: x[c], 1000)
    np.testing.assert_array_equal(got, M @ x)
    assert np.all(seen == 1)
    assert S.entries <= 1.1 * M.nnz + 32 * 32       # sorted slots: almost no padding
    lens = S.len.reshape(-1, 32)
    assert np.all(lens[:-1].min(axis=1) >= lens[1:].max(axis=1))


def test_block_chunks_keep_blocks_apart():
    M = sp.random(700, 120, density=0.05, format="csr", random_state=7)
    rblk = np.array([0, 100, 355, 355, 700])
    S = SellMatrix.by_block_chunks(M, rblk)
    chunks = [-(-(int(rblk[i + 1]) - int(rblk[i])) // 128) for i in range(4)]
    assert S.nslots == 128 * sum(chunks)
    x = np.random.default_rng(3).normal(size=120)
    ref = M @ x
    slot = 0
    for i, nc in enumerate(chunks):
        rows = int(rblk[i + 1]) - int(rblk[i])
        for k in range(nc * 128):
            s = slot + k
            acc = 0.0
            for t in range(int(S.len[s])):
                pos = int(S.sp[s >> 5]) + 32 * t + (s & 31)
                acc = acc + S.val[pos] * x[S.idx[pos]]
            if k < rows:
                assert acc == ref[int(rblk[i]) + k]
            else:
                assert S.len[s] == 0
        slot += nc * 128


@pytest.mark.parametrize("nph,tag", [(1, True), (3, True), (2, False)])
def test_phased_transpose_walks_columns_in_row_order(nph, tag):
    R = sp.random(900, 150, density=0.04, format="csr", random_state=11)
    rmat = np.repeat(np.arange(3, dtype=np.int32), 300)
    w = np.random.default_rng(4).normal(size=900)
    wq = np.array([1.0, 0.0, 2.5])
    bounds, mats = phased_transpose(R, rmat, nph, tag)
    assert bounds[0] == 0 and bounds[-1] == 900 and len(mats) == nph

    def entry(idx):
        if tag:
            return wq[idx >> RT_TAG_SHIFT] * w[idx & ((1 << RT_TAG_SHIFT) - 1)]
        return wq[rmat[idx]] * w[idx]

    out = None
    for S in mats:
        out, seen = walk(S, entry, 150, s0=out if out is not None else np.zeros(150))
        assert np.all(seen == 1)
    Rt = R.T.tocsr()
    Rt.sort_indices()
    np.testing.assert_array_equal(out, Rt @ (wq[rmat] * w))


# ---- property tests (hypothesis): any CSR, any block partition, any phase count
from hypothesis import given, settings, strategies as st  # noqa: E402


@st.composite
def csr_cases(draw):
    rows = draw(st.integers(0, 70))
    cols = draw(st.integers(1, 50))
    seed = draw(st.integers(0, 2 ** 16))
    density = draw(st.sampled_from([0.0, 0.02, 0.1, 0.4, 1.0]))
    rng = np.random.default_rng(seed)
    dense = np.where(rng.uniform(size=(rows, cols)) < density, rng.normal(size=(rows, cols)), 0.0)
    M = sp.csr_matrix(dense)
    cuts = sorted(draw(st.lists(st.integers(0, rows), max_size=4)))
    rblk = np.array([0] + cuts + [rows], dtype=np.int64)
    return M, rblk, rng.normal(size=cols), rng.normal(size=rows), draw(st.integers(1, 5))


@settings(max_examples=60, deadline=None)
@given(csr_cases())
def test_sell_forms_agree_with_scipy(case):
    M, rblk, x, w, nph = case
    rows, cols = M.shape
    ref = M @ x
    for S in (SellMatrix.by_row(M), SellMatrix.by_sorted_length(M)):
        got, _ = walk(S, lambda c: x[c], rows)
        np.testing.assert_array_equal(got, ref)
        assert S.entries == int(S.sp[-1]) and np.all(np.diff(S.sp) % 32 == 0)
    S = SellMatrix.by_block_chunks(M, rblk)
    assert S.nslots == 128 * sum(-(-(int(rblk[i + 1]) - int(rblk[i])) // 128) for i in range(len(rblk) - 1))
    # the transposed gather in row phases, weights per block
    nb = len(rblk) - 1
    rmat = np.repeat(np.arange(nb, dtype=np.int32), np.diff(rblk))
    wq = np.linspace(0.0, 1.5, nb) if nb else np.zeros(0)
    _, mats = phased_transpose(M, rmat, nph, True)
    out = np.zeros(cols)
    for T in mats:
        out, seen = walk(T, lambda idx: wq[idx >> RT_TAG_SHIFT] * w[idx & ((1 << RT_TAG_SHIFT) - 1)], cols, s0=out)
        assert np.all(seen == 1)
    Mt = M.T.tocsr()
    Mt.sort_indices()
    np.testing.assert_array_equal(out, Mt @ (wq[rmat] * w) if rows else np.zeros(cols))
