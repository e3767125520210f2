"""Generic block-sparse API on the device vs the reference's third-party kernels
(SURVEY 8(a) S7 from_triplets, M3 rmatvec / rectangular matvec, blockmat.py:321-360
scale_block_columns / multiply / triple_product; VERDICT r1 "what's missing" 5).

The kernels follow numpy's / scipy's summation orders with separately rounded
products and sums, so everything here is compared BIT-EXACT (np.array_equal)
against scipy.sparse / numpy on the same inputs, except scale_block_columns
(numpy einsum's internal order is not specified: 1e-15).
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P

    return P


def H(t):
    from paper_2007_01941_b200 import _device

    return _device.host(t)


def _ref_from_triplets(nbr, nbc, r, c, blocks):
    """blockmat.py:195-230 restated (np.lexsort + np.add.reduceat)."""
    order = np.lexsort((c, r))
    r, c, blocks = r[order], c[order], blocks[order]
    new = np.empty(len(r), bool)
    new[0] = True
    new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    st = np.flatnonzero(new)
    summed = np.add.reduceat(blocks, st, axis=0)
    ptr = np.zeros(nbr + 1, np.int64)
    np.cumsum(np.bincount(r[st], minlength=nbr), out=ptr[1:])
    return ptr, c[st], summed


def _random_bsr(rng, nbr, nbc, rbs, cbs, density):
    mask = rng.random((nbr, nbc)) < density
    r, c = np.nonzero(mask)
    blocks = rng.standard_normal((len(r), rbs, cbs))
    ptr = np.zeros(nbr + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=nbr), out=ptr[1:])
    return ptr, c.astype(np.int64), blocks


def _dev(P, nbr, nbc, rbs, cbs, ptr, col, blocks):
    return P.BlockSparseMatrix(nbr, nbc, rbs, cbs, ptr, col, blocks)


def _scipy(nbr, nbc, rbs, cbs, ptr, col, blocks):
    return sp.bsr_matrix((blocks, col, ptr), shape=(nbr * rbs, nbc * cbs), blocksize=(rbs, cbs))


@pytest.mark.parametrize("rbs,cbs", [(9, 3), (3, 9), (9, 9), (16, 16), (9, 16), (1, 1)])
def test_from_triplets_bit_exact(P, rbs, cbs):
    rng = np.random.default_rng(rbs * 100 + cbs)
    nbr, nbc, n = 37, 53, 900
    r = rng.integers(0, nbr, n)
    c = rng.integers(0, nbc, n)
    # duplicate runs of every length class of numpy's pairwise sum (<8, 8..128, >128)
    r = np.concatenate([r, np.full(5, 3), np.full(20, 4), np.full(300, 5)])
    c = np.concatenate([c, np.full(5, 7), np.full(20, 8), np.full(300, 9)])
    n = len(r)
    blocks = rng.standard_normal((n, rbs, cbs)) * 10.0 ** rng.integers(-8, 8, (n, 1, 1))
    M = P.BlockSparseMatrix.from_triplets(nbr, nbc, r, c, blocks)
    ptr, col, summed = _ref_from_triplets(nbr, nbc, r, c, blocks)
    np.testing.assert_array_equal(H(M.indptr), ptr)
    np.testing.assert_array_equal(H(M.indices), col)
    assert np.array_equal(H(M.blocks), summed)


def test_from_triplets_validation(P):
    b = np.zeros((2, 3, 3))
    with pytest.raises(ValueError, match="out of range"):
        P.BlockSparseMatrix.from_triplets(4, 4, [0, 1], [0, 4], b)
    with pytest.raises(ValueError, match="out of range"):
        P.BlockSparseMatrix.from_triplets(4, 4, [-1, 1], [0, 1], b)
    with pytest.raises(ValueError, match="disagree"):
        P.BlockSparseMatrix.from_triplets(4, 4, [0, 1, 2], [0, 1], b)
    M = P.BlockSparseMatrix.from_triplets(3, 5, [], [], np.zeros((0, 2, 2)))
    assert M.n_block_entries == 0 and np.array_equal(H(M.indptr), np.zeros(4))


def test_constructor_validation(P):
    blk = np.zeros((3, 2, 2))
    with pytest.raises(ValueError, match="nondecreasing"):
        P.BlockSparseMatrix(3, 3, 2, 2, [0, 2, 1, 3], [0, 1, 2], blk)
    with pytest.raises(ValueError, match="out of range"):
        P.BlockSparseMatrix(3, 3, 2, 2, [0, 1, 2, 3], [0, 1, 3], blk)
    with pytest.raises(ValueError, match="indptr\\[-1\\]"):
        P.BlockSparseMatrix(3, 3, 2, 2, [0, 1, 2, 2], [0, 1, 2], blk)
    with pytest.raises(ValueError, match="indptr has length"):
        P.BlockSparseMatrix(3, 3, 2, 2, [0, 1, 3], [0, 1, 2], blk)


@pytest.mark.parametrize("rbs,cbs", [(9, 3), (3, 9), (9, 16), (16, 9), (2, 5)])
def test_rect_matvec_and_rmatvec_bit_exact(P, rbs, cbs):
    rng = np.random.default_rng(7 + rbs + cbs)
    nbr, nbc = 41, 29
    ptr, col, blocks = _random_bsr(rng, nbr, nbc, rbs, cbs, 0.2)
    M = _dev(P, nbr, nbc, rbs, cbs, ptr, col, blocks)
    S = _scipy(nbr, nbc, rbs, cbs, ptr, col, blocks)
    x = rng.standard_normal(nbc * cbs)
    assert np.array_equal(H(M.matvec(x)), S @ x)
    u = rng.standard_normal(nbr * rbs)
    assert np.array_equal(H(M.rmatvec(u)), S.T @ u)
    T = M.transpose()
    St = sp.bsr_matrix(S.T)
    St.sort_indices()
    np.testing.assert_array_equal(H(T.indptr), St.indptr)
    np.testing.assert_array_equal(H(T.indices), St.indices)
    assert np.array_equal(H(T.blocks), St.data)
    with pytest.raises(ValueError):
        M.matvec(np.zeros(nbc * cbs + 1))
    with pytest.raises(ValueError):
        M.rmatvec(np.zeros(nbr * rbs + 1))


def test_scale_block_columns(P):
    rng = np.random.default_rng(3)
    nbr, nbc, rbs, cbs, k = 20, 30, 9, 3, 3
    ptr, col, blocks = _random_bsr(rng, nbr, nbc, rbs, cbs, 0.3)
    M = _dev(P, nbr, nbc, rbs, cbs, ptr, col, blocks)
    cb = rng.standard_normal((nbc, cbs, k))
    got = H(M.scale_block_columns(cb).blocks)
    want = np.einsum("nij,njk->nik", blocks, cb[col])
    np.testing.assert_allclose(got, want, rtol=1e-15, atol=1e-15 * np.abs(want).max())
    with pytest.raises(ValueError):
        M.scale_block_columns(cb[:-1])


def _scipy_multiply(a, b, rbs, cbs):
    prod = (a.tocsr() @ b.tocsr()).tobsr(blocksize=(rbs, cbs))
    prod.sort_indices()
    return prod


@pytest.mark.parametrize("shape", [(9, 9, 9), (16, 9, 16), (9, 3, 9), (3, 2, 4)])
def test_multiply_bit_exact(P, shape):
    rbs, kbs, cbs = shape
    rng = np.random.default_rng(sum(shape))
    na, nk, nb = 23, 31, 19
    pa, ca, ba = _random_bsr(rng, na, nk, rbs, kbs, 0.15)
    pb, cb_, bb = _random_bsr(rng, nk, nb, kbs, cbs, 0.15)
    A, B = _dev(P, na, nk, rbs, kbs, pa, ca, ba), _dev(P, nk, nb, kbs, cbs, pb, cb_, bb)
    C = P.multiply(A, B)
    want = _scipy_multiply(_scipy(na, nk, rbs, kbs, pa, ca, ba), _scipy(nk, nb, kbs, cbs, pb, cb_, bb), rbs, cbs)
    np.testing.assert_array_equal(H(C.indptr), want.indptr)
    np.testing.assert_array_equal(H(C.indices), want.indices)
    assert np.array_equal(H(C.blocks), want.data)


def test_multiply_zero_drop(P):
    """Exact cancellation: a product block whose every scalar sums to 0 is dropped,
    partially cancelled blocks keep +0 entries (csr_matmat + tobsr)."""
    e = np.eye(2)
    # A = [[I, I]], B = [[X], [-X]] -> A B = 0 exactly; second column block of B keeps one row
    X = np.array([[1.0, 2.0], [3.0, 4.0]])
    Y = np.array([[1.0, 0.0], [0.0, 5.0]])
    A = P.BlockSparseMatrix(1, 2, 2, 2, [0, 2], [0, 1], np.stack([e, e]))
    B = P.BlockSparseMatrix(2, 2, 2, 2, [0, 2, 4], [0, 1, 0, 1], np.stack([X, Y, -X, -Y + np.diag([0, 1.0])]))
    C = P.multiply(A, B)
    sa = _scipy(1, 2, 2, 2, np.array([0, 2]), np.array([0, 1]), np.stack([e, e]))
    sb = _scipy(2, 2, 2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), H(B.blocks))
    want = _scipy_multiply(sa, sb, 2, 2)
    np.testing.assert_array_equal(H(C.indices), want.indices)
    assert np.array_equal(H(C.blocks), want.data)
    assert C.n_block_entries == 1 and np.signbit(H(C.blocks)).sum() == 0


def test_triple_product_galerkin_shape(P):
    rng = np.random.default_rng(11)
    n, na = 40, 13
    agg = rng.integers(0, na, n)
    agg[:na] = np.arange(na)
    Pb = rng.standard_normal((n, 9, 16))
    Pm = P.BlockSparseMatrix(n, na, 9, 16, np.arange(n + 1), agg, Pb)
    pa, ca, ba = _random_bsr(rng, n, n, 9, 9, 0.1)
    A = _dev(P, n, n, 9, 9, pa, ca, ba)
    C = P.triple_product(Pm.transpose(), A, Pm)
    sP = _scipy(n, na, 9, 16, np.arange(n + 1), agg, Pb)
    sPt = sp.bsr_matrix(sP.T)
    sPt.sort_indices()
    want = _scipy_multiply(_scipy_multiply(sPt, _scipy(n, n, 9, 9, pa, ca, ba), 16, 9), sP, 16, 16)
    np.testing.assert_array_equal(H(C.indptr), want.indptr)
    np.testing.assert_array_equal(H(C.indices), want.indices)
    assert np.array_equal(H(C.blocks), want.data)


def test_write_matrix_market_matches_reference_format(P, tmp_path):
    rng = np.random.default_rng(5)
    ptr, col, blocks = _random_bsr(rng, 6, 5, 2, 3, 0.4)
    blocks[0, 0, 0] = 0.0  # stored zero: written like scipy's bsr.tocoo()
    M = _dev(P, 6, 5, 2, 3, ptr, col, blocks)
    path = tmp_path / "m.mtx"
    P.write_matrix_market(M, str(path))
    coo = _scipy(6, 5, 2, 3, ptr, col, blocks).tocoo()
    lines = ["%%MatrixMarket matrix coordinate real general", f"12 15 {coo.nnz}"]
    lines += [f"{i + 1} {j + 1} {v:.17g}" for i, j, v in zip(coo.row, coo.col, coo.data)]
    assert path.read_text().splitlines() == lines
