"""Kernel-level parity on the GPU: primitives, BSR SpMV, block Cholesky-inverse,
aggregation known-answer cases, prolongation QR branches, Chebyshev analytic
cases, PCG hand cases. Each compares against numpy / the CPU oracle."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P

    return P


def D():
    from paper_2007_01941_b200 import _device

    return _device


def test_radix_sort_stable(P):
    import torch

    rng = np.random.default_rng(1)
    for n, bits in [(1, 3), (1000, 5), (70000, 14), (300001, 23)]:
        keys = rng.integers(0, 1 << bits, n).astype(np.uint32)
        vals = np.arange(n, dtype=np.uint32)
        kd = torch.as_tensor(keys.view(np.int32), device="cuda")
        vd = torch.as_tensor(vals.view(np.int32), device="cuda")
        ko = torch.empty_like(kd)
        vo = torch.empty_like(vd)
        D().call("bamg_sort_pairs_u32", kd, vd, ko, vo, n, bits)
        order = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(vo.cpu().numpy().view(np.uint32), order)
        np.testing.assert_array_equal(ko.cpu().numpy().view(np.uint32), keys[order])


def test_scan(P):
    import torch

    rng = np.random.default_rng(2)
    for n in [1, 2047, 2048, 2049, 5_000_000]:
        a = rng.integers(0, 7, n).astype(np.int32)
        t = torch.as_tensor(a, device="cuda")
        tot = torch.empty(1, dtype=torch.int32, device="cuda")
        D().call("bamg_scan_exclusive_i32", t, t, n, tot)
        ref = np.concatenate([[0], np.cumsum(a)[:-1]])
        np.testing.assert_array_equal(t.cpu().numpy(), ref)
        assert int(tot.item()) == int(a.sum())


@pytest.mark.parametrize("bs", [9, 16])
def test_bsr_spmv_and_fused_dot(P, bs):
    rng = np.random.default_rng(bs)
    nb = 300
    m = sp.random(nb, nb, density=0.05, random_state=3, format="csr")
    m = (m + sp.eye(nb)).tocsr()
    m.sort_indices()
    blocks = rng.normal(size=(m.nnz, bs, bs))
    A = P.BlockSparseMatrix(nb, nb, bs, bs, m.indptr, m.indices, blocks)
    x = rng.normal(size=nb * bs)
    ref = sp.bsr_matrix((blocks, m.indices, m.indptr), shape=(nb * bs, nb * bs)) @ x
    y = A.matvec(x)
    assert np.max(np.abs(D().host(y) - ref)) <= 1e-12 * np.max(np.abs(ref))
    out = D().empty(1)
    y2 = D().empty(nb * bs)
    xd = D().f64(x)
    D().call("bamg_bsr_spmv", bs, A._ptr, A._col, A.blocks, xd, y2, nb, out)
    assert abs(float(out.item()) - x @ ref) <= 1e-11 * abs(x @ ref)
    # rerun: bit-identical (deterministic reductions)
    out2 = D().empty(1)
    D().call("bamg_bsr_spmv", bs, A._ptr, A._col, A.blocks, xd, y2, nb, out2)
    assert float(out.item()) == float(out2.item())


def test_symmetric_half_storage_spmv(P):
    """S products from the upper blocks + mirrored transposes equal the full-storage
    BSR product (scipy on the host copy), the fused dot is deterministic, and the
    lower blocks are exact transposes of the upper ones (the premise)."""
    from paper_2007_01941_b200 import scenes

    prob = P.BundleProblem(*scenes.random_problem(1003).arrays())
    _, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    S = P.schur_explicit(s)
    assert S._symop is not None
    ptr, col = D().host(S._ptr).astype(np.int64), D().host(S._col).astype(np.int64)
    blocks = D().host(S.blocks)
    rows = np.repeat(np.arange(S.n_block_rows), np.diff(ptr))
    key = {(int(i), int(j)): q for q, (i, j) in enumerate(zip(rows, col))}
    for q, (i, j) in enumerate(zip(rows, col)):
        assert np.array_equal(blocks[key[(int(j), int(i))]], blocks[q].T)
    rng = np.random.default_rng(5)
    x = rng.normal(size=S.shape[0])
    ref = sp.bsr_matrix((blocks, col, ptr), shape=S.shape) @ x
    y = D().host(S.matvec(x))
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
    xd = D().f64(x)
    outs = []
    for _ in range(2):
        out = D().empty(1)
        y2 = D().empty(S.shape[0])
        D().call("bamg_symop_spmv", S._symop.handle, S.blocks, xd, y2, out)
        outs.append((float(out.item()), D().host(y2)))
    assert abs(outs[0][0] - x @ ref) <= 1e-11 * abs(x @ ref)
    assert outs[0][0] == outs[1][0] and np.array_equal(outs[0][1], outs[1][1])
    # with and without the fused dot, and the residual epilogue: the same sums,
    # bit for bit, on every rerun
    for _ in range(3):
        y1 = D().empty(S.shape[0])
        D().call("bamg_symop_spmv", S._symop.handle, S.blocks, xd, y1, None)
        assert np.array_equal(D().host(y1), outs[0][1])
    b = rng.normal(size=S.shape[0])
    bd = D().f64(b)
    r1 = D().empty(S.shape[0])
    D().call("bamg_symop_residual", S._symop.handle, S.blocks, xd, bd, r1)
    assert np.array_equal(D().host(r1), b - outs[0][1])


def test_symmetric_half_storage_coarse_operator(P):
    """The same view for a 16x16 Galerkin operator (pattern-derived mirror map):
    product, residual and Chebyshev epilogues against the full-storage kernels."""
    from paper_2007_01941_b200 import scenes

    prob = P.BundleProblem(*scenes.street(n_cameras=60, n_points=4000, seed=3).arrays())
    _, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    s.mode = P.choose_mode(s)
    h = P.build_hierarchy(s, P.gauge_nullspace(prob), P.visibility_strength(prob), max_coarse_dim=40)
    assert h.n_levels >= 3
    A = h.levels[1].explicit
    assert A._symop is not None and A.row_block_size == 16
    blocks = D().host(A.blocks)
    ptr, col = D().host(A._ptr).astype(np.int64), D().host(A._col).astype(np.int64)
    full = sp.bsr_matrix((blocks, col, ptr), shape=A.shape)
    assert abs(full - full.T).max() == 0.0  # exactly symmetric: the premise
    rng = np.random.default_rng(9)
    x, b = rng.normal(size=A.shape[0]), rng.normal(size=A.shape[0])
    ref = full @ x
    assert np.max(np.abs(D().host(A.matvec(x)) - ref)) <= 1e-12 * np.max(np.abs(ref))
    xd, bd = D().f64(x), D().f64(b)
    r_sym, r_full = D().empty(A.shape[0]), D().empty(A.shape[0])
    D().call("bamg_symop_residual", A._symop.handle, A.blocks, xd, bd, r_sym)
    D().call("bamg_bsr_residual", 16, A._ptr, A._col, A.blocks, xd, bd, r_full, A.n_block_rows)
    assert np.max(np.abs(D().host(r_sym) - D().host(r_full))) <= 1e-12 * np.max(np.abs(ref))
    Dinv = h.levels[1].smoother.jacobi.inverse_blocks()
    outs = []
    for fn in ("sym", "full"):
        d = D().f64(np.ones(A.shape[0]))
        o = D().empty(A.shape[0])
        if fn == "sym":
            D().call("bamg_symop_cheb_step", A._symop.handle, A.blocks, xd, bd, Dinv, d, o, 0.3, 0.7, 0)
        else:
            D().call("bamg_cheb_step", 16, A._ptr, A._col, A.blocks, xd, bd, Dinv, d, o, A.n_block_rows, 0.3, 0.7, 0)
        outs.append(D().host(o))
    assert np.max(np.abs(outs[0] - outs[1])) <= 1e-10 * np.max(np.abs(outs[1]))


@pytest.mark.parametrize("bs", [1, 3, 9, 16])
def test_block_cholesky_inverse(P, bs):
    rng = np.random.default_rng(10 + bs)
    raw = rng.normal(size=(50, bs, bs))
    blocks = np.einsum("nij,nkj->nik", raw, raw) + bs * np.eye(bs)
    M = P.BlockDiagMatrix(blocks).factor()
    np.testing.assert_allclose(D().host(M.inverse_blocks()), np.linalg.inv(blocks), rtol=1e-10, atol=1e-12)
    x = rng.normal(size=50 * bs)
    want = np.einsum("nij,nj->ni", np.linalg.inv(blocks), x.reshape(50, bs)).ravel()
    assert relerr(D().host(M.solve(x)), want) <= 1e-12
    bad = blocks.copy()
    bad[7] = -np.eye(bs)
    bad[20] = -np.eye(bs)
    with pytest.raises(P.IndefiniteBlockError) as e:
        P.BlockDiagMatrix(bad).factor()
    assert e.value.block_index == 7


@pytest.mark.parametrize("name", ["chain", "star", "isolated", "random_ties", "clique30"])
def test_aggregate_known_answers(P, name):
    g = golden("aggregate_cases")
    n = len(g[f"{name}_indptr"]) - 1
    G = P.StrengthMatrix(g[f"{name}_indptr"], g[f"{name}_indices"], g[f"{name}_data"], n)
    agg = P.aggregate(G)
    np.testing.assert_array_equal(D().host(agg.assignment), g[f"{name}_assign"])


def test_prolongation_branches(P):
    from paper_2007_01941_b200.multigrid import Aggregation

    rng = np.random.default_rng(72)
    # full-rank (economic, sign-fixed) branch: equals numpy QR with positive diag R
    assign = np.array([0, 0, 1, 1, 1, 2, 2])
    K = rng.normal(size=(63, 16))
    Pm, kc, padded = P.build_prolongation(Aggregation(assign, 3), P.DenseTall(K), 9)
    pd, kcd = D().host(Pm.to_dense()), D().host(kc.data)
    np.testing.assert_allclose(pd.T @ pd, np.eye(48), atol=1e-12)
    np.testing.assert_allclose(pd @ kcd, K, atol=1e-12)
    for a in range(3):
        mem = np.flatnonzero(assign == a)
        rows = (mem[:, None] * 9 + np.arange(9)).ravel()
        qo, ro = np.linalg.qr(K[rows])
        s = np.where(np.diag(ro) < 0, -1.0, 1.0)
        np.testing.assert_allclose(pd[np.ix_(rows, np.arange(16 * a, 16 * a + 16))], qo * s, atol=1e-12)
        np.testing.assert_allclose(kcd[16 * a:16 * a + 16], ro * s[:, None], atol=1e-12)
    assert len(padded) == 0
    # singletons pad (multigrid.py:228-230)
    K2 = rng.normal(size=(18, 16))
    Pm, kc, padded = P.build_prolongation(Aggregation(np.array([0, 1]), 2), P.DenseTall(K2), 9)
    pd = D().host(Pm.to_dense())
    np.testing.assert_allclose(pd @ D().host(kc.data), K2, atol=1e-12)
    assert len(padded) == 14
    kept = sorted(set(range(32)) - set(D().host(padded).tolist()))
    np.testing.assert_allclose((pd.T @ pd)[np.ix_(kept, kept)], np.eye(18), atol=1e-12)
    # rank-deficient completion
    K3 = rng.normal(size=(27, 16))
    K3[:, 5] = K3[:, 3]
    Pm, kc, _ = P.build_prolongation(Aggregation(np.zeros(3, dtype=np.int64), 1), P.DenseTall(K3), 9)
    pd = D().host(Pm.to_dense())
    np.testing.assert_allclose(pd.T @ pd, np.eye(16), atol=1e-12)
    np.testing.assert_allclose(pd @ D().host(kc.data), K3, atol=1e-12)
    assert int(D().host(Pm.qr_info)[0, 0]) == 1 and int(D().host(Pm.qr_info)[0, 1]) == 15


def test_pcg_hand_cases(P):
    n = 12
    b = np.arange(1.0, n + 1)
    ident = P.BlockDiagMatrix(np.ones((n, 1, 1)))
    x, rep = P.pcg(ident.matvec, ident.matvec, b, tau=1e-30)
    np.testing.assert_allclose(D().host(x), b, rtol=1e-14)
    assert rep.iterations == 1
    rng = np.random.default_rng(4)
    M = rng.normal(size=(n, n))
    A = M @ M.T + n * np.eye(n)
    Ad = P.BlockDiagMatrix(A[None])
    x, rep = P.pcg(Ad.matvec, ident.matvec, b, tau=1e-30, max_iterations=200)
    assert relerr(D().host(x), np.linalg.solve(A, b)) <= 1e-8
    z, rep = P.pcg(Ad.matvec, ident.matvec, np.zeros(n), tau=0.1)
    assert rep.iterations == 0 and rep.stop_reason == "residual_tol"
    with pytest.raises(P.CgDivergence):
        P.pcg(P.BlockDiagMatrix(-np.ones((n, 1, 1))).matvec, ident.matvec, b, tau=0.1)


def test_chebyshev_matches_oracle(P):
    from oracle import bamg_oracle as O

    rng = np.random.default_rng(5)
    nb, bs = 40, 9
    m = sp.random(nb, nb, density=0.1, random_state=6, format="csr")
    m = (m + m.T + sp.eye(nb)).tocsr()
    m.sort_indices()
    raw = rng.normal(size=(m.nnz, bs, bs)) * 0.05
    A = sp.bsr_matrix((raw, m.indices, m.indptr), shape=(nb * bs, nb * bs)).toarray()
    A = A + A.T + 4 * nb * np.eye(nb * bs) * 0.1
    Ab = sp.bsr_matrix(A, blocksize=(bs, bs))
    Ab.sort_indices()
    Bd = P.BlockSparseMatrix(nb, nb, bs, bs, Ab.indptr, Ab.indices, Ab.data)
    Dblk = np.stack([A[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] for i in range(nb)])
    jac = P.BlockDiagMatrix(Dblk)
    sm = P.ChebyshevSmoother(jac, 2.0, 0.6, 2.2)
    ch = O.Cheb(np.linalg.inv(Dblk), 2.0, 0.6, 2.2)
    b = rng.normal(size=nb * bs)
    x0 = rng.normal(size=nb * bs)
    mv = lambda v: A @ v  # noqa: E731
    got = D().host(sm.apply(Bd.matvec, None, b))
    assert relerr(got, ch.apply(mv, None, b)) <= 1e-12
    got = D().host(sm.apply(Bd.matvec, x0, b))
    assert relerr(got, ch.apply(mv, x0, b)) <= 1e-12


@pytest.mark.parametrize("seed,n,deg,max_size,levels", [
    (1, 300, 6, 20, 4), (2, 2000, 12, 20, 8), (3, 700, 30, 3, 3), (4, 500, 9, 2, 5), (5, 4000, 40, 20, 16),
    (6, 1500, 3, 20, 2)])
def test_aggregate_speculative_scan_matches_oracle(P, seed, n, deg, max_size, levels):
    """The aggregation scan (k_aggregate_seq by default; the speculative batch scan
    k_aggregate_spec under BAMG_AGG_SEQ=0) against the oracle's sequential
    greedy scan (multigrid.py:127-176) on random graphs built to collide: local
    neighbourhoods (consecutive nodes are neighbours, as coarse aggregates are),
    few distinct strengths (ties everywhere), rows longer than the 8-entry head,
    tiny aggregate caps (full aggregates)."""
    import scipy.sparse as sp

    from oracle import bamg_oracle as O

    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(n), deg)
    c = (r + rng.integers(-3 * deg, 3 * deg + 1, r.size)) % n
    keep = r != c
    v = rng.integers(1, levels + 1, r.size) / levels
    g = sp.csr_matrix((v[keep], (r[keep], c[keep])), shape=(n, n))
    g = g.maximum(g.T).tocsr()
    g.sort_indices()
    G = P.StrengthMatrix(g.indptr, g.indices, g.data, n)
    agg = P.aggregate(G, max_size=max_size)
    want, na = O.aggregate(g, max_size)
    assert agg.n_aggregates == na
    np.testing.assert_array_equal(D().host(agg.assignment), want)


def test_aggregate_alternative_kernels_still_match():
    """The scan kernels that are no longer the default (speculative rounds, BAMG_AGG_SEQ=0;
    cooperative head scan, BAMG_AGG_SPEC=0 as well) stay bit-exact: the aggregation tests
    of this file re-run in a subprocess with the environment switches set (they are read
    once per process)."""
    import os
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    here = os.path.abspath(__file__)
    for env in ({"BAMG_AGG_SEQ": "0"}, {"BAMG_AGG_SEQ": "0", "BAMG_AGG_SPEC": "0"}):
        p = subprocess.run([sys.executable, "-m", "pytest", here, "-q", "-x", "-k",
                            "aggregate_known_answers or aggregate_speculative_scan"],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, (env, p.stdout[-2000:], p.stderr[-2000:])
