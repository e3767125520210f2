"""Visibility block-Jacobi (precond.py:59-144) on the GPU: clusters bit-exact with
the reference, apply / PCG / LM against the reference's golden runs, and the
reference's own test cases (tests/test_precond.py:148-215) restated."""

import numpy as np
import pytest

from conftest import VJ_CASES, golden, relerr, vj_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P

    return P


@pytest.fixture(scope="module")
def g():
    return golden("vj_cases")


def H(t):
    from paper_2007_01941_b200 import _device

    return _device.host(t)


def system(P, prob, radius=1e4):
    _, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, radius))
    s.mode = P.choose_mode(s)
    return s


@pytest.mark.parametrize("tag", VJ_CASES)
def test_vj_matches_reference(P, g, tag):
    prob = P.BundleProblem(*vj_inputs(tag, g))
    s = system(P, prob)
    G = P.visibility_strength(prob)
    for cap in (100, 6):
        cl = P.visibility_cluster(G, cap)
        np.testing.assert_array_equal(H(cl.assignment), g[f"{tag}_cap{cap}_assign"])
        assert cl.n_aggregates == int(g[f"{tag}_cap{cap}_n"])
        vj = P.vj_setup(s, cl)
        for v, want in zip(g[f"{tag}_vin"], g[f"{tag}_cap{cap}_vout"]):
            assert relerr(H(vj.apply(v)), want) <= 1e-10
        x, rep = P.pcg(s.matvec, vj.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
        want_its = int(g[f"{tag}_cap{cap}_pcg_its"])
        assert abs(rep.iterations - want_its) <= 1
        if rep.iterations == want_its:
            assert relerr(H(x), g[f"{tag}_cap{cap}_pcg_x"]) <= 1e-7


@pytest.mark.parametrize("tag", ["ring", "r1003"])
def test_vj_lm_matches_reference(P, g, tag):
    prob = P.BundleProblem(*vj_inputs(tag, g))
    cfg = P.SolveConfig(preconditioner="visibility", tau=1e-30, max_iterations=10, function_tolerance=0.0,
                        gradient_tolerance=0.0, parameter_tolerance=0.0, initial_radius=1e4,
                        cg_max_iterations=20000, cg_residual_tolerance=1e-6)
    sol, rep = P.lm_solve(prob, cfg)
    cg = np.array([r.cg_iterations for r in rep.records])
    acc = np.array([r.accepted for r in rep.records])
    want = g[f"{tag}_lm_cg"]
    assert len(cg) == len(want)
    # step 1 solves the identical system: +-1
    assert abs(cg[1] - want[1]) <= 1
    # VJ needs hundreds of CG iterations per step, and after step 1 every valid
    # implementation's trajectory differs at the CG stop tolerance: the reference's
    # own counts move by up to 9% when its CG solutions are perturbed at 1e-7
    # (make_golden_vj.py envelope). Compare inside that envelope, widened by 3%,
    # on the steps whose state is numerically determined (objective still > 1e-9
    # relative above its final value, as in test_gpu_parity.test_lm_records).
    obj = g[f"{tag}_lm_obj"]
    determined = np.abs(obj - obj[-1]) > 1e-9 * abs(obj[-1])
    determined = np.concatenate([[True], determined[:-1]])
    slack = np.maximum(1, np.ceil(0.03 * g[f"{tag}_lm_cg_max"]))
    lo, hi = g[f"{tag}_lm_cg_min"] - slack, g[f"{tag}_lm_cg_max"] + slack
    ok = (cg >= lo) & (cg <= hi)
    assert np.all(ok[determined]), (cg, want, lo, hi)
    np.testing.assert_array_equal(acc[determined], g[f"{tag}_lm_accepted"][determined])
    assert abs(rep.records[-1].objective - obj[-1]) <= 1e-8 * abs(obj[-1])


# -- the reference's own cases (tests/test_precond.py), restated -----------------


def _sys(P, seed, nc, npt, radius=100.0, **kw):
    from paper_2007_01941_b200 import scenes

    prob = P.BundleProblem(*scenes.random_problem(seed, n_cameras=nc, n_points=npt, **kw).arrays())
    return prob, system(P, prob, radius)


def test_vj_singleton_clusters_match_pbj(P):
    _, s = _sys(P, 54, 5, 15)
    vj = P.vj_setup(s, P.Aggregation(np.arange(5), 5))
    pbj = P.pbj_setup(s)
    r = np.random.default_rng(1).normal(size=45)
    np.testing.assert_allclose(H(vj.apply(r)), H(pbj.apply(r)), atol=1e-10)


def test_vj_global_cluster_is_dense_inverse(P):
    _, s = _sys(P, 55, 5, 20)
    vj = P.vj_setup(s, P.Aggregation(np.zeros(5, dtype=np.int64), 1))
    dense = H(s.ensure_explicit().to_dense())
    r = np.random.default_rng(2).normal(size=45)
    assert relerr(H(vj.apply(r)), np.linalg.solve(dense, r)) <= 1e-8


def test_vj_assembled_and_accumulated_routes_agree(P):
    prob, s = _sys(P, 56, 6, 18)
    cl = P.visibility_cluster(P.visibility_strength(prob))
    s.S_explicit = None
    implicit_route = P.vj_setup(s, cl)
    s.ensure_explicit()
    explicit_route = P.vj_setup(s, cl)
    r = np.random.default_rng(3).normal(size=54)
    np.testing.assert_allclose(H(implicit_route.apply(r)), H(explicit_route.apply(r)), atol=1e-10)


def test_vj_decoupled_components_make_cg_exact(P):
    _, s = _sys(P, 57, 6, 18, decoupled=True)
    vj = P.vj_setup(s, P.Aggregation(np.arange(6) % 2, 2))
    _, rep = P.pcg(s.matvec, vj.apply, s.rhs_cam, tau=1e-12, residual_tolerance=1e-10)
    assert rep.iterations <= 2


def test_vj_rejects_wrong_partition_size(P):
    _, s = _sys(P, 58, 4, 12)
    with pytest.raises(ValueError):
        P.vj_setup(s, P.Aggregation(np.zeros(3, dtype=np.int64), 1))


def test_vj_indefinite_cluster_raises(P):
    from paper_2007_01941_b200.blockmat import IndefiniteBlockError

    _, s = _sys(P, 58, 4, 12)
    S = s.ensure_explicit()
    S.blocks[S._ptr[2].item():S._ptr[3].item()] *= -1.0  # camera 2's row: not PD any more
    S._symop = None
    with pytest.raises(IndefiniteBlockError) as e:
        P.vj_setup(s, P.Aggregation(np.array([0, 0, 1, 1]), 2))
    assert e.value.block_index == 1


def test_vj_spd_probes(P):
    prob, s = _sys(P, 59, 8, 24)
    vj = P.vj_setup(s, P.visibility_cluster(P.visibility_strength(prob)))
    rng = np.random.default_rng(4)
    for _ in range(10):
        x, y = rng.normal(size=72), rng.normal(size=72)
        mx, my = H(vj.apply(x)), H(vj.apply(y))
        scale = np.linalg.norm(mx) * np.linalg.norm(y) + 1e-30
        assert abs(x @ my - y @ mx) <= 1e-10 * scale
        assert x @ mx > 0


def test_vj_native_pcg_matches_stepwise(P, g):
    """The native PCG loop with the VJ handle == the Python loop over the same apply."""
    prob = P.BundleProblem(*vj_inputs("r1004", g))
    s = system(P, prob)
    vj = P.vj_setup(s, P.visibility_cluster(P.visibility_strength(prob)))
    x1, r1 = P.pcg(s.matvec, vj.apply, s.rhs_cam, tau=1e-30, max_iterations=2000, residual_tolerance=1e-6)
    x2, r2 = P.pcg(s.matvec, lambda v: vj.apply(v), s.rhs_cam, tau=1e-30, max_iterations=2000,
                   residual_tolerance=1e-6)
    assert r1.iterations == r2.iterations
    assert relerr(H(x1), H(x2)) <= 1e-10
