"""End-to-end parity of the CUDA path with the reference (golden fixtures from
oracle/make_golden.py) and with the CPU oracle on the same seeded inputs.
Tolerances follow SURVEY Appendix B:
  bit-exact  : S / W patterns, visibility strength (pattern + values), level-0
               aggregation, choose_mode, number of levels, QR branch flags
  1e-10 rel  : F, E, res, objective, A, C, C^-1, W, rhs, S, gauge K,
               full-rank-branch P blocks, level-0 lambda_max
  projector  : pivoted-branch P blocks (Q_r Q_r^T), P K_c = K, P^T P = I
  end-to-end : PCG iterations +-1 per LM step, same accept/reject sequence,
               final objective within 1e-8 relative.
"""

import numpy as np
import pytest

from conftest import block_rel, golden, max_entry_rel, relerr

pytestmark = pytest.mark.gpu

CASES = ["ring_c1", "small_1001", "small_1002", "small_1003", "small_1004", "huber_1005", "implicit_1006"]


def _inputs(name, g):
    from paper_2007_01941_b200 import scenes

    if name == "ring_c1":
        sc = scenes.ring()
        assert sc.digest() == str(g["digest"])
        return sc.camera_params, sc.points, sc.cam_index, sc.pt_index, sc.pixels
    return g["in_cams"], g["in_pts"], g["in_ci"], g["in_pi"], g["in_pix"]


@pytest.fixture(scope="module", params=CASES)
def case(request):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P

    g = golden(request.param)
    prob = P.BundleProblem(*_inputs(request.param, g), loss=str(g["loss"]) if "loss" in g else "trivial")
    obj, jac = P.evaluate(prob)
    damp = P.Damping.from_jacobian(jac, 1e4)
    s = P.build_system(jac, damp)
    return request.param, g, P, prob, obj, jac, damp, s


def H(t):
    from paper_2007_01941_b200 import _device

    return _device.host(t)


def test_evaluate(case):
    _, g, P, prob, obj, jac, *_ = case
    sel = g["obs_sel"]
    assert abs(obj - g["objective"]) <= 1e-10 * abs(g["objective"])
    # per-entry error normalised by the observation block's max-abs entry (App. B.2:
    # entries created by cancellation, e.g. E = D R, carry absolute roundoff)
    assert block_rel(H(jac.camera)[sel], g["F"]) <= 1e-10
    assert block_rel(H(jac.point)[sel], g["E"]) <= 1e-10
    assert block_rel(H(jac.residual)[sel], g["res"]) <= 1e-10


def test_gradient_damping_system(case):
    _, g, P, prob, obj, jac, damp, s = case
    ps = g["pt_sel"]
    gc, gp = jac.gradient()
    assert relerr(H(gc), g["g_cam"]) <= 1e-10
    assert relerr(H(gp)[ps], g["g_pt"]) <= 1e-10
    assert max_entry_rel(H(damp.cam_diag), g["damp_cam"]) <= 1e-10
    assert max_entry_rel(H(damp.pt_diag)[ps], g["damp_pt"]) <= 1e-10
    assert block_rel(H(s.A.blocks), g["A"]) <= 1e-10
    assert block_rel(H(s.C.blocks)[ps], g["C"]) <= 1e-10
    assert block_rel(H(s.C.inverse_blocks())[ps], g["Cinv"]) <= 1e-10
    W = s.W
    np.testing.assert_array_equal(H(W.indptr), g["W_indptr"])
    np.testing.assert_array_equal(H(W.indices), g["W_indices"])
    assert block_rel(H(W.blocks)[g["W_sel"]], g["W_blocks"]) <= 1e-10
    assert relerr(H(s.rhs_cam), g["rhs"]) <= 1e-10
    assert max_entry_rel(H(s.grad_pt).reshape(-1, 3)[ps], g["grad_pt"], 1e-300) <= 1e-10


def test_choose_mode_and_covisibility(case):
    _, g, P, prob, obj, jac, damp, s = case
    assert P.covisibility_block_count(s) == int(g["covis"])
    assert P.choose_mode(s) == str(g["mode"])


def test_schur_explicit(case):
    _, g, P, prob, obj, jac, damp, s = case
    S = s.ensure_explicit()
    np.testing.assert_array_equal(H(S.indptr), g["S_indptr"])
    np.testing.assert_array_equal(H(S.indices), g["S_indices"])
    assert block_rel(H(S.blocks), g["S_blocks"]) <= 1e-10
    # both deterministic assemblies (row-owned / pair-list) agree and rerun bit-identically
    from paper_2007_01941_b200 import schur as SC

    S2 = SC.schur_explicit(s, variant="pairs")
    assert block_rel(H(S2.blocks), H(S.blocks)) <= 1e-12
    S3 = SC.schur_explicit(s)
    assert np.array_equal(H(S3.blocks), H(S.blocks))
    # point-chunk phased assembly, cut into several chunks (partial sums handed over
    # between chunks through the S slots)
    from paper_2007_01941_b200 import problem as PR

    st, old = prob.structure, PR._CHUNK_RECORDS
    try:
        PR._CHUNK_RECORDS, st._chunks = max(8, st.k // 7), None
        S4 = SC.schur_explicit(s, variant="chunks")
        assert st.chunk_plan["n_chunks"] >= 4
        S5 = SC.schur_explicit(s, variant="chunks")
    finally:
        PR._CHUNK_RECORDS, st._chunks = old, None
    assert block_rel(H(S4.blocks), g["S_blocks"]) <= 1e-10
    assert block_rel(H(S4.blocks), H(S.blocks)) <= 1e-12
    assert np.array_equal(H(S5.blocks), H(S4.blocks))
    # implicit operator == explicit operator (schur.py:84-91)
    rng = np.random.default_rng(0)
    x = rng.normal(size=S.shape[0])
    assert relerr(H(s.implicit_matvec(x)), H(S.matvec(x))) <= 1e-10


def test_visibility_strength_bit_exact(case):
    _, g, P, prob, *_ = case
    G = P.visibility_strength(prob)
    np.testing.assert_array_equal(H(G.indptr), g["G_indptr"])
    np.testing.assert_array_equal(H(G.indices), g["G_indices"])
    np.testing.assert_array_equal(H(G.data), g["G_data"])


def test_gauge_nullspace(case):
    _, g, P, prob, *_ = case
    got = H(P.gauge_nullspace(prob).data).reshape(-1, 9, 16)
    assert block_rel(got, g["K"].reshape(-1, 9, 16)) <= 1e-12


@pytest.fixture(scope="module")
def hier(case):
    name, g, P, prob, obj, jac, damp, s = case
    s.mode = P.choose_mode(s)
    G = P.visibility_strength(prob)
    h = P.build_hierarchy(s, P.gauge_nullspace(prob), G, max_coarse_dim=int(g["max_coarse"]))
    return h


def test_hierarchy_structure(case, hier):
    name, g, P, prob, *_ = case
    h = hier
    assert h.n_levels == int(g["n_levels"])
    for li, lvl in enumerate(h.levels):
        assert lvl.scalar_dim == int(g[f"L{li}_dim"])
    if h.n_levels > 1:
        np.testing.assert_array_equal(H(h.levels[0].aggregation.assignment), g["L0_agg"])
        lam = h.levels[0].smoother.lambda_max
        assert abs(lam - g["L0_lambda"]) <= 1e-9 * g["L0_lambda"]


def test_prolongation_level0(case, hier):
    name, g, P, prob, *_ = case
    h = hier
    if h.n_levels < 2:
        pytest.skip("single level")
    lvl = h.levels[0]
    Pb = H(lvl.P.blocks)
    info = H(lvl.P.qr_info)
    agg = H(lvl.aggregation.assignment)
    gold = g["L0_P_blocks"]
    K = H(P.gauge_nullspace(prob).data)
    Pd = H(lvl.P.to_dense())
    Kc = H(h.levels[1].nullspace.data)
    assert np.max(np.abs(Pd @ Kc - K)) <= 1e-12 * np.max(np.abs(K))
    kept = np.abs(Pd).sum(0) > 0
    PtP = Pd.T @ Pd
    np.testing.assert_allclose(PtP[np.ix_(kept, kept)], np.eye(kept.sum()), atol=1e-12)
    for a in range(int(lvl.aggregation.n_aggregates)):
        mem = np.flatnonzero(agg == a)
        mine, ref = Pb[mem].reshape(-1, 16), gold[mem].reshape(-1, 16)
        if info[a, 0] == 0:
            assert np.max(np.abs(mine - ref)) <= 1e-10
        else:
            # the reference's pivoted basis is roundoff-dependent (SURVEY TL;DR hazard 1);
            # the projector onto its first `rank` columns (= range of K_agg) is not
            r = int(info[a, 1])
            pm, pr = mine[:, :r] @ mine[:, :r].T, ref[:, :r] @ ref[:, :r].T
            assert np.max(np.abs(pm - pr)) <= 1e-10


def test_vcycle_symmetric_and_spd(case, hier):
    name, g, P, prob, obj, jac, damp, s = case
    h = hier
    rng = np.random.default_rng(1)
    n = h.levels[0].scalar_dim
    u, v = rng.normal(size=n), rng.normal(size=n)
    Mu, Mv = H(h.apply(u)), H(h.apply(v))
    assert abs(u @ Mv - v @ Mu) <= 1e-10 * abs(u @ Mv)
    assert u @ Mu > 0
    if not H(h.levels[0].P.qr_info)[:, 0].any() if h.n_levels > 1 else True:
        for vin, vout in zip(g["mg_in"], g["mg_out"]):
            assert relerr(H(h.apply(vin)), vout) <= 1e-9


def test_native_runtime_matches_stepwise_path(case, hier):
    """The recorded V-cycle graph / native PCG equal the kernel-by-kernel path."""
    name, g, P, prob, obj, jac, damp, s = case
    from paper_2007_01941_b200 import multigrid as MG

    h = hier
    if h.n_levels > 1 and s.mode == "explicit":
        assert h._plan is not None
    rng = np.random.default_rng(2)
    v = rng.normal(size=h.levels[0].scalar_dim)
    a = H(h.apply(v))
    b = H(MG.mgcycle(h, 0, None, P._device.f64(v)))
    # Same kernels in both paths, but the native plan chunks the coarse-level SpMV and
    # the stepwise one does not (different summation order). cond(S) reaches 7e8 on
    # small_1001; there the two valid roundings differ by ~2e-13 of max|z|.
    assert np.max(np.abs(a - b)) <= 1e-11 * np.max(np.abs(b))
    x1, r1 = P.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=2000, residual_tolerance=1e-6)
    x2, r2 = P.pcg(lambda u: s.matvec(u), lambda u: h.apply(u), s.rhs_cam, tau=1e-30, max_iterations=2000,
                   residual_tolerance=1e-6)
    assert r1.iterations == r2.iterations and r1.stop_reason == r2.stop_reason
    assert relerr(H(x1), H(x2)) <= 1e-10
    np.testing.assert_allclose(r1.q_history, r2.q_history, rtol=1e-10)


def test_pcg_iterations(case, hier):
    name, g, P, prob, obj, jac, damp, s = case
    x, rep = P.pcg(s.matvec, hier.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
    assert abs(rep.iterations - int(g["pcg_its"])) <= 1
    assert relerr(H(x), g["pcg_x"]) <= 1e-4
    pb = P.pbj_setup(s)
    xb, repb = P.pcg(s.matvec, pb.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
    assert abs(repb.iterations - int(g["pbj_its"])) <= 1
    dp = P.back_substitute(s, x)
    assert relerr(H(dp).reshape(-1, 3)[g["pt_sel"]], g["dp"]) <= 1e-4


def test_lm_records(case):
    name, g, P, prob, *_ = case
    if "lm_cg" not in g:
        pytest.skip("no LM record")
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, max_iterations=10, function_tolerance=0.0,
                        gradient_tolerance=0.0, parameter_tolerance=0.0, initial_radius=1e4,
                        cg_max_iterations=20000, mg_max_coarse_dim=int(g["max_coarse"]), cg_residual_tolerance=1e-6)
    sol, rep = P.lm_solve(prob, cfg)
    cg = np.array([r.cg_iterations for r in rep.records])
    acc = np.array([r.accepted for r in rep.records])
    assert len(cg) == len(g["lm_cg"])
    # +-1 around the reference's own envelope over 1-ulp input perturbations
    # (make_golden.py): the pivoted-QR completion is set by roundoff in the
    # reference itself, which moves its own counts by up to 2 on config 1
    lo, hi = g["lm_cg_min"] - 1, g["lm_cg_max"] + 1
    assert np.all((cg >= lo) & (cg <= hi)), (cg, g["lm_cg"], g["lm_cg_min"], g["lm_cg_max"])
    assert np.mean(np.abs(cg - g["lm_cg"])) <= 0.5
    # accept/reject parity on the steps whose ratio is numerically determined: the
    # objective still has > 1e-9 relative decrease left (afterwards both sides
    # compare roundoff-level objective differences)
    obj = g["lm_obj"]
    determined = np.abs(obj - obj[-1]) > 1e-9 * abs(obj[-1])
    determined = np.concatenate([[True], determined[:-1]])
    np.testing.assert_array_equal(acc[determined], g["lm_accepted"][determined])
    assert abs(rep.final_objective - obj[-1]) <= 1e-8 * abs(obj[-1])
