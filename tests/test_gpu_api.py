"""Drop-in API behaviour on the GPU, mirroring the reference's own unit tests
(fabricated Jacobians, choose_mode cases, error classes with their payloads) and
live comparisons with the CPU oracle on mid-size BASELINE scenes."""

import numpy as np
import pytest

from conftest import block_rel, relerr

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


def fabricate_jac(P, rng, cam_index, pt_index, n_cameras, n_points):
    """Same construction as the reference's tests/test_schur.py:19-30."""
    k = len(cam_index)
    return P.JacobianBlocks(camera=rng.normal(size=(k, 2, 9)), point=rng.normal(size=(k, 2, 3)),
                            residual=rng.normal(size=(k, 2)), weight=np.ones(k), cam_index=np.asarray(cam_index),
                            pt_index=np.asarray(pt_index), n_cameras=n_cameras, n_points=n_points)


def test_choose_mode_cases(P):
    # reference tests/test_schur.py:182-209
    rng = np.random.default_rng(8)
    jac = fabricate_jac(P, rng, [0, 1, 2, 3, 4], [0, 0, 0, 0, 0], 5, 1)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1.0))
    assert P.covisibility_block_count(s) == 25
    assert P.choose_mode(s) == "implicit"
    rng = np.random.default_rng(9)
    jac = fabricate_jac(P, rng, [0, 1], [0, 1], 2, 2)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1.0))
    assert P.covisibility_block_count(s) == 2
    assert P.choose_mode(s) == "explicit"
    rng = np.random.default_rng(10)
    jac = fabricate_jac(P, rng, [0, 1], [0, 0], 2, 6)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1.0))
    assert 2 * P.covisibility_block_count(s) * 81 == 2 * (s.A.nnz_scalar() + 2 * s.W.nnz_scalar() + s.C.nnz_scalar())
    assert P.choose_mode(s) == "explicit"


def test_fabricated_system_matches_oracle(P):
    from oracle import bamg_oracle as O

    rng = np.random.default_rng(3)
    ci = np.array([0, 1, 2, 0, 2, 3, 1, 3, 4, 4, 0])
    pi = np.array([0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3])
    k = len(ci)
    F, E, r = rng.normal(size=(k, 2, 9)), rng.normal(size=(k, 2, 3)), rng.normal(size=(k, 2))
    jac = P.JacobianBlocks(F, E, r, np.ones(k), ci, pi, 5, 4)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 10.0))
    oj = O.Jac(F, E, r, np.ones(k), ci, pi, 5, 4)
    os_ = O.build_system(oj, O.damping(oj, 10.0))
    assert relerr(H(s.rhs_cam), os_.rhs) <= 1e-12
    S, So = s.ensure_explicit(), os_.explicit()
    np.testing.assert_array_equal(H(S.indptr), So.indptr)
    np.testing.assert_array_equal(H(S.indices), So.indices)
    assert block_rel(H(S.blocks), So.blocks) <= 1e-11
    x = rng.normal(size=45)
    assert relerr(H(s.implicit_matvec(x)), os_.matvec(x)) <= 1e-11
    dc = rng.normal(size=45)
    assert relerr(H(P.back_substitute(s, dc)), O.back_substitute(os_, dc)) <= 1e-11
    assert abs(P.model_decrease(s, dc) - O.model_decrease(os_, dc)) <= 1e-10 * abs(O.model_decrease(os_, dc))


def test_pbj_insufficient_damping_raises(P):
    # reference tests/test_precond.py:95-110
    jac = P.JacobianBlocks(np.zeros((1, 2, 9)), np.zeros((1, 2, 3)), np.ones((1, 2)), np.ones(1), np.array([0]),
                           np.array([0]), 1, 1)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1.0))
    s.A.blocks[0] = 0.0
    s.A.blocks[0, 0, 0] = -1.0
    with pytest.raises(P.IndefiniteBlockError) as e:
        P.pbj_setup(s)
    assert e.value.block_index == 0 and "insufficient damping" in str(e.value)


def test_behind_camera_indices_match_oracle(P):
    from oracle import bamg_oracle as O
    from paper_2007_01941_b200 import scenes

    sc = scenes.ring()
    pts = sc.points.copy()
    # push two points far behind the cameras that see them
    pts[[5, 77]] *= 40.0
    prob = P.BundleProblem(sc.camera_params, pts, sc.cam_index, sc.pt_index, sc.pixels)
    op = O.Problem.of(sc)
    with pytest.raises(O.BehindCamera) as ref:
        O.evaluate(op, None, pts)
    with pytest.raises(P.BehindCameraError) as got:
        P.evaluate(prob)
    np.testing.assert_array_equal(got.value.observation_indices, ref.value.observation_indices)


def test_native_pcg_errors(P):
    rng = np.random.default_rng(0)
    nb = 4
    blocks = np.stack([-(np.eye(9) * (2 + i)) for i in range(nb)])
    A = P.BlockSparseMatrix(nb, nb, 9, 9, np.arange(nb + 1), np.arange(nb), blocks)
    pbj = P.PointBlockJacobi(P.BlockDiagMatrix(np.stack([np.eye(9)] * nb)).factor())
    b = rng.normal(size=nb * 9)
    with pytest.raises(P.CgDivergence, match="nonpositive curvature"):
        P.pcg(A.matvec, pbj.apply, b, tau=0.1)
    A2 = P.BlockSparseMatrix(nb, nb, 9, 9, np.arange(nb + 1), np.arange(nb), -blocks)
    bad = P.BlockDiagMatrix(np.stack([np.eye(9)] * nb), _inv=P._device.f64(np.stack([-np.eye(9)] * nb)))
    with pytest.raises(P.PreconditionerNotSPD, match="at iteration 0"):
        P.pcg(A2.matvec, P.PointBlockJacobi(bad).apply, b, tau=0.1)
    x, rep = P.pcg(A2.matvec, pbj.apply, np.zeros(nb * 9), tau=0.1)
    assert rep.iterations == 0 and rep.stop_reason == "residual_tol"


def _lm_cfg(P, pre, max_coarse=400):
    return P.SolveConfig(preconditioner=pre, tau=1e-30, max_iterations=10, function_tolerance=0.0,
                         gradient_tolerance=0.0, parameter_tolerance=0.0, initial_radius=1e4,
                         cg_max_iterations=20000, mg_max_coarse_dim=max_coarse, cg_residual_tolerance=1e-6)


def test_lm_pbj_matches_oracle(P):
    from oracle import bamg_oracle as O
    from paper_2007_01941_b200 import scenes

    sc = scenes.random_problem(1003, n_cameras=12, n_points=60)
    sol, rep = P.lm_solve(P.BundleProblem(*sc.arrays()), _lm_cfg(P, "pbj"))
    # the oracle's own envelope over 1-ulp perturbations of the cameras: once the LM
    # iterate has converged, PBJ-PCG counts to rel-res 1e-6 are roundoff-sensitive
    runs = []
    for trial in range(4):
        op = O.Problem.of(sc)
        if trial:
            mask = np.random.default_rng(trial).random(op.cams.shape) < 0.5
            op.cams = np.where(mask, np.nextafter(op.cams, np.inf), op.cams)
        _, _, recs, _ = O.lm_solve(op, preconditioner="pbj")
        runs.append(recs)
    cg = np.array([r.cg_iterations for r in rep.records])
    env = np.array([[r.cg_iterations for r in recs] for recs in runs])
    obj = np.array([r.objective for r in runs[0]])
    determined = np.concatenate([[True], (np.abs(obj - obj[-1]) > 1e-9 * abs(obj[-1]))[:-1]])
    lo, hi = env.min(0) - 1, env.max(0) + 1
    assert np.all(((cg >= lo) & (cg <= hi))[determined]), (cg, env)
    np.testing.assert_array_equal(np.array([r.accepted for r in rep.records])[determined],
                                  np.array([r.accepted for r in runs[0]])[determined])
    assert abs(rep.final_objective - obj[-1]) <= 1e-8 * abs(obj[-1])


@pytest.mark.parametrize("which", ["street", "loop", "large"])
def test_midsize_scene_matches_oracle(P, which):
    """Down-scaled BASELINE scenes: structure bit-exact, values 1e-10, PCG counts."""
    from oracle import bamg_oracle as O
    from paper_2007_01941_b200 import scenes

    if which == "street":
        sc = scenes.street(n_points=15_000)
    elif which == "loop":
        sc = scenes.loop(n_cameras=600, n_points=40_000)
    else:
        sc = scenes.large(n_clusters=1, n_points=60_000, threads=4)
    prob = P.BundleProblem(*sc.arrays())
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    s.mode = P.choose_mode(s)
    op = O.Problem.of(sc)
    oobj, ojac = O.evaluate(op)
    os_ = O.build_system(ojac, O.damping(ojac, 1e4))
    os_.mode = O.choose_mode(os_)
    assert abs(obj - oobj) <= 1e-10 * abs(oobj)
    assert s.mode == os_.mode
    S, So = s.ensure_explicit(), os_.explicit()
    np.testing.assert_array_equal(H(S.indptr), So.indptr)
    np.testing.assert_array_equal(H(S.indices), So.indices)
    assert block_rel(H(S.blocks), So.blocks) <= 1e-10
    G = P.visibility_strength(prob)
    Go = O.visibility_strength(op.ci, op.pi, op.nc, op.npt)
    np.testing.assert_array_equal(H(G.data), Go.data)
    agg = P.aggregate(G)
    np.testing.assert_array_equal(H(agg.assignment), O.aggregate(Go)[0])
    h = P.build_hierarchy(s, P.gauge_nullspace(prob), G)
    lv = O.hierarchy(os_, O.gauge_nullspace(op.cams), Go)
    assert [l.scalar_dim for l in h.levels] == [l.dim for l in lv]
    x, rep = P.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
    xo, repo = O.pcg(os_.matvec, lambda r: O.vcycle(lv, 0, None, r), os_.rhs, 1e-30, 20000, 1e-6)
    assert abs(rep.iterations - repo.iterations) <= 1, (rep.iterations, repo.iterations)
    # both solutions meet rel-res 1e-6; they differ by the solvers' own residual error
    assert relerr(H(x), xo) <= 1e-4


def test_lm_trial_decision_on_device(P):
    """bamg_lm_trial (solver.py:276-301): the device decision reproduces the host
    formulas -- decrease, rho, acceptance, step norm -- and on acceptance moves the
    canonicalised candidate into the parameters; rejection and behind-camera
    candidates leave them untouched."""
    import math

    from paper_2007_01941_b200 import _device as D

    nc, npt = 3, 4
    rng = np.random.default_rng(0)
    cams0 = rng.normal(size=(nc, 9))
    cand = cams0 + 0.01
    cand[1, :3] = [4.0, 0.0, 0.0]  # |aa| > pi: canonicalised on acceptance
    pts0, cpts = rng.normal(size=(npt, 3)), rng.normal(size=(npt, 3))

    def run(tvals, behind, min_rho=1e-3, radius=1e4):
        cams, pts = D.f64(cams0.copy()), D.f64(pts0.copy())
        t = D.f64(np.array(tvals + [radius]))
        nb = D.i32(np.array([behind], dtype=np.int32))
        out = D.empty(6)
        D.call("bamg_lm_trial", t, nb, min_rho, cams, D.f64(cand), nc, pts, D.f64(cpts), npt, out)
        return H(out), H(cams), H(pts)

    a, b, c, dcn, dpn, f, fn = 3.0, 2.5, 0.75, 0.04, 0.09, 10.0, 9.0
    out, cams, pts = run([a, b, c, dcn, dpn, f, fn], 0)
    dec = a - 0.5 * b + 0.5 * c
    rho = 0.5 * (f - fn) / dec
    assert out[0] == rho and out[1] == 1.0 and out[2] == dec and out[3] == math.sqrt(dcn + dpn) and out[4] == fn
    np.testing.assert_array_equal(pts, cpts)
    np.testing.assert_array_equal(cams[0], cand[0])
    th = 4.0
    assert abs(cams[1, 0] - th * (1.0 - 2.0 * math.pi / th)) < 1e-15 and np.linalg.norm(cams[1, :3]) <= math.pi
    # rejected: f_new > f
    out, cams, pts = run([a, b, c, dcn, dpn, f, 11.0], 0)
    assert out[0] < 0 and out[1] == 0.0
    np.testing.assert_array_equal(cams, cams0)
    np.testing.assert_array_equal(pts, pts0)
    # candidate behind a camera: rho = -inf, objective kept
    out, cams, _ = run([a, b, c, dcn, dpn, f, fn], 3)
    assert out[0] == -np.inf and out[1] == 0.0 and out[4] == f
    np.testing.assert_array_equal(cams, cams0)
    # nonpositive model decrease: rho = -inf
    out, _, _ = run([0.0, 2.0, 0.0, dcn, dpn, f, fn], 0)
    assert out[0] == -np.inf and out[1] == 0.0
    # the trust-region update (solver.py:134-149) on the device, bit for bit the host's
    # TrustRegion.accept / reject: decrease = 1 and f_new = 0 make rho = f / 2 exactly
    rng = np.random.default_rng(5)
    for rho_want in [1e-3 + 1e-9, 0.25, 0.5, 0.75, 1.0, 1.7, 3.0] + list(rng.uniform(0.002, 2.0, 200)):
        for radius in (1e4, 3.3333e-7, float(rng.uniform(1e-3, 1e6))):
            out, _, _ = run([1.0, 0.0, 0.0, dcn, dpn, 2.0 * rho_want, 0.0], 0, radius=radius)
            assert out[0] == rho_want and out[1] == 1.0
            tr = P.TrustRegion(radius=radius)
            tr.accept(rho_want)
            assert out[5] == tr.radius, (rho_want, radius)
    out, _, _ = run([a, b, c, dcn, dpn, f, 11.0], 0, radius=7.0)
    tr = P.TrustRegion(radius=7.0)
    tr.reject()
    assert out[1] == 0.0 and out[5] == tr.radius


def test_pinned_inputs_match_host_inputs(P):
    """BundleProblem from pinned host tensors (uploads on a copy stream, structural
    passes in their shadow, point-major pixels gathered at the first evaluate) gives
    bit-for-bit the objective, system and step of the plain host-array path, and its
    points / pixels properties read the uploaded values."""
    import torch

    from paper_2007_01941_b200 import scenes, solver

    sc = scenes.street(n_cameras=40, n_points=3000, seed=11)
    arrays = sc.arrays()
    pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrays]
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, cg_max_iterations=2000, mg_max_coarse_dim=40,
                        cg_residual_tolerance=1e-6)
    out = []
    for args in (arrays, pinned):
        prob = P.BundleProblem(*args)
        obj, jac = P.evaluate(prob)
        dc, dp, cg, sys_, *_ = solver.linear_solve(prob, jac, 1e4, cfg)
        out.append((obj, H(dc), H(dp), cg.iterations, H(sys_.rhs_cam), H(prob.points), H(prob.pixels)))
    a, b = out
    assert a[0] == b[0] and a[3] == b[3]
    for u, v in zip(a[1:3] + a[4:], b[1:3] + b[4:]):
        assert np.array_equal(u, v)
    np.testing.assert_array_equal(a[5], arrays[1])
    np.testing.assert_array_equal(a[6], arrays[4])
