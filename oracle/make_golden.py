"""Generate tests/golden/*.npz by running the REAL reference (build container only).

Test infrastructure. Imports the reference package from
``/root/reference/pkg/src`` (read-only, Python + numpy + scipy), runs it on
seeded inputs, and stores its outputs as small fixtures. The committed fixtures
pin both the oracle restatement (``tests/test_oracle_golden.py``, CPU) and the
CUDA path (``tests/test_gpu_parity.py``, GPU box, where the reference is absent).

Run:  python oracle/make_golden.py            (writes tests/golden/)

Reference settings follow SURVEY 8(d): trivial loss, tau=1e-30, 10 LM steps,
zero stop tolerances, initial radius 1e4, CG residual tolerance 1e-6 patched in
(`solver.py:269-272` does not forward it).
"""

from __future__ import annotations

import functools
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")


def load_reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import bamg  # noqa: F401
    return bamg


def problem_of(bamg, sc):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return bamg.BundleProblem(sc.camera_params, sc.points, sc.cam_index, sc.pt_index, sc.pixels)


def dump_problem(bamg, prob, tag, sample=None, extra=None, lm=True, store_inputs=False,
                 max_coarse=400):
    from bamg import multigrid as mg
    from bamg import schur, solver
    from bamg.problem import evaluate, gauge_nullspace

    out = {}
    if store_inputs:
        out.update(in_cams=prob.camera_params, in_pts=prob.points, in_ci=prob.cam_index,
                   in_pi=prob.pt_index, in_pix=prob.pixels)
    k = prob.n_observations
    sel = np.arange(k) if sample is None else np.arange(0, k, sample)
    out["obs_sel"] = sel
    obj, jac = evaluate(prob)
    out["objective"] = np.float64(obj)
    out["F"] = jac.camera[sel]
    out["E"] = jac.point[sel]
    out["res"] = jac.residual[sel]
    gc, gp = jac.gradient()
    out["g_cam"] = gc
    psel = np.arange(prob.n_points) if sample is None else np.arange(0, prob.n_points, sample)
    out["pt_sel"] = psel
    out["g_pt"] = gp[psel]
    dmp = schur.Damping.from_jacobian(jac, 1e4)
    out["damp_cam"] = dmp.cam_diag
    out["damp_pt"] = dmp.pt_diag[psel]
    s = schur.build_system(jac, dmp)
    out["A"] = s.A.blocks
    out["C"] = s.C.blocks[psel]
    out["Cinv"] = s.C.inverse_blocks()[psel]
    out["W_indptr"] = s.W.indptr
    out["W_indices"] = s.W.indices
    wsel = np.arange(len(s.W.indices)) if sample is None else np.arange(0, len(s.W.indices), sample)
    out["W_sel"] = wsel
    out["W_blocks"] = s.W.blocks[wsel]
    out["rhs"] = s.rhs_cam
    out["grad_pt"] = s.grad_pt.reshape(-1, 3)[psel]
    out["mode"] = np.array(schur.choose_mode(s))
    out["covis"] = np.int64(schur.covisibility_block_count(s))
    S = s.ensure_explicit()
    out["S_indptr"], out["S_indices"], out["S_blocks"] = S.indptr, S.indices, S.blocks
    s.mode = schur.choose_mode(s)
    G = mg.visibility_strength((prob.cam_index, prob.pt_index, prob.n_cameras, prob.n_points))
    out["G_indptr"], out["G_indices"], out["G_data"] = G.g.indptr, G.g.indices, G.g.data
    K = gauge_nullspace(prob)
    out["K"] = K.data
    h = mg.build_hierarchy(s, K, G, max_coarse_dim=max_coarse)
    out["max_coarse"] = np.int64(max_coarse)
    out["n_levels"] = np.int64(h.n_levels)
    for li, lvl in enumerate(h.levels):
        out[f"L{li}_dim"] = np.int64(lvl.scalar_dim)
        if lvl.smoother is not None:
            out[f"L{li}_lambda"] = np.float64(lvl.smoother.lambda_max)
        if lvl.aggregation is not None:
            out[f"L{li}_agg"] = lvl.aggregation.assignment
            out[f"L{li}_P_blocks"] = lvl.P.blocks
            out[f"L{li}_P_indices"] = lvl.P.indices
        if li > 0:
            out[f"L{li}_Kc"] = lvl.nullspace.data
            op = lvl.explicit
            out[f"L{li}_indptr"], out[f"L{li}_indices"] = op.indptr, op.indices
            out[f"L{li}_blocks"] = op.blocks
    rng = np.random.default_rng(5)
    vs = rng.standard_normal((3, prob.n_cameras * 9))
    out["mg_in"] = vs
    out["mg_out"] = np.stack([h.apply(v) for v in vs])
    x, rep = solver.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=20000,
                        residual_tolerance=1e-6)
    out["pcg_x"], out["pcg_its"], out["pcg_reason"] = x, np.int64(rep.iterations), np.array(rep.stop_reason)
    out["pcg_q"] = np.asarray(rep.q_history)
    dp = schur.back_substitute(s, x)
    out["dp"] = dp.reshape(-1, 3)[psel]
    out["model_decrease"] = np.float64(schur.model_decrease(s, x))
    pb = bamg.pbj_setup(s)
    xb, repb = solver.pcg(s.matvec, pb.apply, s.rhs_cam, tau=1e-30, max_iterations=20000,
                          residual_tolerance=1e-6)
    out["pbj_its"] = np.int64(repb.iterations)
    out["pbj_x"] = xb
    if lm:
        orig = solver.pcg
        solver.pcg = functools.partial(orig, residual_tolerance=1e-6)
        try:
            cfg = solver.SolveConfig(preconditioner="multigrid", tau=1e-30, max_iterations=10,
                                     function_tolerance=0.0, gradient_tolerance=0.0,
                                     parameter_tolerance=0.0, initial_radius=1e4,
                                     cg_max_iterations=20000,
                                     mg_max_coarse_dim=max_coarse)
            sol, rep = solver.lm_solve(prob, cfg)
        finally:
            solver.pcg = orig
        recs = rep.records
        # the reference's own sensitivity: the same LM run on 1-ulp perturbed camera
        # parameters (SURVEY TL;DR hazard 1: the pivoted-QR completion is set by
        # roundoff), recorded as a per-step envelope of CG iteration counts
        cgs = [[r.cg_iterations for r in recs]]
        solver.pcg = functools.partial(orig, residual_tolerance=1e-6)
        try:
            for trial in range(1, 5):
                rng = np.random.default_rng(trial)
                cams = prob.camera_params.copy()
                mask = rng.random(cams.shape) < 0.5
                cams = np.where(mask, np.nextafter(cams, np.inf), cams)
                pp = problem_of(bamg, type("S", (), dict(camera_params=cams, points=prob.points,
                                                         cam_index=prob.cam_index, pt_index=prob.pt_index,
                                                         pixels=prob.pixels))())
                _, rp = solver.lm_solve(pp, cfg)
                if len(rp.records) == len(recs):
                    cgs.append([r.cg_iterations for r in rp.records])
        finally:
            solver.pcg = orig
        cgs = np.array(cgs)
        out["lm_cg_min"], out["lm_cg_max"] = cgs.min(0), cgs.max(0)
        out["lm_cg"] = np.array([r.cg_iterations for r in recs])
        out["lm_obj"] = np.array([r.objective for r in recs])
        out["lm_radius"] = np.array([r.radius for r in recs])
        out["lm_accepted"] = np.array([r.accepted for r in recs])
        out["lm_rho"] = np.array([r.rho for r in recs])
        out["lm_final_cams"] = sol.camera_params
    if extra:
        out.update(extra)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{tag}.npz"), **out)
    return out


def main():
    sys.path.insert(0, ROOT)
    bamg = load_reference()
    from paper_2007_01941_b200 import scenes

    sc = scenes.ring()
    prob = problem_of(bamg, sc)
    dump_problem(bamg, prob, "ring_c1", sample=16,
                 extra={"digest": np.array(sc.digest())})
    print("ring_c1 done", flush=True)

    # small problems in the shape of the reference's own test builder
    for seed, nc, npt in [(1001, 6, 20), (1002, 8, 30), (1003, 12, 60), (1004, 30, 200)]:
        sc = scenes.random_problem(seed, n_cameras=nc, n_points=npt)
        prob = problem_of(bamg, sc)
        dump_problem(bamg, prob, f"small_{seed}", store_inputs=True, lm=(nc <= 12),
                     max_coarse=40, sample=(4 if nc > 12 else None))
        print(f"small_{seed} done", flush=True)

    # robust loss (problem.py:179-196): large pixel noise puts many residuals in
    # the Huber region
    sc = scenes.random_problem(1005, n_cameras=12, n_points=60, pixel_noise=3.0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        prob = bamg.BundleProblem(sc.camera_params, sc.points, sc.cam_index, sc.pt_index, sc.pixels,
                                  loss="huber")
    dump_problem(bamg, prob, "huber_1005", store_inputs=True, max_coarse=40,
                 extra={"loss": np.array("huber")})
    print("huber_1005 done", flush=True)

    # dense covisibility with few points: choose_mode picks the implicit operator
    # (schur.py:162-168), so the level-0 smoother runs on A x - W C^-1 W^T x
    sc = scenes.random_problem(1006, n_cameras=50, n_points=15)
    prob = problem_of(bamg, sc)
    dump_problem(bamg, prob, "implicit_1006", store_inputs=True, max_coarse=40)
    print("implicit_1006 done", flush=True)

    # unit known-answer cases (reference tests' hand cases, re-derived by running
    # the reference on the same small inputs)
    from bamg import multigrid as mg
    import scipy.sparse as sp

    def strength(rows, cols, n, v=0.5):
        g = sp.csr_matrix((np.full(len(rows), v), (rows, cols)), shape=(n, n))
        return mg.StrengthMatrix((g + g.T).tocsr())

    cases = {
        "chain": strength([0, 1, 2], [1, 2, 3], 4),
        "star": strength([0, 0, 0], [1, 2, 3], 4),
        "isolated": strength([0], [1], 3),
    }
    rng = np.random.default_rng(3)
    n = 60
    r = rng.integers(0, n, 400)
    c = rng.integers(0, n, 400)
    keep = r != c
    g = sp.csr_matrix((rng.uniform(0.05, 1.0, keep.sum()), (r[keep], c[keep])), shape=(n, n))
    g = (g + g.T).tocsr()
    g.data = np.round(g.data, 2)  # force ties
    cases["random_ties"] = mg.StrengthMatrix(g)
    big = sp.csr_matrix(np.ones((30, 30)) - np.eye(30))
    cases["clique30"] = mg.StrengthMatrix(big)
    agg_out = {}
    for name, st in cases.items():
        a = mg.aggregate(st)
        st.g.sort_indices()
        agg_out[f"{name}_indptr"] = st.g.indptr
        agg_out[f"{name}_indices"] = st.g.indices
        agg_out[f"{name}_data"] = st.g.data
        agg_out[f"{name}_assign"] = a.assignment
    np.savez_compressed(os.path.join(OUT, "aggregate_cases.npz"), **agg_out)
    print("aggregate cases done")


if __name__ == "__main__":
    main()
