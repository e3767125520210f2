"""Full-size golden fingerprints of the REAL reference on the BASELINE configs 2-5.

Test infrastructure (north-star "Results must match the
reference ... on config 4"). Runs the reference package -- imported from
``/root/reference/pkg/src`` in the build container, or from its pip install
under ``baseline/_ref`` (``--ref``) on a host with more RAM, for config 4 --
on the seeded scene of ``paper_2007_01941_b200.scenes`` and stores what a
full-size parity test needs without storing gigabytes:

* the scene digest (the generator is deterministic across hosts; checked first);
* sha256 fingerprints of every integer pattern that must be bit-exact: S
  (indptr / indices), the visibility strength (indptr / indices / data bytes),
  every coarse operator's pattern, plus the full aggregation assignment of every
  level (small: <= n_cameras entries);
* fixed-stride samples of the floating-point arrays (F, E, residual, A, C^-1, rhs,
  S blocks, W blocks) with their indices, for 1e-10 checks;
* level dims, lambda_0, PCG iterations / stop reason / solution samples for the
  multigrid and point-block-Jacobi preconditioners at the first linear solve,
  the model decrease;
* optionally the first ``--lm-steps`` LM records (CG iterations, objective,
  radius, accepted, rho) with the reference settings of SURVEY 8(d);
* the reference's own timings on this host (setup/solve seconds per LM step,
  evaluate seconds) and the host description -- evidence for bench.py's CPU arm.

Run (build container):   python oracle/make_golden_full.py 2 --lm-steps 10
Run (GPU box, c4):       python oracle/make_golden_full.py 4 --ref baseline/_ref --lm-steps 2 --out gpurun_out
"""

from __future__ import annotations

import argparse
import functools
import hashlib
import os
import platform
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
N_SAMPLE = 4096


def fp(a) -> str:
    """Fingerprint of an integer / float array, dtype-normalised (int64 / float64)."""
    a = np.asarray(a)
    a = a.astype(np.int64 if a.dtype.kind in "iub" else np.float64)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def sample_idx(n: int, m: int = N_SAMPLE) -> np.ndarray:
    if n <= m:
        return np.arange(n)
    return np.unique(np.linspace(0, n - 1, m).round().astype(np.int64))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--lm-steps", type=int, default=0)
    ap.add_argument("--pbj-lm-steps", type=int, default=0)
    ap.add_argument("--no-pbj", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--tag", default="", help="file suffix (e.g. _pbj for a comparator-only run)")
    ap.add_argument("--lm-only", action="store_true", help="only the LM runs, no per-function fingerprints")
    args = ap.parse_args()
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.abspath(args.ref))
    import bamg
    from bamg import multigrid as mg
    from bamg import schur, solver
    from bamg.problem import evaluate, gauge_nullspace

    from paper_2007_01941_b200 import scenes

    log = functools.partial(print, f"[c{args.config}]", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    sc = scenes.config(args.config)
    out = {"digest": np.array(sc.digest()), "n_cameras": np.int64(sc.n_cameras),
           "n_points": np.int64(sc.n_points), "n_observations": np.int64(sc.n_observations)}
    log(f"scene {sc.digest()} {sc.n_cameras} cams {sc.n_observations} obs ({time.perf_counter() - t0:.1f}s)")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        prob = bamg.BundleProblem(*sc.arrays())
    k = prob.n_observations

    def lm(precond: str, steps: int, prefix: str):
        orig = solver.pcg
        solver.pcg = functools.partial(orig, residual_tolerance=1e-6)
        try:
            cfg = solver.SolveConfig(preconditioner=precond, tau=1e-30, max_iterations=steps,
                                     function_tolerance=0.0, gradient_tolerance=0.0, parameter_tolerance=0.0,
                                     initial_radius=1e4, cg_max_iterations=20000)
            t = time.perf_counter()
            sol, rp = solver.lm_solve(prob, cfg)
            wall = time.perf_counter() - t
        finally:
            solver.pcg = orig
        recs = rp.records
        out[f"{prefix}_cg"] = np.array([r.cg_iterations for r in recs])
        out[f"{prefix}_obj"] = np.array([r.objective for r in recs])
        out[f"{prefix}_radius"] = np.array([r.radius for r in recs])
        out[f"{prefix}_accepted"] = np.array([r.accepted for r in recs])
        out[f"{prefix}_rho"] = np.array([r.rho for r in recs])
        out[f"{prefix}_setup_s"] = np.array([r.setup_seconds for r in recs])
        out[f"{prefix}_solve_s"] = np.array([r.solve_seconds for r in recs])
        out[f"{prefix}_wall_s"] = np.float64(wall)
        log(f"{prefix} {wall:.1f}s cg {out[f'{prefix}_cg'].tolist()} acc {out[f'{prefix}_accepted'].astype(int).tolist()}")

    def finish():
        import numpy
        import scipy

        out["host"] = np.array(f"{platform.processor() or platform.machine()} cpus={os.cpu_count()} "
                               f"numpy={numpy.__version__} scipy={scipy.__version__} "
                               f"OMP_NUM_THREADS={os.environ.get('OMP_NUM_THREADS', '')}")
        out["ref_path"] = np.array(os.path.abspath(args.ref))
        os.makedirs(args.out, exist_ok=True)
        path = os.path.join(args.out, f"full_c{args.config}{args.tag}.npz")
        np.savez_compressed(path, **out)
        log(f"wrote {path} ({os.path.getsize(path) / 1e6:.1f} MB) total {time.perf_counter() - t0:.0f}s")

    if args.lm_only:
        if args.lm_steps:
            lm("multigrid", args.lm_steps, "lm")
        if args.pbj_lm_steps:
            lm("pbj", args.pbj_lm_steps, "pbj_lm")
        return finish()

    t = time.perf_counter()
    obj, jac = evaluate(prob)
    out["time_evaluate"] = np.float64(time.perf_counter() - t)
    out["objective"] = np.float64(obj)
    osel = sample_idx(k, 2048)
    out["obs_sel"] = osel
    out["F"], out["E"], out["res"] = jac.camera[osel], jac.point[osel], jac.residual[osel]
    gc, gp = jac.gradient()
    csel = sample_idx(prob.n_cameras, 512)
    dsel = sample_idx(prob.n_cameras * 9, 16384)
    out["cam_sel"], out["dof_sel"] = csel, dsel
    out["g_cam"] = gc.reshape(-1)[dsel]
    psel = sample_idx(prob.n_points, 2048)
    out["pt_sel"] = psel
    out["g_pt"] = gp[psel]
    log(f"evaluate {out['time_evaluate']:.1f}s objective {obj:.17g}")

    t = time.perf_counter()
    dmp = schur.Damping.from_jacobian(jac, 1e4)
    s = schur.build_system(jac, dmp)
    s.mode = schur.choose_mode(s)
    out["time_build_system"] = np.float64(time.perf_counter() - t)
    out["A"] = s.A.blocks[csel]
    out["Cinv"] = s.C.inverse_blocks()[psel]
    out["W_indptr_fp"], out["W_indices_fp"] = np.array(fp(s.W.indptr)), np.array(fp(s.W.indices))
    wsel = sample_idx(len(s.W.indices), 1024)
    out["W_sel"], out["W_blocks"] = wsel, s.W.blocks[wsel]
    out["rhs"] = s.rhs_cam[dsel]
    out["rhs_norm"] = np.float64(np.linalg.norm(s.rhs_cam))
    out["grad_pt"] = s.grad_pt.reshape(-1, 3)[psel]
    out["mode"] = np.array(s.mode)
    out["covis"] = np.int64(schur.covisibility_block_count(s))
    log(f"build_system {out['time_build_system']:.1f}s mode {s.mode}")

    t = time.perf_counter()
    S = s.ensure_explicit()
    out["time_schur"] = np.float64(time.perf_counter() - t)
    out["S_nnzb"] = np.int64(len(S.indices))
    out["S_indptr_fp"], out["S_indices_fp"] = np.array(fp(S.indptr)), np.array(fp(S.indices))
    ssel = sample_idx(len(S.indices), 1024)
    out["S_sel"], out["S_blocks"] = ssel, S.blocks[ssel]
    # the row / column of each sampled block, so a test can address it
    out["S_sel_col"] = S.indices[ssel]
    out["S_sel_row"] = np.searchsorted(S.indptr, ssel, side="right") - 1
    log(f"schur_explicit {out['time_schur']:.1f}s nnzb {len(S.indices)}")

    t = time.perf_counter()
    G = mg.visibility_strength((prob.cam_index, prob.pt_index, prob.n_cameras, prob.n_points))
    out["G_indptr_fp"], out["G_indices_fp"] = np.array(fp(G.g.indptr)), np.array(fp(G.g.indices))
    out["G_data_fp"] = np.array(fp(G.g.data))
    K = gauge_nullspace(prob)
    h = mg.build_hierarchy(s, K, G)
    out["time_mg_setup"] = np.float64(time.perf_counter() - t)
    out["n_levels"] = np.int64(h.n_levels)
    for li, lvl in enumerate(h.levels):
        out[f"L{li}_dim"] = np.int64(lvl.scalar_dim)
        if lvl.smoother is not None:
            out[f"L{li}_lambda"] = np.float64(lvl.smoother.lambda_max)
        if lvl.aggregation is not None:
            out[f"L{li}_agg"] = lvl.aggregation.assignment
        if li > 0:
            op = lvl.explicit
            out[f"L{li}_nnzb"] = np.int64(len(op.indices))
            out[f"L{li}_indptr_fp"], out[f"L{li}_indices_fp"] = np.array(fp(op.indptr)), np.array(fp(op.indices))
    log(f"mg setup {out['time_mg_setup']:.1f}s levels {[int(out[f'L{i}_dim']) for i in range(h.n_levels)]}")

    t = time.perf_counter()
    x, rep = solver.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
    out["time_pcg"] = np.float64(time.perf_counter() - t)
    out["pcg_its"], out["pcg_reason"] = np.int64(rep.iterations), np.array(rep.stop_reason)
    out["pcg_rel"] = np.float64(rep.relative_residual)
    out["pcg_x"] = x[dsel]
    out["pcg_x_norm"] = np.float64(np.linalg.norm(x))
    dp = schur.back_substitute(s, x)
    out["dp"] = dp.reshape(-1, 3)[psel]
    out["model_decrease"] = np.float64(schur.model_decrease(s, x))
    log(f"pcg {out['time_pcg']:.1f}s its {rep.iterations}")
    if not args.no_pbj:
        t = time.perf_counter()
        pb = bamg.pbj_setup(s)
        xb, repb = solver.pcg(s.matvec, pb.apply, s.rhs_cam, tau=1e-30, max_iterations=20000,
                              residual_tolerance=1e-6)
        out["time_pbj_pcg"] = np.float64(time.perf_counter() - t)
        out["pbj_its"] = np.int64(repb.iterations)
        out["pbj_x"] = xb[dsel]
        log(f"pbj pcg {out['time_pbj_pcg']:.1f}s its {repb.iterations}")
    del h, S, s, jac

    if args.lm_steps:
        lm("multigrid", args.lm_steps, "lm")
    if args.pbj_lm_steps:
        lm("pbj", args.pbj_lm_steps, "pbj_lm")
    finish()


if __name__ == "__main__":
    main()
