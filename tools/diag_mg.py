"""Diagnostics (dev tool): compare the GPU hierarchy / LM trace with a golden fixture."""

import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import golden  # noqa: E402

import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D, scenes  # noqa: E402


def main(name="ring_c1"):
    g = golden(name)
    if name == "ring_c1":
        sc = scenes.ring()
        args = sc.arrays()
    else:
        args = (g["in_cams"], g["in_pts"], g["in_ci"], g["in_pi"], g["in_pix"])
    prob = P.BundleProblem(*args)
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    s.mode = P.choose_mode(s)
    G = P.visibility_strength(prob)
    h = P.build_hierarchy(s, P.gauge_nullspace(prob), G, max_coarse_dim=int(g["max_coarse"]))
    for li, lvl in enumerate(h.levels[:-1]):
        print(f"L{li} lambda gpu={lvl.smoother.lambda_max:.15g} ref={float(g[f'L{li}_lambda']):.15g}")
    lvl = h.levels[0]
    Pb = D.host(lvl.P.blocks)
    info = D.host(lvl.P.qr_info)
    agg = D.host(lvl.aggregation.assignment)
    gold = g["L0_P_blocks"]
    for a in range(min(lvl.aggregation.n_aggregates, 6)):
        mem = np.flatnonzero(agg == a)
        mine, ref = Pb[mem].reshape(-1, 16), gold[mem].reshape(-1, 16)
        print(f"agg {a} size {len(mem)} piv={info[a,0]} rank={info[a,1]} maxdiff cols:",
              np.round(np.max(np.abs(mine - ref), axis=0), 3))
    if h.n_levels > 1:
        A1 = D.host(h.levels[1].explicit.blocks)
        print("L1 nnz", A1.shape, "ref", g["L1_blocks"].shape)
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, max_iterations=10, function_tolerance=0.0,
                        gradient_tolerance=0.0, parameter_tolerance=0.0, initial_radius=1e4,
                        cg_max_iterations=20000, mg_max_coarse_dim=int(g["max_coarse"]), cg_residual_tolerance=1e-6)
    sol, rep = P.lm_solve(prob, cfg)
    for r, c, a, rho, rr in zip(rep.records, g["lm_cg"], g["lm_accepted"], g["lm_rho"], g["lm_radius"]):
        print(f"it {r.iteration} cg {r.cg_iterations}/{c} acc {r.accepted}/{a} rho {r.rho:.6g}/{rho:.6g} "
              f"obj {r.objective:.12g} radius {r.radius:.6g}/{rr:.6g}")
    print("final obj", rep.final_objective, g["lm_obj"][-1])


if __name__ == "__main__":
    main(*sys.argv[1:])
