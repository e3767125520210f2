"""Phase breakdown of one LM linear solve on the GPU (dev tool; sync-timed, not a bench number)."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

T = {}


def tic():
    torch.cuda.synchronize()
    return time.perf_counter()


def toc(name, t0):
    torch.cuda.synchronize()
    T[name] = T.get(name, 0.0) + time.perf_counter() - t0


def main(config=4, reps=2):
    config, reps = int(config), int(reps)
    sc = bench.scene_for(config)
    print(f"config {config}: {sc.n_cameras} cams {sc.n_points} pts {sc.n_observations} obs", flush=True)
    t0 = tic()
    prob = P.BundleProblem(*sc.arrays())
    toc("problem+orders", t0)
    t0 = tic()
    st = prob.structure
    S_ptr, S_col, nnz, maxrow = st.covis
    toc("covis", t0)
    t0 = tic()
    G = P.visibility_strength(prob)
    toc("strength", t0)
    t0 = tic()
    sym = st.symbolic
    toc("schur_symbolic", t0)
    print(f"nnzS={nnz} max_row={maxrow} pairs={sym['n_pairs']} upper={sym['n_up']}", flush=True)
    for rep in range(reps):
        T.clear()
        t0 = tic()
        obj, jac = P.evaluate(prob)
        toc("evaluate", t0)
        t0 = tic()
        jac.normal_blocks()
        toc("normal_blocks", t0)
        t0 = tic()
        d = P.Damping.from_jacobian(jac, 1e4)
        s = P.build_system(jac, d)
        s.mode = P.choose_mode(s)
        toc("build_system", t0)
        t0 = tic()
        S = s.ensure_explicit()
        toc("schur_numeric", t0)
        # hierarchy, instrumented
        K = P.gauge_nullspace(prob)
        levels = [MG.MgLevel(0, s.matvec, s.n_cameras * 9, s, S, K)]
        Kc = K
        while levels[-1].scalar_dim > 400:
            cur = levels[-1]
            t0 = tic()
            agg = MG._aggregate_cached(G, 20) if cur.index == 0 else MG.aggregate(MG.operator_strength(cur.explicit))
            toc(f"aggregate_L{cur.index}", t0)
            if agg.n_aggregates * 16 / cur.scalar_dim > 0.7:
                break
            t0 = tic()
            Pm, Kn, pad = MG.build_prolongation(agg, Kc, 9 if cur.index == 0 else 16)
            toc(f"prolong_L{cur.index}", t0)
            t0 = tic()
            An = MG.galerkin(Pm, cur.explicit, agg)
            toc(f"galerkin_L{cur.index}", t0)
            cur.P, cur.aggregation = Pm, agg
            levels.append(MG.MgLevel(cur.index + 1, An.matvec, agg.n_aggregates * 16, An, An, Kn))
            Kc = Kn
        for lvl in levels[:-1]:
            t0 = tic()
            jacobi = P.BlockDiagMatrix(lvl.explicit.diagonal_blocks())
            lvl.smoother = MG.make_smoother(lvl.matvec, jacobi, lvl.scalar_dim, seed=20210607 + lvl.index)
            toc(f"smoother_L{lvl.index}", t0)
        t0 = tic()
        levels[-1].coarse_factor = MG._coarse_factor(levels[-1].explicit)
        toc("coarse_factor", t0)
        h = MG.MgHierarchy(levels)
        t0 = tic()
        x, rep_ = P.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=20000, residual_tolerance=1e-6)
        toc("pcg", t0)
        t0 = tic()
        P.back_substitute(s, x)
        toc("back_sub", t0)
        r = np.random.default_rng(0).standard_normal(s.n_cameras * 9)
        t0 = tic()
        for _ in range(5):
            h.apply(r)
        toc("vcycle_x5", t0)
        t0 = tic()
        for _ in range(20):
            S.matvec(r)
        toc("spmv_x20", t0)
        print(f"rep {rep}: cg={rep_.iterations} levels={len(levels)} dims={[l.scalar_dim for l in levels]} "
              f"nnz={[l.explicit.n_block_entries for l in levels]}")
        tot = 0
        for k, v in T.items():
            print(f"  {k:18s} {v * 1e3:9.2f} ms")
        print(f"  lambdas {[round(l.smoother.lambda_max, 4) for l in levels[:-1]]}", flush=True)


def kernels(config=4):
    """CUPTI kernel table (torch.profiler) of one full linear solve after warm-up."""
    from torch.profiler import ProfilerActivity, profile

    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, cg_max_iterations=20000, cg_residual_tolerance=1e-6)
    for _ in range(2):
        obj, jac = P.evaluate(prob)
        solver.linear_solve(prob, jac, 1e4, cfg)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        obj, jac = P.evaluate(prob)
        out = solver.linear_solve(prob, jac, 1e4, cfg)
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name.split("(")[0]
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else e.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"cg={out[2].iterations} setup={out[4]*1e3:.1f}ms solve={out[5]*1e3:.1f}ms kernel-sum={tot/1e3:.1f}ms")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"  {k[:50]:50s} n={v[0]:5d} {v[1]/1e3:8.2f} ms")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "kernels":
        kernels(*sys.argv[2:])
    else:
        main(*sys.argv[1:])
