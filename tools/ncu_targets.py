"""Kernels of interest inside an NVTX range "target" (profile with
`ncu --nvtx --nvtx-include "target/" ...`): level-0 S SpMV, one V-cycle (all
levels), the explicit Schur assembly, the Jacobian evaluation."""

import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402
from paper_2007_01941_b200 import schur as SC  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4, what="spmv,vcycle,schur,evaluate"):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(**bench.CFG)
    obj, jac = P.evaluate(prob)
    dc, dp, cg, s, *_ , h = solver.linear_solve(prob, jac, 1e4, cfg)
    S = s.ensure_explicit()
    x = D.f64(torch.randn(S.shape[0], dtype=torch.float64))
    y = D.empty(S.shape[0])
    torch.cuda.synchronize()
    what = what.split(",")
    torch.cuda.nvtx.range_push("target")
    if "spmv" in what:
        D.call("bamg_bsr_spmv", 9, S._ptr, S._col, S.blocks, x, y, S.n_block_rows, None)
    if "galerkin" in what:
        from paper_2007_01941_b200 import multigrid as MG

        lv = h.levels[0]
        MG.galerkin(lv.P, lv.explicit, lv.aggregation)  # level 0 -> 1
    if "agg" in what:
        from paper_2007_01941_b200 import multigrid as MG

        MG.aggregate(P.visibility_strength(prob), 20)  # level-0 greedy scan, uncached
    if "agg1" in what:
        from paper_2007_01941_b200 import multigrid as MG

        MG.aggregate(MG.operator_strength(h.levels[1].explicit), 20)  # level-1 scan
    if "sym" in what:
        S.matvec(x)  # half-storage product (k_sym9_upper + k_sym9_finish)
    if "vcycle" in what:
        h.apply(x)
    if "schur" in what:
        SC.schur_explicit(s)
    if "evaluate" in what:
        P.evaluate(prob)
    if "backsub" in what:
        P.back_substitute(s, dc)
    if "build" in what:
        P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("done", cg.iterations)


if __name__ == "__main__":
    main(*sys.argv[1:])
