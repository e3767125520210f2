"""Where the end-to-end step goes (dev tool): the bench's e2e step from pinned host
arrays, with a synchronised timer around each structural stage."""

import os
import sys
import time

os.environ["BAMG_PHASES"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4, reps=3):
    sc = bench.scene_for(int(config))
    cfg = P.SolveConfig(**bench.CFG)
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in sc.arrays()]
    for rep in range(int(reps)):
        T = {}

        def mark(name, t0):
            torch.cuda.synchronize()
            T[name] = (time.perf_counter() - t0) * 1e3
            return time.perf_counter()

        solver.PHASES.clear()
        torch.cuda.synchronize()
        t_all = t = time.perf_counter()
        prob = P.BundleProblem(*host)
        t = mark("problem(h2d+orders)", t)
        st = prob.structure
        st.covis
        t = mark("covis", t)
        P.visibility_strength(prob)
        t = mark("strength", t)
        st.pair_lists
        t = mark("pair_lists", t)
        st.symop
        t = mark("symop", t)
        from paper_2007_01941_b200.blockmat import SymmetricPattern

        S_ptr, S_col, nnz, _ = st.covis
        p = st.pair_lists
        SymmetricPattern(S_ptr, S_col, p["dpos"], p["up_blk"], p["up_tpos"], p["n_up"], st.nc)
        t = mark("symop_again", t)
        obj, jac = P.evaluate(prob)
        t = mark("evaluate", t)
        dc, dp, cg, *_ = solver.linear_solve(prob, jac, cfg.initial_radius, cfg)
        t = mark("linear_solve", t)
        dc_h = torch.empty(dc.numel(), dtype=torch.float64, pin_memory=True)
        dp_h = torch.empty(dp.numel(), dtype=torch.float64, pin_memory=True)
        t = mark("pin_alloc", t)
        dc_h.copy_(dc.reshape(-1), non_blocking=True)
        dp_h.copy_(dp.reshape(-1), non_blocking=True)
        t = mark("d2h", t)
        T["total"] = (time.perf_counter() - t_all) * 1e3
        print(f"rep {rep}:", {k: round(v, 2) for k, v in T.items()},
              {k: round(v * 1e3, 2) for k, v in solver.PHASES.items()}, flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
