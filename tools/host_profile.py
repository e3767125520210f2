"""cProfile of the host side of one warm LM linear solve at a config (dev tool): where
the Python / ctypes time between kernels goes. `python tools/host_profile.py [config=4]`"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(**bench.CFG)
    G = P.visibility_strength(prob)
    _ = prob.structure.pair_lists
    MG._aggregate_cached(G, cfg.mg_max_aggregate)

    def step():
        obj, jac = P.evaluate(prob)
        return solver.linear_solve(prob, jac, cfg.initial_radius, cfg, G)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    step()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)
    st.sort_stats("cumulative").print_stats(45)


if __name__ == "__main__":
    main(*sys.argv[1:])
