"""Aggregation scan A/B at a config (dev tool): level-0 (visibility strength) and level-1
(operator strength) scans timed with CUDA events; BAMG_AGG_SEQ=0/1 picks the kernel.
  python tools/agg_ab.py [config=4]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main(config=4):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(**bench.CFG)
    obj, jac = P.evaluate(prob)
    *_, h = solver.linear_solve(prob, jac, 1e4, cfg)
    G0 = P.visibility_strength(prob)
    print(f"config {config} level 0 ({G0.n} nodes): {timed(lambda: MG.aggregate(G0, 20)):.3f} ms (sort + heads + scan)")
    for l in range(1, len(h.levels) - 1):
        G = MG.operator_strength(h.levels[l].explicit)
        print(f"  level {l} ({G.n} nodes): {timed(lambda: MG.aggregate(G, 20)):.3f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
