import sys, time, os
sys.path.insert(0, ".")
import torch
import bench
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import _device as D
sc = bench.scene_for(5)
for pre in ("multigrid", "multigrid"):
    cfg = P.SolveConfig(**dict(bench.CFG, preconditioner=pre))
    prob = P.BundleProblem(*sc.arrays())
    D.PHASES.clear()
    sol, rep = P.lm_solve(prob, cfg)
    print([round(r.setup_seconds + r.solve_seconds, 4) for r in rep.records[1:]])
    print({k: round(v, 4) for k, v in sorted(D.PHASES.items(), key=lambda kv: -kv[1])[:14]})
