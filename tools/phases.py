"""Phase timing of repeated linear solves on one problem (dev tool)."""
import os, sys, time
os.environ["BAMG_PHASES"] = "1"
sys.path.insert(0, ".")
import torch
import bench
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import solver

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
for rep in range(4):
    solver.PHASES.clear()
    t0 = time.perf_counter()
    obj, jac = P.evaluate(prob)
    out = solver.linear_solve(prob, jac, 1e4, cfg)
    torch.cuda.synchronize()
    print(f"rep {rep}: total {(time.perf_counter()-t0)*1e3:.1f} ms cg={out[2].iterations}",
          {k: round(v * 1e3, 2) for k, v in solver.PHASES.items()}, flush=True)
