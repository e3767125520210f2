"""Phase timing of repeated linear solves on one problem (dev tool)."""
import os, sys, time
os.environ["BAMG_PHASES"] = "1"
sys.path.insert(0, ".")
import torch
import bench
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import solver

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
for rep in range(reps):
    solver.PHASES.clear()
    t0 = time.perf_counter()
    obj, jac = P.evaluate(prob)
    out = solver.linear_solve(prob, jac, 1e4, cfg)
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    print(f"rep {rep}: total {(time.perf_counter()-t0)*1e3:.1f} ms cg={out[2].iterations} "
          f"alloc={torch.cuda.memory_allocated()/1e9:.1f}G reserved={torch.cuda.memory_reserved()/1e9:.1f}G "
          f"free={free/1e9:.1f}G", {k: round(v * 1e3, 2) for k, v in solver.PHASES.items()}, flush=True)
    del out, jac
