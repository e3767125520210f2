"""cProfile of one bench step (evaluate + linear_solve) at a config (dev tool).
Blocking readbacks show up as time in .item/.tolist/.cpu/synchronize."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _lib  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)


def step():
    obj, jac = P.evaluate(prob)
    return solver.linear_solve(prob, jac, cfg.initial_radius, cfg)


for _ in range(3):
    step()
torch.cuda.synchronize()
n0 = _lib.lib().bamg_launch_count()
pr = cProfile.Profile()
pr.enable()
out = step()
torch.cuda.synchronize()
pr.disable()
print("kernel launches in the step:", _lib.lib().bamg_launch_count() - n0)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
