"""Reference cycles left behind by one public-API step (dev tool): objects only the
cyclic collector can free keep their device tensors until a collection runs.
  python tools/find_cycles.py"""
import gc
import sys
from collections import Counter

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import scenes, solver  # noqa: E402


def main():
    sc = scenes.street(n_cameras=60, n_points=6000, seed=1)
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in sc.arrays()]
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, cg_max_iterations=500, cg_residual_tolerance=1e-6,
                        mg_max_coarse_dim=40)

    def step():
        prob = P.BundleProblem(*host)
        obj, jac = P.evaluate(prob)
        dc, dp, cg, *_ = solver.linear_solve(prob, jac, 1e4, cfg)
        torch.cuda.synchronize()

    for _ in range(3):
        step()
    gc.collect()
    gc.set_debug(gc.DEBUG_SAVEALL)
    step()
    n = gc.collect()
    print("unreachable objects found by the collector after one step:", n)
    cnt = Counter(type(o).__module__ + "." + type(o).__qualname__ for o in gc.garbage)
    for k, v in cnt.most_common(25):
        print(f"  {v:5d} {k}")
    ours = [o for o in gc.garbage if type(o).__module__.startswith("paper_2007")]
    for o in ours[:12]:
        refs = [type(r).__qualname__ for r in gc.get_referrers(o) if r is not gc.garbage and r is not ours][:6]
        print("  ", type(o).__qualname__, "<-", refs)
    tens = [o for o in gc.garbage if isinstance(o, torch.Tensor)]
    print("tensors held by cycles:", len(tens), "bytes", sum(t.numel() * t.element_size() for t in tens))


if __name__ == "__main__":
    main()
