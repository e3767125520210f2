"""Per-level aggregation diagnostics: strength row lengths, ties, ring-kernel time (dev tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
obj, jac = P.evaluate(prob)
out = solver.linear_solve(prob, jac, 1e4, cfg)
h = out[6]
for li, lv in enumerate(h.levels[:-1]):
    G = P.visibility_strength(prob) if li == 0 else MG.operator_strength(lv.explicit)
    ptr = G.indptr.cpu().numpy()
    val = G._val[: ptr[-1]].cpu().numpy()
    L = np.diff(ptr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    MG.aggregate(G, 20)
    torch.cuda.synchronize()
    e0.record()
    a = MG.aggregate(G, 20)
    e1.record()
    torch.cuda.synchronize()
    asg = a.assignment.cpu().numpy()
    print(f"L{li}: n={G.n} E={ptr[-1]} row mean {L.mean():.1f} max {L.max()} p99 {np.percentile(L, 99):.0f}; "
          f"G==1: {np.mean(val == 1.0):.3f}; n_agg {a.n_aggregates}; aggregate() {e0.elapsed_time(e1) * 1e3:.0f} us",
          flush=True)
