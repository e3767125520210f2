"""Kernel table of V-cycle applications (graph replay) at a config (dev tool)."""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
obj, jac = P.evaluate(prob)
out = solver.linear_solve(prob, jac, 1e4, cfg)
h = out[6]
r = D.f64(np.random.default_rng(1).standard_normal(h.levels[0].scalar_dim))
for _ in range(3):
    h.apply(r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    h.apply(r)
e1.record()
torch.cuda.synchronize()
print(f"per V-cycle (events, 20 back to back): {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
reps = 10
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        h.apply(r)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name.split("(")[0]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else e.device_time_total
tot = sum(v[1] for v in agg.values())
print(f"per V-cycle: kernel sum {tot / reps:.1f} us; levels {[l.scalar_dim for l in h.levels]}; "
      f"nnz {[l.explicit.n_block_entries for l in h.levels]}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"  {k[:40]:40s} n/cycle={v[0] / reps:5.1f} {v[1] / reps:8.1f} us")
