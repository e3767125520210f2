"""Ordered kernel timeline of one V-cycle (graph replay) at a config: start offset,
duration and gap per kernel, plus the span (dev tool)."""
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
print("levels", [(l.explicit.row_block_size, l.explicit.n_block_rows, l.explicit.n_block_entries) for l in h.levels])
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
print(f"events: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per cycle")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        h.apply(r)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
# last cycle: split at synchronize gaps (largest gaps)
starts = [e.time_range.start for e in ev]
n = len(ev) // 3
cyc = ev[-n:]
t0 = cyc[0].time_range.start
prev_end = t0
tot_k = 0.0
for e in cyc:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    print(f"  +{s - t0:8.1f} gap {s - prev_end:6.1f} dur {d:7.1f}  {e.name.split('(')[0][:50]}")
    prev_end = e.time_range.end
    tot_k += d
print(f"span {prev_end - t0:.1f} us, kernel sum {tot_k:.1f} us, {len(cyc)} kernels")
