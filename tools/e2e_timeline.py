"""Kernel/copy timeline of one bench e2e step (BundleProblem from pinned host arrays,
evaluate, linear solve, D2H): span, busy, idle gaps, per-kernel totals (dev tool)."""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
cfg = P.SolveConfig(**bench.CFG)
host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in sc.arrays()]
dc_h = torch.empty(sc.n_cameras * 9, dtype=torch.float64, pin_memory=True)
dp_h = torch.empty(sc.n_points * 3, dtype=torch.float64, pin_memory=True)


def step():
    prob = P.BundleProblem(*host)
    obj, jac = P.evaluate(prob)
    dc, dp, *_ = solver.linear_solve(prob, jac, cfg.initial_radius, cfg)
    dc_h.copy_(dc.reshape(-1), non_blocking=True)
    dp_h.copy_(dp.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = max(e.time_range.end for e in ev)
print(f"span {(end - t0) / 1e3:.2f} ms, {len(ev)} device events")
prev = t0
with open(sys.argv[2] if len(sys.argv) > 2 else "/dev/null", "w") as fh:
    for e in ev:
        s_, f_ = e.time_range.start, e.time_range.end
        fh.write(f"{(s_ - t0) / 1e3:9.3f} gap {s_ - prev:8.1f} dur {f_ - s_:8.1f}  {e.name.split('(')[0][:60]}\n")
        prev = max(prev, f_)
agg = {}
for e in ev:
    k = e.name.split("(")[0][:50]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.elapsed_us()
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"  {k:50s} n={v[0]:5d} {v[1] / 1e3:8.2f} ms")
