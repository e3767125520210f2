"""Kernel timeline of one bench step (evaluate + linear solve) at a config: span,
kernel busy time, idle gaps (host round trips) and per-kernel totals (dev tool)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
strength = P.visibility_strength(prob)


def step():
    obj, jac = P.evaluate(prob)
    return solver.linear_solve(prob, jac, 1e4, cfg)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = max(e.time_range.end for e in ev)
# busy = union of intervals (side streams overlap)
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for e in ev:
    s, f = e.time_range.start, e.time_range.end
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_e - t0, e.name.split("(")[0][:40]))
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
print(f"span {(end - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, idle {(end - t0 - busy) / 1e3:.2f} ms, "
      f"{len(ev)} device events")
gaps.sort(reverse=True)
print("largest idle gaps (us, at ms, next kernel):")
for g, at, name in gaps[:25]:
    print(f"  {g:8.1f} at {at / 1e3:7.2f}  {name}")
if len(sys.argv) > 2:  # full ordered listing (start ms, gap us, duration us, stream)
    with open(sys.argv[2], "w") as fh:
        prev = t0
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
print("per kernel:")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {k:50s} n={v[0]:5d} {v[1] / 1e3:8.2f} ms")
