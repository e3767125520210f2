"""Device timeline of ONE e2e bench step (pinned host inputs -> BundleProblem ->
evaluate -> linear solve -> D2H), from torch.profiler's CUDA activity (dev tool):
the copies, the largest kernels and the idle gaps, in start order.

  python tools/e2e_timeline.py [config=4] [min_us=200] [from_us] [to_us]
(with a window, every activity inside it is listed)
"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4, min_us=200.0, w0=None, w1=None):
    sc = bench.scene_for(int(config))
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
    ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    busy_end = t0
    idle = 0.0
    for e in ev:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = s - busy_end
        if gap > 0:
            idle += gap
        inwin = w0 is not None and float(w0) <= s - t0 <= float(w1)
        if gap >= float(min_us) or (inwin and gap >= 3):
            print(f"  gap {gap:9.1f} us", flush=True)
        if inwin or d >= float(min_us) or "Memcpy" in e.name and d >= 20:
            print(f"  {s - t0:9.1f} +{d:8.1f} us  {e.name.split('(')[0][:60]}")
        busy_end = max(busy_end, e.time_range.end)
    print(f"config {config}: span {busy_end - t0:.1f} us, device idle {idle:.1f} us, {len(ev)} activities")


if __name__ == "__main__":
    main(*sys.argv[1:])
