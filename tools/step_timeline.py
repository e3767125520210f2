"""Kernel timeline of ONE bench step at a config (dev tool): every device activity in
start order with its stream, duration and the idle gap before it on the device, plus
the total idle time (host synchronisations / launch latency show up as gaps).

  python tools/step_timeline.py [config=4] [min_gap_us=15] [dump_path]   (dump: every activity)
"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4, min_gap=15.0, dump=None):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(**bench.CFG)
    G = P.visibility_strength(prob)
    _ = prob.structure.symbolic
    MG._aggregate_cached(G, cfg.mg_max_aggregate)

    def step():
        obj, jac = P.evaluate(prob)
        return solver.linear_solve(prob, jac, cfg.initial_radius, cfg, G)

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
        if gap >= float(min_gap):
            print(f"  gap {gap:8.1f} us before {e.name.split('(')[0][:40]:40s} at {s - t0:9.1f}")
        busy_end = max(busy_end, e.time_range.end)
    if dump:
        with open(dump, "w") as fh:
            for e in ev:
                fh.write(f"{e.time_range.start - t0:10.1f} {e.time_range.end - e.time_range.start:9.1f} "
                         f"{e.name.split('(')[0][:60]}\n")
    print(f"config {config}: span {busy_end - t0:.1f} us, device idle {idle:.1f} us, {len(ev)} activities")


if __name__ == "__main__":
    main(*sys.argv[1:])
