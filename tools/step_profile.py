"""Per-kernel device time of ONE bench step (evaluate + linear solve) at a config,
after warm-up, from torch.profiler's CUDA activity (dev tool; not a bench number).

  python tools/step_profile.py [config=4] [top=45] [detail=kernel,kernel]
"""

import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def main(config=4, top=45, detail=""):
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
    from paper_2007_01941_b200 import _device as D

    if D._PHASE_ON:  # BAMG_PHASES=1: sync-timed phases of one step (diagnostic)
        D.PHASES.clear()
        step()
        print("phases (ms):", {k: round(v * 1e3, 2) for k, v in D.PHASES.items()})
    t0 = time.perf_counter()
    out = step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = step()
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name.split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_total
    tot = sum(v[1] for v in agg.values())
    for name in filter(None, detail.split(",")):  # individual launches of these kernels, in order
        evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA" and name in e.name),
                     key=lambda e: e.time_range.start)
        print(f"  {name}: " + " ".join(f"{e.device_time_total:.0f}" for e in evs) + " us")
    print(f"config {config}: wall {wall * 1e3:.2f} ms, kernel sum {tot / 1e3:.2f} ms, cg {out[2].iterations}, "
          f"levels {[l.scalar_dim for l in out[6].levels]}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(top)]:
        print(f"  {k[:60]:60s} n={v[0]:5d} {v[1] / 1e3:8.3f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
