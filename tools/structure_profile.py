"""Per-kernel device time of the per-problem structure pass (orders, covisibility,
strength + level-0 aggregation, Schur pair lists, symmetric view) at a config,
from torch.profiler (dev tool).

  python tools/structure_profile.py [config=4] [top=30]
"""
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import multigrid as MG  # noqa: E402


def main(config=4, top=30):
    sc = bench.scene_for(int(config))
    dev_in = [torch.as_tensor(np.ascontiguousarray(a)).cuda() for a in sc.arrays()]

    def structure():
        pr = P.BundleProblem(*dev_in)
        G = P.visibility_strength(pr)
        _ = pr.structure.symbolic
        _ = pr.structure.pair_lists
        _ = pr.structure.symop
        MG._aggregate_cached(G, 20)
        return pr

    structure()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    structure()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        structure()
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
    print(f"structure pass, config {config}: wall {wall * 1e3:.2f} ms, kernel sum {tot / 1e3:.2f} ms")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(top)]:
        print(f"  {k[:60]:60s} n={v[0]:5d} {v[1] / 1e3:8.3f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
