"""Kernel table of the multigrid setup alone (build_hierarchy after S is assembled):
device time per kernel vs the synchronised wall time, to separate kernel work from
launch gaps / host synchronisation (dev tool)."""

import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402


def main(config=4):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    G = P.visibility_strength(prob)
    K = P.gauge_nullspace(prob)

    def setup():
        obj, jac = P.evaluate(prob)
        s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
        s.mode = P.choose_mode(s)
        s.ensure_explicit()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = P.build_hierarchy(s, K, G)
        torch.cuda.synchronize()
        return h, time.perf_counter() - t0

    for _ in range(2):
        setup()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        h, wall = setup()
    agg = {}
    t_lo, t_hi = None, None
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name.split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else e.device_time_total
    tot = sum(v[1] for v in agg.values())
    print(f"build_hierarchy wall {wall * 1e3:.1f} ms, kernel sum {tot / 1e3:.1f} ms, "
          f"{sum(v[0] for v in agg.values())} device ops; levels {[l.scalar_dim for l in h.levels]}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"  {k[:50]:50s} n={v[0]:5d} {v[1] / 1e3:8.3f} ms")
    if len(sys.argv) > 2:  # timeline of the hierarchy build: start offset, duration, gap
        ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"),
                    key=lambda e: e.time_range.start)
        first = next(i for i, e in enumerate(ev) if e.name.startswith("k_aggregate") or "sort_desc" in e.name
                     or "op_strength" in e.name or "block_fro" in e.name)
        t0 = ev[first].time_range.start
        prev_end = t0
        for e in ev[first:]:
            st, en = e.time_range.start, e.time_range.end
            print(f"  {(st - t0) / 1e3:8.3f} ms  {en - st:8.1f} us  gap {st - prev_end:7.1f}  {e.name.split('(')[0][:44]}")
            prev_end = max(prev_end, en)


if __name__ == "__main__":
    main(*sys.argv[1:2])
