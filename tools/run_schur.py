"""Run the explicit-S assembly variants once each on a config (dev tool for ncu / timing)."""

import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import schur as SC  # noqa: E402


def main(config=4, variants="rows,pairs", reps=3):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    st = prob.structure
    _ = st.symbolic
    if "pairs" in variants:
        _ = st.pair_lists
    torch.cuda.synchronize()
    if "chunks" in variants:
        t0 = time.perf_counter()
        ch = st.chunk_plan
        torch.cuda.synchronize()
        print(f"chunk plan: {(time.perf_counter() - t0) * 1e3:.1f} ms, segments {ch['n_seg']}, "
              f"work {ch['n_work']}, chunks {ch['n_chunks']}", flush=True)
    for v in variants.split(","):
        SC.schur_explicit(s, variant=v)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(int(reps)):
            SC.schur_explicit(s, variant=v)
        torch.cuda.synchronize()
        print(f"{v}: {(time.perf_counter() - t0) / int(reps) * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
