"""Explicit-S assembly variants on one scene: time, agreement with each other and,
with --oracle, with the CPU oracle (dev tool).

  python tools/schur_check.py ring|street|loop_small|large1|large1m|c4 [pairs,rows] [--oracle]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import scenes  # noqa: E402
from paper_2007_01941_b200 import schur as SC  # noqa: E402

SCENES = {"ring": lambda: scenes.ring(), "street": lambda: scenes.street(),
          "loop_small": lambda: scenes.loop(n_cameras=600, n_points=40_000),
          "large1": lambda: scenes.large(n_clusters=1, n_points=112_500),
          "large1m": lambda: scenes.large(n_clusters=1, n_points=30_000),
          "c4": lambda: scenes.config(4)}


def main(which="ring"):
    sc = SCENES[which]()
    prob = P.BundleProblem(*sc.arrays())
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    _ = prob.structure.pair_lists
    _ = prob.structure.chunk_plan
    torch.cuda.synchronize()
    vs = [a for a in sys.argv[2:] if not a.startswith("--")]
    out = {}
    for v in vs[0].split(",") if vs else ("pairs", "rows"):
        SC.schur_explicit(s, variant=v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            S = SC.schur_explicit(s, variant=v)
        e1.record()
        torch.cuda.synchronize()
        out[v] = S.blocks.cpu().numpy()
        print(f"{which} {v}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
    if "--oracle" in sys.argv:
        from oracle import bamg_oracle as O

        op = O.Problem.of(sc)
        oobj, ojac = O.evaluate(op)
        So = O.build_system(ojac, O.damping(ojac, 1e4)).explicit().blocks
        sc_ = np.abs(So).reshape(len(So), -1).max(1)
        for v, a in out.items():
            d = np.abs(a - So).reshape(len(So), -1).max(1) / np.where(sc_ > 0, sc_, 1)
            print(f"{which} {v} vs oracle: max rel {d.max():.3e}, bad {np.flatnonzero(d > 1e-10)[:10]}", flush=True)
    names = list(out)
    for v in names[1:]:
        a, b = out[names[0]], out[v]
        sc_ = np.abs(a).reshape(len(a), -1).max(1)
        d = np.abs(a - b).reshape(len(a), -1).max(1) / np.where(sc_ > 0, sc_, 1)
        print(f"{which} {names[0]} vs {v}: max rel {d.max():.3e}, bad {np.flatnonzero(d > 1e-12)[:10]}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
