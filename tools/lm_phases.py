"""10-step LM at a config with per-step linear-solve seconds, the sync-timed phase
totals (BAMG_PHASES=1) and the time Python's garbage collector spent per step (dev
tool): `BAMG_PHASES=1 python tools/lm_phases.py [config=5] [preconditioner=multigrid] [runs=2]`."""
import gc
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402

GC = {"t": 0.0, "n": 0, "start": 0.0}


def _gc_cb(phase, info):
    if phase == "start":
        GC["start"] = time.perf_counter()
    else:
        GC["t"] += time.perf_counter() - GC["start"]
        GC["n"] += info.get("generation", 0) == 2


def main(config=5, pre="multigrid", runs=2):
    sc = bench.scene_for(int(config))
    gc.callbacks.append(_gc_cb)
    for _ in range(int(runs)):
        cfg = P.SolveConfig(**dict(bench.CFG, preconditioner=pre))
        prob = P.BundleProblem(*sc.arrays())
        D.PHASES.clear()
        GC.update(t=0.0, n=0)
        sol, rep = P.lm_solve(prob, cfg)
        print("linear solve s:", [round(r.setup_seconds + r.solve_seconds, 4) for r in rep.records[1:]])
        print(f"gc: {GC['t'] * 1e3:.1f} ms, {GC['n']} gen-2 collections")
        print({k: round(v, 4) for k, v in sorted(D.PHASES.items(), key=lambda kv: -kv[1])[:14]})


if __name__ == "__main__":
    main(*sys.argv[1:])
