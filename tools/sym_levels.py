"""Half-storage product of every level that has a symmetric view, timed alone at a
config (dev tool): CUDA events over 50 back-to-back products, bytes as bench.sym_bytes.

  python tools/sym_levels.py [config=4]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402
from paper_2007_01941_b200 import solver  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main(config=4):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(**bench.CFG)
    obj, jac = P.evaluate(prob)
    out = solver.linear_solve(prob, jac, 1e4, cfg)
    h = out[6]
    peak, _ = bench.measured_peak_hbm()
    rows = []
    for li, lvl in enumerate(h.levels):
        A = lvl.explicit
        sym = getattr(A, "_symop", None)
        if sym is None:
            continue
        b, n = A.row_block_size, A.n_block_rows
        x = D.f64(np.random.default_rng(li).standard_normal(n * b))
        y = D.empty(n * b)
        t = timeit(lambda: D.call("bamg_symop_spmv", sym.handle, A.blocks, x, y, None))
        by = bench.sym_bytes(A.n_block_entries, n, sym.nch, b)
        rows.append(dict(level=li, bs=b, rows=n, nnzb=A.n_block_entries, us=round(t, 2),
                         gbs=round(by / t / 1e3, 1), frac=round(by / t / 1e3 / peak, 3)))
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
