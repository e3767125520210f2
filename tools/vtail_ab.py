"""V-cycle time at a config with the coarse tail off / row-CTA levels only / every
16x16 level up to N MB (dev tool): `python tools/vtail_ab.py [config=4]`."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402
from paper_2007_01941_b200 import _lib, solver  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
obj, jac = P.evaluate(prob)
out = solver.linear_solve(prob, jac, 1e4, cfg)
h = out[6]
r = D.f64(np.random.default_rng(1).standard_normal(h.levels[0].scalar_dim))
ref = None
for mb in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,2,16,32,0,16".split(","))]:
    _lib.call("bamg_mg_set_tail", h._plan.handle, mb)
    h._plan.prepare()
    kinds = [int(_lib.lib().bamg_mg_level_kind(h._plan.handle, li)) for li in range(h.n_levels)]
    for _ in range(3):
        z = h.apply(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        h.apply(r)
    e1.record()
    torch.cuda.synchronize()
    zz = D.host(h.apply(r))
    if ref is None:
        ref = zz
    d = np.max(np.abs(zz - ref)) / np.max(np.abs(ref))
    print(f"tail_mb {mb:4d}: kinds {kinds} V-cycle {e0.elapsed_time(e1) / 50 * 1e3:8.1f} us  rel diff vs off {d:.2e}",
          flush=True)
