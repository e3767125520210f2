"""Pair-list statistics of the explicit-S assembly (dev tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
st = prob.structure
p = st.pair_lists
ptr = p["blk_ptr"].cpu().numpy().astype(np.int64)
pa = p["pair_a"].cpu().numpy()[: ptr[-1]]
pb = p["pair_b"].cpu().numpy()[: ptr[-1]]
cnt = np.diff(ptr)
up = p["up_blk"].cpu().numpy()[: p["n_up"]]
c = cnt[up]
print("n_pairs", ptr[-1], "n_up", p["n_up"], "pairs/block mean", c.mean(), "median", np.median(c), "max", c.max())
print("pairs in blocks with <=4 pairs:", c[c <= 4].sum() / c.sum(), "blocks:", (c <= 4).mean())
lo = pa[ptr[up][c > 0]]
hi = pa[ptr[up][c > 0] + c[c > 0] - 1]
sp = hi - lo
print("record spread per block: median", np.median(sp), "p90", np.percentile(sp, 90), "of", pa.max())
print("bytes if each pair reads 2x192B:", ptr[-1] * 384 / 1e9, "GB; records once:", (int(pa.max()) + 1) * 256 / 1e9, "GB")
