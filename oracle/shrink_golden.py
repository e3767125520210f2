"""Sub-sample the fixed-stride samples of a full-size golden (oracle/make_golden_full.py)
to the generator's current sample sizes, keeping every (index, value) pair aligned.
Test infrastructure: only thins reference outputs, computes nothing.

  python oracle/shrink_golden.py tests/golden/full_c2.npz
"""

import sys

import numpy as np

GROUPS = {  # selection key -> (arrays indexed by it, target size)
    "obs_sel": (["F", "E", "res"], 2048),
    "pt_sel": (["g_pt", "Cinv", "grad_pt", "dp"], 2048),
    "cam_sel": (["A"], 512),
    "W_sel": (["W_blocks"], 1024),
    "S_sel": (["S_blocks", "S_sel_col", "S_sel_row"], 1024),
}


def main(path):
    g = dict(np.load(path, allow_pickle=False))
    if "cam_sel" not in g:  # older layout: A stored for every camera
        g["cam_sel"] = np.arange(g["A"].shape[0])
    for key, (names, m) in GROUPS.items():
        n = len(g[key])
        if n <= m:
            continue
        keep = np.unique(np.linspace(0, n - 1, m).round().astype(np.int64))
        g[key] = g[key][keep]
        for nm in names:
            if nm in g:
                g[nm] = g[nm][keep]
    np.savez_compressed(path, **g)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
