"""cProfile of build_hierarchy at a config (dev tool): host time per function,
including time blocked in device synchronisation (.item(), readbacks)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402

sc = bench.scene_for(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = P.BundleProblem(*sc.arrays())
G = P.visibility_strength(prob)
K = P.gauge_nullspace(prob)


def once():
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    s.mode = P.choose_mode(s)
    s.ensure_explicit()
    torch.cuda.synchronize()
    return s


for _ in range(2):
    s = once()
    P.build_hierarchy(s, K, G)
s = once()
pr = cProfile.Profile()
pr.enable()
h = P.build_hierarchy(s, K, G)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
