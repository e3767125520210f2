import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import solver
sc = bench.scene_for(4)
prob = P.BundleProblem(*sc.arrays())
cfg = P.SolveConfig(**bench.CFG)
for _ in range(3):
    obj, jac = P.evaluate(prob)
    solver.linear_solve(prob, jac, 1e4, cfg)
torch.cuda.synchronize()
obj, jac = P.evaluate(prob)
pr = cProfile.Profile()
pr.enable()
solver.linear_solve(prob, jac, 1e4, cfg)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
