import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import golden, vj_inputs
import paper_2007_01941_b200 as P
g = golden("vj_cases")
for tag in ("ring", "r1003"):
    prob = P.BundleProblem(*vj_inputs(tag, g))
    cfg = P.SolveConfig(preconditioner="visibility", tau=1e-30, max_iterations=10, function_tolerance=0.0,
                        gradient_tolerance=0.0, parameter_tolerance=0.0, initial_radius=1e4,
                        cg_max_iterations=20000, cg_residual_tolerance=1e-6)
    sol, rep = P.lm_solve(prob, cfg)
    for r, o, rho, c in zip(rep.records, g[f"{tag}_lm_obj"], g[f"{tag}_lm_rho"], g[f"{tag}_lm_cg"]):
        print(tag, r.iteration, r.cg_iterations, c, "obj rel %.2e" % (abs(r.objective - o) / o), "rho %.6f %.6f" % (r.rho, rho))
