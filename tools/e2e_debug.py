import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import solver
sc = bench.scene_for(4)
cfg = P.SolveConfig(**bench.CFG)
prob = P.BundleProblem(*sc.arrays())
for _ in range(3):
    obj, jac = P.evaluate(prob); out = solver.linear_solve(prob, jac, cfg.initial_radius, cfg)
del out, jac
torch.cuda.synchronize()
host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in sc.arrays()]
dc_h = torch.empty(sc.n_cameras * 9, dtype=torch.float64, pin_memory=True)
dp_h = torch.empty(sc.n_points * 3, dtype=torch.float64, pin_memory=True)
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    prob2 = P.BundleProblem(*host)
    obj, jac = P.evaluate(prob2)
    dc, dp, cg, *_ = solver.linear_solve(prob2, jac, cfg.initial_radius, cfg)
    dc_h.copy_(dc.reshape(-1), non_blocking=True); dp_h.copy_(dp.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    free, tot = torch.cuda.mem_get_info()
    print(it, "%.1f ms" % ((time.perf_counter() - t0) * 1e3), "reserved %.1fG free %.1fG" % (torch.cuda.memory_reserved() / 1e9, free / 1e9), flush=True)
    st = torch.cuda.memory_stats()
    print("   retries", st.get("num_alloc_retries"), "device_alloc", st.get("num_device_alloc"), "device_free", st.get("num_device_free"), "peak %.1fG" % (st["reserved_bytes.all.peak"] / 1e9), flush=True)
    if len(sys.argv) > 1:
        del prob2, obj, jac, dc, dp, cg
