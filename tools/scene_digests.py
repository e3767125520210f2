import sys, time
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_01941_b200 import scenes
for n in [int(a) for a in sys.argv[1:]]:
    t=time.time(); sc = scenes.config(n)
    print(n, sc.digest(), sc.n_cameras, sc.n_points, sc.n_observations, f"{time.time()-t:.1f}s", flush=True)
