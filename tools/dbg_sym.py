import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_parity import _inputs, golden
import paper_2007_01941_b200 as P
from paper_2007_01941_b200 import multigrid as MG, _device as D
name = "small_1001"
g = golden(name)
prob = P.BundleProblem(*_inputs(name, g))
obj, jac = P.evaluate(prob)
s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
s.mode = P.choose_mode(s)
h = P.build_hierarchy(s, P.gauge_nullspace(prob), P.visibility_strength(prob), max_coarse_dim=int(g["max_coarse"]))
print("levels", h.n_levels, [l.scalar_dim for l in h.levels], s.mode)
S = s.ensure_explicit()
print("nbr", S.n_block_rows, "nnz", S.n_block_entries)
v = np.random.default_rng(2).normal(size=h.levels[0].scalar_dim)
a1 = D.host(h.apply(v)); a2 = D.host(h.apply(v))
b1 = D.host(MG.mgcycle(h, 0, None, D.f64(v))); b2 = D.host(MG.mgcycle(h, 0, None, D.f64(v)))
print("native repeat", np.max(np.abs(a1-a2)), "step repeat", np.max(np.abs(b1-b2)), "a-b", np.max(np.abs(a1-b1)), np.max(np.abs(b1)))
x = D.f64(v)
y1 = D.host(S.matvec(x)); y2 = D.host(S.matvec(x))
full = D.empty(S.shape[0]); D.call("bamg_bsr_spmv", 9, S._ptr, S._col, S.blocks, x, full, S.n_block_rows, None)
print("spmv repeat", np.max(np.abs(y1-y2)), "sym-full", np.max(np.abs(y1-D.host(full))), np.max(np.abs(y1)))
# stepwise with the full-storage kernels for level 0
S._symop = None
b3 = D.host(MG.mgcycle(h, 0, None, D.f64(v)))
print("step(full) - native", np.max(np.abs(b3 - a1)), "step(full)-step(sym)", np.max(np.abs(b3 - b1)))
# one smoother application both ways
lvl = h.levels[0]
sm = lvl.smoother
bb = D.f64(v)
S._symop = s._jac._st.symop
x1 = D.host(sm.apply(lvl.matvec, None, bb))
S._symop = None
x2 = D.host(sm.apply(lvl.matvec, None, bb))
print("smoother sym vs full", np.max(np.abs(x1 - x2)), np.max(np.abs(x1)))
S._symop = None
plan_full = MG._NativePlan(h.levels)
c1 = D.host(plan_full.apply(D.f64(v)))
print("native(full)-native(sym)", np.max(np.abs(c1 - a1)), "native(full)-step(full)", np.max(np.abs(c1 - b3)),
      "native(full)-step(sym)", np.max(np.abs(c1 - b1)))
S._symop = s._jac._st.symop
rng = np.random.default_rng(7)
n = S.shape[0]
xx, bb2 = D.f64(rng.normal(size=n)), D.f64(rng.normal(size=n))
Dinv = sm.jacobi.inverse_blocks()
d0 = D.f64(rng.normal(size=n))
outs = {}
for nm in ("sym", "full"):
    d = d0.clone(); o = D.empty(n)
    if nm == "sym":
        D.call("bamg_symop_cheb_step", S._symop.handle, S.blocks, xx, bb2, Dinv, d, o, 0.3, 0.7, 0)
    else:
        D.call("bamg_cheb_step", 9, S._ptr, S._col, S.blocks, xx, bb2, Dinv, d, o, S.n_block_rows, 0.3, 0.7, 0)
    outs[nm] = (D.host(o), D.host(d))
    rr = D.empty(n)
    if nm == "sym":
        D.call("bamg_symop_residual", S._symop.handle, S.blocks, xx, bb2, rr)
    else:
        D.call("bamg_bsr_residual", 9, S._ptr, S._col, S.blocks, xx, bb2, rr, S.n_block_rows)
    outs[nm + "r"] = D.host(rr)
Sd = np.zeros((n, n)); ptr = D.host(S._ptr); col = D.host(S._col); blk = D.host(S.blocks)
for i in range(S.n_block_rows):
    for q in range(ptr[i], ptr[i+1]):
        Sd[9*i:9*i+9, 9*col[q]:9*col[q]+9] = blk[q]
r = D.host(bb2) - Sd @ D.host(xx)
Di = D.host(Dinv)
z = np.concatenate([Di[i] @ r[9*i:9*i+9] for i in range(S.n_block_rows)])
dn = 0.3 * D.host(d0) + 0.7 * z
ref = D.host(xx) + dn
for nm in ("sym", "full"):
    print(nm, "cheb err", np.max(np.abs(outs[nm][0] - ref)) / np.max(np.abs(ref)), "resid err",
          np.max(np.abs(outs[nm + "r"] - r)) / np.max(np.abs(r)))
print("cond S", np.linalg.cond(Sd))
