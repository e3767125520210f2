"""Level-0 S product timings at a config (dev tool): full-storage BSR SpMV vs the
symmetric half-storage pair (CUDA events, 50 reps after warm-up)."""

import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2007_01941_b200 as P  # noqa: E402
from paper_2007_01941_b200 import _device as D  # noqa: E402


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
    return e0.elapsed_time(e1) / reps


def main(config=4):
    sc = bench.scene_for(int(config))
    prob = P.BundleProblem(*sc.arrays())
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    S = s.ensure_explicit()
    n = S.shape[0]
    x = D.f64(torch.randn(n, dtype=torch.float64))
    y = D.empty(n)
    nnz = S.n_block_entries
    full = timeit(lambda: D.call("bamg_bsr_spmv", 9, S._ptr, S._col, S.blocks, x, y, S.n_block_rows, None))
    sym = timeit(lambda: D.call("bamg_symop_spmv", S._symop.handle, S.blocks, x, y, None))
    dot = D.empty(1)
    two = timeit(lambda: D.call("bamg_symop_spmv", S._symop.handle, S.blocks, x, y, dot))
    B = nnz * (8 * 81 + 4) + 4 * (S.n_block_rows + 1) + 16 * n
    print(f"nnzb={nnz} full {full*1e3:.1f} us ({B/full/1e6:.0f} GB/s)  sym {sym*1e3:.1f} us "
          f"(effective {B/sym/1e6:.0f} GB/s)  two-pass+dot {two*1e3:.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
