"""Parameter-independent observation structure on the GPU (problem.py ObsStructure):
the point-major / camera-major orders, the covisibility pattern, the shared-point
counts and the Schur pair lists, checked bit-exactly against a numpy restatement of
their definitions (schur.py:128-144 via blockmat.py:217-230: W's block order is
(camera, point); S_ij sums over the points cameras i and j share, in point order)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P

    return P


def H(t):
    from paper_2007_01941_b200 import _device

    return _device.host(t)


def expected_structure(ci, pi, nc, npt):
    ci = np.asarray(ci, dtype=np.int64)
    pi = np.asarray(pi, dtype=np.int64)
    pm = np.lexsort((ci, pi))  # point-major, cameras ascending inside a point
    cam_pm, pt_pm = ci[pm], pi[pm]
    pt_ptr = np.concatenate([[0], np.cumsum(np.bincount(pt_pm, minlength=npt))])
    cm = np.lexsort((np.arange(len(pm)), cam_pm))  # point-major positions by camera
    cam_ptr = np.concatenate([[0], np.cumsum(np.bincount(cam_pm, minlength=nc))])
    # every pair of observations of one point, a < b (cameras ascending)
    m = np.diff(pt_ptr)
    pa, pb = [], []
    for d in range(1, int(m.max()) if len(m) else 1):
        seg = np.repeat(np.arange(npt), np.maximum(m - d, 0))
        start = pt_ptr[:-1][seg]
        off = np.arange(len(seg)) - np.repeat(np.cumsum(np.maximum(m - d, 0)) - np.maximum(m - d, 0),
                                              np.maximum(m - d, 0))
        pa.append(start + off)
        pb.append(start + off + d)
    pa = np.concatenate(pa) if pa else np.zeros(0, np.int64)
    pb = np.concatenate(pb) if pb else np.zeros(0, np.int64)
    # covisibility rows (diagonal included), sorted
    keys = np.unique(np.concatenate([cam_pm[pa] * nc + cam_pm[pb], cam_pm[pb] * nc + cam_pm[pa],
                                     np.arange(nc) * nc + np.arange(nc)]))
    S_ptr = np.concatenate([[0], np.cumsum(np.bincount(keys // nc, minlength=nc))])
    S_col = keys % nc
    # block slot of every pair; inside a block, point order (= first observation order)
    slot = np.searchsorted(keys, cam_pm[pa] * nc + cam_pm[pb])
    order = np.lexsort((pa, slot))
    blk_ptr = np.concatenate([[0], np.cumsum(np.bincount(slot, minlength=len(keys)))])
    return dict(pm=pm, cam_pm=cam_pm, pt_pm=pt_pm, pt_ptr=pt_ptr, cm=cm, cam_ptr=cam_ptr, S_ptr=S_ptr, S_col=S_col,
                pair_a=pa[order], pair_b=pb[order], blk_ptr=blk_ptr)


def _scene(name):
    from paper_2007_01941_b200 import scenes

    if name == "street":
        return scenes.street(n_points=15_000)
    if name == "large":
        return scenes.large(n_clusters=1, n_points=60_000, threads=4)
    return scenes.random_problem(1003, n_cameras=12, n_points=60)


@pytest.mark.parametrize("name", ["small", "street", "large"])
def test_structure_matches_definition(P, name):
    sc = _scene(name)
    cams, pts, ci, pi, pix = sc.arrays()
    ex = expected_structure(ci, pi, len(cams), len(pts))
    prob = P.BundleProblem(cams, pts, ci, pi, pix)
    st = prob._st
    np.testing.assert_array_equal(H(st.pm_perm), ex["pm"])
    np.testing.assert_array_equal(H(st.obs_cam_pm), ex["cam_pm"])
    np.testing.assert_array_equal(H(st.obs_pt_pm), ex["pt_pm"])
    np.testing.assert_array_equal(H(st.pt_ptr), ex["pt_ptr"])
    np.testing.assert_array_equal(H(st.cm_list), ex["cm"])
    np.testing.assert_array_equal(H(st.cam_ptr), ex["cam_ptr"])
    S_ptr, S_col, nnz, _ = st.covis
    np.testing.assert_array_equal(H(S_ptr), ex["S_ptr"])
    np.testing.assert_array_equal(H(S_col), ex["S_col"])
    # shared-point counts: off-diagonal = block list lengths, diagonal = camera degree
    shared = H(st.strength["shared"]).astype(np.int64)
    sym_len = np.diff(ex["blk_ptr"])
    rows = np.repeat(np.arange(len(cams)), np.diff(ex["S_ptr"]))
    cols = ex["S_col"]
    up = cols > rows
    np.testing.assert_array_equal(shared[up], sym_len[up])
    diag = cols == rows
    np.testing.assert_array_equal(shared[diag], np.diff(ex["cam_ptr"]))
    nc = len(cams)
    lo = cols < rows  # (i, j), j < i: the count of slot (j, i)
    tpos = np.searchsorted(rows * nc + cols, cols[lo] * nc + rows[lo])
    np.testing.assert_array_equal(shared[lo], sym_len[tpos])

    p = st.pair_lists
    n = p["n_pairs"]
    assert n == len(ex["pair_a"])
    np.testing.assert_array_equal(H(p["blk_ptr"]), ex["blk_ptr"])
    np.testing.assert_array_equal(H(p["pair_a"])[:n], ex["pair_a"])
    np.testing.assert_array_equal(H(p["pair_b"])[:n], ex["pair_b"])
    # shared counts read off the pair lists (the eager structure path) = the sweep's
    from paper_2007_01941_b200 import _device as D

    cnt = D.empty(max(nnz, 1), dtype=st.cam_ptr.dtype)
    D.call("bamg_shared_from_pairs", p["up_blk"], p["up_tpos"], p["n_up"], p["blk_ptr"], p["dpos"], st.cam_ptr, nc,
           cnt)
    np.testing.assert_array_equal(H(cnt)[:nnz], shared)
