"""Block-Jacobi preconditioners on the device (drop-in for `bamg.precond`, precond.py:1-144).

* Point block Jacobi (precond.py:24-56): inverses of the 9x9 diagonal blocks of S.
* Visibility block Jacobi (precond.py:59-144, the paper's second comparator):
  dense principal submatrices of S, one per cluster of covisible cameras found by
  the same greedy aggregation as the multigrid hierarchy with a cap of 100; factored
  and inverted by batched tiled kernels, applied as one batched gather-GEMV.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .blockmat import BlockDiagMatrix, IndefiniteBlockError
from .multigrid import Aggregation, StrengthMatrix, aggregate
from .problem import CAMERA_SIZE
from .schur import SchurSystem

DEFAULT_CLUSTER_CAP = 100


class PointBlockJacobi:
    def __init__(self, blocks: BlockDiagMatrix):
        self.blocks = blocks

    def apply(self, r):
        return self.blocks.solve(r)


def _schur_diagonal_blocks(sys: SchurSystem):
    """Diagonal 9x9 blocks of S without forming S (precond.py:24-31): the diagonal
    kernel of the explicit assembly run alone."""
    st = sys._jac._st
    nc = sys.n_cameras
    out = D.empty(nc, CAMERA_SIZE, CAMERA_SIZE)
    dpos = torch.arange(nc, device=D.dev(), dtype=torch.int32)
    sys._own_H()
    if sys._damping is not None and sys._A is None:  # one camera-major pass: S_ii, rhs, damping
        # (a materialised A is authoritative: the caller may have changed it)
        from .schur import _camera_pass

        _camera_pass(sys, dpos, out)
        return out
    D.call("bamg_schur_numeric", st.cam_ptr, st.cm_list, sys._jac._J, sys.A.blocks, dpos, nc,
           None, None, 0, None, None, None, None, None, None, out)
    return out


def pbj_setup(sys: SchurSystem) -> PointBlockJacobi:
    """Factor the true diagonal blocks of S (precond.py:42-56)."""
    if sys.S_explicit is not None:
        blocks = sys.S_explicit.diagonal_blocks()
    else:
        blocks = _schur_diagonal_blocks(sys)
    try:
        return PointBlockJacobi(BlockDiagMatrix(blocks).factor())
    except IndefiniteBlockError as e:
        raise IndefiniteBlockError(e.block_index, "insufficient damping") from None


def visibility_cluster(strength: StrengthMatrix, max_cluster: int = DEFAULT_CLUSTER_CAP) -> Aggregation:
    """Cluster cameras by visibility strength, capped at ``max_cluster`` (precond.py:59-62)."""
    return aggregate(strength, max_size=max_cluster)


class VisibilityJacobi:
    """Per-cluster inverses of principal submatrices of S (precond.py:65-78).

    ``apply`` is one batched kernel: for each cluster, gather the members' residual
    slots, multiply by the cluster's explicit inverse, scatter.
    """

    def __init__(self, clusters: Aggregation, cptr, mem, dims_host, offs_host, factor, inv):
        from . import _lib

        self.clusters = clusters
        self._cptr, self._mem = cptr, mem
        self._dims_host, self._offs_host = dims_host, offs_host
        self._dims = D.i32(torch.as_tensor(dims_host, dtype=torch.int32))
        self._offs = torch.as_tensor(offs_host, dtype=torch.int64).to(D.dev())
        self._L, self._inv = factor, inv
        self.dim_max = int(dims_host.max()) if len(dims_host) else 0
        self.handle = _lib.lib().bamg_vj_create(len(dims_host), self.dim_max, self._offs.data_ptr(),
                                                self._dims.data_ptr(), cptr.data_ptr(), mem.data_ptr(),
                                                inv.data_ptr())

    @property
    def members(self):
        return self.clusters.members()

    @property
    def factors(self):
        """Lower Cholesky factor of each cluster's submatrix (the reference keeps cho_factor tuples)."""
        out = []
        for n, o in zip(self._dims_host, self._offs_host):
            out.append(torch.tril(self._L[int(o):int(o) + int(n) * int(n)].view(int(n), int(n))))
        return out

    def apply(self, r):
        r = D.f64(r).reshape(-1)
        z = D.empty(r.numel())
        D.call("bamg_vj_apply", self.handle, r, z)
        return z

    def __del__(self):
        try:
            from . import _lib

            _lib.lib().bamg_vj_destroy(self.handle)
        except Exception:
            pass


def vj_setup(sys: SchurSystem, clusters: Aggregation) -> VisibilityJacobi:
    """Assemble, factor and invert each cluster's principal submatrix of S (precond.py:82-144).

    Blocks come from the assembled S when present; otherwise S is assembled by the
    same deterministic Schur kernels (the reference accumulates the in-cluster
    point contributions from A, W and C directly -- the same sums, another order).
    """
    nc = sys.n_cameras
    if clusters._a32.numel() != nc:
        raise ValueError(f"partition covers {clusters._a32.numel()} cameras, system has {nc}")
    from .schur import schur_explicit

    S = sys.S_explicit if sys.S_explicit is not None else schur_explicit(sys)
    cptr, mem = clusters.member_lists()
    sizes = np.diff(D.host(cptr)).astype(np.int64)
    dims = CAMERA_SIZE * sizes
    sq = dims * dims
    offs = np.concatenate([[0], np.cumsum(sq)[:-1]]).astype(np.int64)
    total = int(sq.sum())
    ncl = clusters.n_aggregates
    vj_dims = D.i32(torch.as_tensor(dims, dtype=torch.int32))
    vj_offs = torch.as_tensor(offs, dtype=torch.int64).to(D.dev())
    work = D.empty(max(total, 1))
    D.call("bamg_vj_assemble", S._ptr, S._col, S.blocks, nc, clusters._a32, cptr, mem, vj_offs, vj_dims, work,
           total)
    tmp = D.empty(max(total, 1))
    inv = D.empty(max(total, 1))
    flags = D.empty(max(ncl, 1), dtype=torch.int32)
    D.call("bamg_vj_factor", ncl, int(dims.max()) if ncl else 0, vj_offs, vj_dims, work, tmp, inv, flags)
    bad = np.flatnonzero(D.host(flags)[:ncl])
    if bad.size:
        raise IndefiniteBlockError(int(bad[0]), "visibility cluster not positive definite")
    del tmp
    return VisibilityJacobi(clusters, cptr, mem, dims, offs, work, inv)
