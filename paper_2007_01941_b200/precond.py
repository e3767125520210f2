"""Point-block-Jacobi preconditioner on the device (drop-in for `bamg.precond`, precond.py:24-56).

The visibility block-Jacobi comparator (precond.py:59-144) is outside the
north-star path and is not provided by this package.
"""

from __future__ import annotations

import torch

from . import _device as D
from .blockmat import BlockDiagMatrix, IndefiniteBlockError
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
    D.call("bamg_schur_numeric", st.cam_ptr, st.cm_list, sys._jac._J, sys.A.blocks, dpos, nc,
           None, None, 0, None, None, None, out)
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
