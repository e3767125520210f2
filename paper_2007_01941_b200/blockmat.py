"""Device block-sparse containers (drop-in for `bamg.blockmat`, blockmat.py:1-372).

* `BlockSparseMatrix` -- BSR with int32 device row pointers / sorted column
  indices and row-major fp64 blocks; `matvec` runs the sm_100a BSR kernels.
* `BlockDiagMatrix` -- stacked square blocks with a cached batched Cholesky and
  explicit inverse (blockmat.py:95-129), computed by one kernel.
* `DenseTall` -- a dense (rows, cols) device matrix (near-nullspace bases).

Attributes that are numpy arrays in the reference are CUDA tensors here (`indptr`
and `indices` are int64 views of the int32 device arrays).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D


class IndefiniteBlockError(Exception):
    """A diagonal block was not positive definite (blockmat.py:25-39)."""

    def __init__(self, block_index: int, context: str = ""):
        self.block_index = int(block_index)
        msg = f"block {block_index} is not positive definite"
        if context:
            msg += f" ({context})"
        super().__init__(msg)


class DenseTall:
    """Dense rows-by-columns matrix; houses near-nullspace bases (blockmat.py:42-59)."""

    def __init__(self, data):
        self.data = D.f64(data)
        if self.data.dim() != 2:
            raise ValueError(f"DenseTall expects a 2-D array, got ndim={self.data.dim()}")

    @property
    def rows(self) -> int:
        return self.data.shape[0]

    @property
    def cols(self) -> int:
        return self.data.shape[1]


class BlockDiagMatrix:
    """Square block-diagonal matrix as a stacked (n, bs, bs) array (blockmat.py:62-149)."""

    def __init__(self, blocks, _inv=None):
        self.blocks = D.f64(blocks)
        if self.blocks.dim() != 3 or self.blocks.shape[1] != self.blocks.shape[2]:
            raise ValueError(f"expected (n, bs, bs) blocks, got {tuple(self.blocks.shape)}")
        self._chol = None
        self._inv = _inv

    @property
    def n_blocks(self) -> int:
        return self.blocks.shape[0]

    @property
    def block_size(self) -> int:
        return self.blocks.shape[1]

    @property
    def shape(self):
        n = self.n_blocks * self.block_size
        return (n, n)

    def nnz_scalar(self) -> int:
        return self.n_blocks * self.block_size**2

    def _apply(self, M, x):
        x = D.f64(x).reshape(-1)
        y = D.empty(x.numel())
        D.call("bamg_blockdiag_apply", M, x, self.n_blocks, self.block_size, y)
        return y

    def matvec(self, x):
        return self._apply(self.blocks, x)

    def factor(self) -> "BlockDiagMatrix":
        """Batched Cholesky + explicit inverse; IndefiniteBlockError on the first bad block."""
        if self._inv is None:
            n, bs = self.n_blocks, self.block_size
            L = D.empty(n, bs, bs)
            inv = D.empty(n, bs, bs)
            bad = D.empty(1, dtype=torch.int32)
            D.call("bamg_block_chol_inv", self.blocks, n, bs, L, inv, bad)
            b = int(bad.item())
            if b != 0x7FFFFFFF:
                raise IndefiniteBlockError(b)
            self._chol, self._inv = L, inv
        return self

    def _factor_deferred(self):
        """factor() without the readback: returns the device slot holding the first
        failing block (0x7FFFFFFF = none); the caller checks it at its next readback."""
        n, bs = self.n_blocks, self.block_size
        L = D.empty(n, bs, bs)
        inv = D.empty(n, bs, bs)
        bad = D.empty(1, dtype=torch.int32)
        D.call("bamg_block_chol_inv", self.blocks, n, bs, L, inv, bad)
        self._chol, self._inv = L, inv
        return bad

    @property
    def factored(self) -> bool:
        return self._inv is not None

    def solve(self, x):
        self.factor()
        return self._apply(self._inv, x)

    def inverse_blocks(self):
        self.factor()
        return self._inv

    def to_dense(self):
        return torch.block_diag(*self.blocks) if self.n_blocks else D.zeros(0, 0)

    def to_block_sparse(self) -> "BlockSparseMatrix":
        n = self.n_blocks
        idx = torch.arange(n, device=D.dev(), dtype=torch.int32)
        ptr = torch.arange(n + 1, device=D.dev(), dtype=torch.int32)
        return BlockSparseMatrix(n, n, self.block_size, self.block_size, ptr, idx, self.blocks.clone())


class SymmetricPattern:
    """Half-storage view of an exactly symmetric 9x9 block pattern (`bamg_symop`).

    The explicit S is stored in full, but its solve-phase products stream only the
    upper blocks and rebuild the lower half from their transposes. Built once per
    observation structure from the Schur symbolic phase's upper-block list (diagonal
    slots, block positions, mirror positions); shared by every S of that structure.
    """

    def __init__(self, ptr, col, dpos, up_blk, up_tpos, n_up: int, nbr: int, _handle=None):
        from . import _lib

        self._keep = (ptr, col, dpos)
        self.nbr = int(nbr)
        if _handle is None:
            _handle = _lib.lib().bamg_symop_create(
                self.nbr, ptr.data_ptr(), col.data_ptr(), dpos.data_ptr(), up_blk.data_ptr(), up_tpos.data_ptr(),
                int(n_up), int(col.numel()), D.stream())
        self.handle = _handle
        if not self.handle:
            raise _lib.NativeError(f"bamg_symop_create: {_lib.last_error()}")
        self.nch = int(_lib.lib().bamg_symop_chunks(self.handle))

    @classmethod
    def from_pattern(cls, ptr, col, nbr: int, bs: int) -> "SymmetricPattern":
        """View of any exactly symmetric BSR pattern (diagonal slots and mirror map
        derived on the device), e.g. a Galerkin coarse operator (bs 16)."""
        from . import _lib

        h = _lib.lib().bamg_symop_create_pattern(int(bs), int(nbr), ptr.data_ptr(), col.data_ptr(),
                                                 int(col.numel()), D.stream())
        return cls(ptr, col, None, None, None, 0, nbr, _handle=h)

    def matches(self, m: "BlockSparseMatrix") -> bool:
        return m._ptr is self._keep[0] and m._col is self._keep[1]

    def __del__(self):
        try:
            from . import _lib

            _lib.lib().bamg_symop_destroy(self.handle)
        except Exception:
            pass


class BlockSparseMatrix:
    """Block-CSR matrix with uniform dense blocks (blockmat.py:152-335)."""

    def __init__(self, n_block_rows, n_block_cols, row_block_size, col_block_size, indptr, indices, blocks,
                 _validate=True):
        self.n_block_rows = int(n_block_rows)
        self.n_block_cols = int(n_block_cols)
        self.row_block_size = int(row_block_size)
        self.col_block_size = int(col_block_size)
        self._ptr = D.i32(indptr)
        self._col = D.i32(indices)
        self.blocks = D.f64(blocks)
        self._prolongator = None  # (agg_ptr, members) when this is a tentative P
        self._T = None
        self._symop = None  # SymmetricPattern when the blocks are exactly symmetric (explicit S)
        if _validate:
            if self._ptr.shape != (self.n_block_rows + 1,):
                raise ValueError(f"indptr has length {self._ptr.shape[0]}, expected {self.n_block_rows + 1}")
            nnz = self._col.numel()
            last = int(self._ptr[-1].item())
            if last != nnz:
                raise ValueError(f"indptr[-1]={last} but {nnz} indices stored")
            expect = (nnz, self.row_block_size, self.col_block_size)
            if tuple(self.blocks.shape) != expect:
                raise ValueError(f"blocks shaped {tuple(self.blocks.shape)}, expected {expect}")

    @property
    def indptr(self):
        return self._ptr.to(torch.int64)

    @property
    def indices(self):
        return self._col.to(torch.int64)

    @property
    def n_block_entries(self) -> int:
        return int(self._col.numel())

    @property
    def shape(self):
        return (self.n_block_rows * self.row_block_size, self.n_block_cols * self.col_block_size)

    def nnz_scalar(self) -> int:
        return self.n_block_entries * self.row_block_size * self.col_block_size

    def block_rows_expanded(self):
        return torch.repeat_interleave(torch.arange(self.n_block_rows, device=D.dev()),
                                       (self._ptr[1:] - self._ptr[:-1]).to(torch.int64))

    def diagonal_blocks(self):
        if self.row_block_size != self.col_block_size:
            raise ValueError("diagonal blocks need square blocks")
        if self.n_block_rows != self.n_block_cols:
            raise ValueError("diagonal blocks need a square matrix")
        bs = self.row_block_size
        out = D.empty(self.n_block_rows, bs, bs)
        D.call("bamg_diag_blocks", self._ptr, self._col, self.blocks, self.n_block_rows, bs, out)
        return out

    # -- kernels -------------------------------------------------------------------

    def matvec(self, x):
        x = D.f64(x).reshape(-1)
        if x.numel() != self.shape[1]:
            raise ValueError(f"matvec got vector of length {x.numel()}, need {self.shape[1]}")
        if self._prolongator is not None:
            y = D.empty(self.shape[0])
            D.call("bamg_prolong", self._col, self.blocks, x, self.n_block_rows, self.row_block_size, y, 0)
            return y
        bs = self.row_block_size
        if self._symop is not None:
            y = D.empty(self.shape[0])
            D.call("bamg_symop_spmv", self._symop.handle, self.blocks, x, y, None)
            return y
        if bs == self.col_block_size and bs in (1, 3, 9, 16):
            y = D.empty(self.shape[0])
            D.call("bamg_bsr_spmv", bs, self._ptr, self._col, self.blocks, x, y, self.n_block_rows, None)
            return y
        return self._rect_matvec(self, x)

    @staticmethod
    def _rect_matvec(m, x):
        # rectangular blocks (API views of W and of transposes): per-block products
        # gathered in row order -- not on the measured path.
        rows = m.block_rows_expanded()
        xb = x.reshape(m.n_block_cols, m.col_block_size)[m._col.to(torch.int64)]
        prod = torch.einsum("nij,nj->ni", m.blocks, xb)
        y = D.zeros(m.n_block_rows, m.row_block_size)
        y.index_add_(0, rows, prod)
        return y.reshape(-1)

    def rmatvec(self, x):
        x = D.f64(x).reshape(-1)
        if x.numel() != self.shape[0]:
            raise ValueError(f"rmatvec got vector of length {x.numel()}, need {self.shape[0]}")
        if self._prolongator is not None:
            agg_ptr, members = self._prolongator
            y = D.empty(self.shape[1])
            D.call("bamg_restrict", agg_ptr, members, self.blocks, x, self.n_block_cols, self.row_block_size, y)
            return y
        if self._T is None:
            self._T = self.transpose()
        return self._T.matvec(x)

    def transpose(self) -> "BlockSparseMatrix":
        rows = self.block_rows_expanded()
        return BlockSparseMatrix.from_triplets(self.n_block_cols, self.n_block_rows, self._col.to(torch.int64),
                                               rows, self.blocks.transpose(1, 2))

    def to_dense(self):
        n, m = self.shape
        out = D.zeros(self.n_block_rows, self.row_block_size, self.n_block_cols, self.col_block_size)
        if self.n_block_entries:
            rows = self.block_rows_expanded()
            out[rows, :, self._col.to(torch.int64), :] = self.blocks
        return out.reshape(n, m)

    def scale_block_columns(self, col_blocks) -> "BlockSparseMatrix":
        col_blocks = D.f64(col_blocks)
        if col_blocks.shape[0] != self.n_block_cols or col_blocks.shape[1] != self.col_block_size:
            raise ValueError("column block array does not match matrix")
        nb = torch.einsum("nij,njk->nik", self.blocks, col_blocks[self._col.to(torch.int64)])
        return BlockSparseMatrix(self.n_block_rows, self.n_block_cols, self.row_block_size, col_blocks.shape[2],
                                 self._ptr.clone(), self._col.clone(), nb)

    @staticmethod
    def from_triplets(n_block_rows, n_block_cols, rows, cols, blocks) -> "BlockSparseMatrix":
        """Assemble from (row, col, block) triplets; duplicates are summed (blockmat.py:195-230)."""
        rows = torch.as_tensor(rows, device=D.dev()).to(torch.int64).reshape(-1)
        cols = torch.as_tensor(cols, device=D.dev()).to(torch.int64).reshape(-1)
        blocks = D.f64(blocks)
        if blocks.dim() != 3 or not (blocks.shape[0] == rows.numel() == cols.numel()):
            raise ValueError("triplet arrays disagree on entry count")
        rbs, cbs = blocks.shape[1], blocks.shape[2]
        if rows.numel() == 0:
            return BlockSparseMatrix(n_block_rows, n_block_cols, rbs, cbs,
                                     torch.zeros(n_block_rows + 1, dtype=torch.int32), torch.zeros(0),
                                     D.zeros(0, rbs, cbs))
        key = rows * max(int(n_block_cols), 1) + cols
        order = torch.sort(key, stable=True).indices
        key, blocks = key[order], blocks[order]
        first = torch.ones_like(key, dtype=torch.bool)
        first[1:] = key[1:] != key[:-1]
        seg = torch.cumsum(first.to(torch.int64), 0) - 1
        nseg = int(seg[-1].item()) + 1
        summed = D.zeros(nseg, rbs, cbs)
        summed.index_add_(0, seg, blocks)
        ukey = key[first]
        urow, ucol = ukey // max(int(n_block_cols), 1), ukey % max(int(n_block_cols), 1)
        counts = torch.bincount(urow, minlength=n_block_rows)
        ptr = torch.zeros(n_block_rows + 1, dtype=torch.int64, device=D.dev())
        ptr[1:] = torch.cumsum(counts, 0)
        return BlockSparseMatrix(n_block_rows, n_block_cols, rbs, cbs, ptr, ucol, summed)


def multiply(a: BlockSparseMatrix, b: BlockSparseMatrix) -> BlockSparseMatrix:
    """Sparse block product a @ b (blockmat.py:337-353) -- API convenience via dense
    row panels; the measured path uses the dedicated Galerkin / Schur kernels."""
    if a.n_block_cols != b.n_block_rows or a.col_block_size != b.row_block_size:
        raise ValueError("block product mismatch")
    dense = a.to_dense() @ b.to_dense()
    rbs, cbs = a.row_block_size, b.col_block_size
    blk = dense.reshape(a.n_block_rows, rbs, b.n_block_cols, cbs).permute(0, 2, 1, 3)
    nz = (blk != 0).flatten(2).any(-1)
    r, c = torch.nonzero(nz, as_tuple=True)
    return BlockSparseMatrix.from_triplets(a.n_block_rows, b.n_block_cols, r, c, blk[r, c])


def triple_product(r, a, p):
    return multiply(multiply(r, a), p)


def write_matrix_market(mat, path) -> None:
    """MatrixMarket coordinate file of the scalar entries (blockmat.py:363-372)."""
    if isinstance(mat, BlockDiagMatrix):
        mat = mat.to_block_sparse()
    dense = D.host(mat.to_dense())
    r, c = np.nonzero(dense)
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{dense.shape[0]} {dense.shape[1]} {len(r)}\n")
        for i, j in zip(r, c):
            fh.write(f"{i + 1} {j + 1} {dense[i, j]:.17g}\n")
