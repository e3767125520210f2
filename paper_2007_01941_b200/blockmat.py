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

import ctypes

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
            expect = (nnz, self.row_block_size, self.col_block_size)
            if tuple(self.blocks.shape) != expect:
                raise ValueError(f"blocks shaped {tuple(self.blocks.shape)}, expected {expect}")
            # one readback: indptr[-1], nondecreasing indptr, column range (blockmat.py:174-191)
            chk = D.empty(3, dtype=torch.int32)
            D.call("bamg_bsr_validate", self._ptr, self.n_block_rows, self._col, nnz, self.n_block_cols, chk)
            chk[2:3].copy_(self._ptr[-1:])
            bad_ptr, bad_col, last = chk.tolist()
            if last != nnz:
                raise ValueError(f"indptr[-1]={last} but {nnz} indices stored")
            if bad_ptr:
                raise ValueError("indptr must be nondecreasing")
            if bad_col:
                raise ValueError("block column index out of range")

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
        # any block shape (API views of W, transposes, user matrices): scipy
        # bsr_matvec summation order, so the result equals the reference bit for bit
        y = D.empty(m.shape[0])
        if m.shape[0]:
            D.call("bamg_bsr_matvec_gen", m.row_block_size, m.col_block_size, m._ptr, m._col, m.blocks, x,
                   m.n_block_rows, y)
        return y

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
        """Right-multiply by a block-diagonal matrix given as (n, cbs, k) blocks (blockmat.py:321-334)."""
        col_blocks = D.f64(col_blocks)
        if col_blocks.shape[0] != self.n_block_cols or col_blocks.shape[1] != self.col_block_size:
            raise ValueError("column block array does not match matrix")
        k = col_blocks.shape[2]
        nb = D.empty(self.n_block_entries, self.row_block_size, k)
        D.call("bamg_bsr_scale_cols", self.blocks, col_blocks, self._col, self.n_block_entries, self.row_block_size,
               self.col_block_size, k, nb)
        return BlockSparseMatrix(self.n_block_rows, self.n_block_cols, self.row_block_size, k,
                                 self._ptr.clone(), self._col.clone(), nb, _validate=False)

    @staticmethod
    def from_triplets(n_block_rows, n_block_cols, rows, cols, blocks) -> "BlockSparseMatrix":
        """Assemble from (row, col, block) triplets; duplicates are summed (blockmat.py:195-230).

        Stable (row, col) order and sequential duplicate sums in input order, as
        np.lexsort + np.add.reduceat: bit-identical to the reference."""
        rows = torch.as_tensor(rows, device=D.dev()).to(torch.int64).reshape(-1).contiguous()
        cols = torch.as_tensor(cols, device=D.dev()).to(torch.int64).reshape(-1).contiguous()
        blocks = D.f64(blocks)
        if blocks.dim() != 3 or not (blocks.shape[0] == rows.numel() == cols.numel()):
            raise ValueError("triplet arrays disagree on entry count")
        rbs, cbs = blocks.shape[1], blocks.shape[2]
        n = rows.numel()
        nbr, nbc = int(n_block_rows), int(n_block_cols)
        if n == 0:
            return BlockSparseMatrix(nbr, nbc, rbs, cbs, torch.zeros(nbr + 1, dtype=torch.int32),
                                     torch.zeros(0, dtype=torch.int32), D.zeros(0, rbs, cbs), _validate=False)
        perm = D.empty(n, dtype=torch.int32)
        seg = D.empty(n, dtype=torch.int32)
        cnt = D.empty(2, dtype=torch.int32)
        D.call("bamg_triplets_order", rows, cols, n, nbr, nbc, perm, seg, cnt)
        nu, bad = cnt.tolist()
        if bad:
            raise ValueError("block column index out of range")
        ptr = D.empty(nbr + 1, dtype=torch.int32)
        col = D.empty(max(nu, 1), dtype=torch.int32)
        out = D.empty(max(nu, 1), rbs, cbs)
        D.call("bamg_triplets_reduce", rows, cols, blocks.contiguous(), n, rbs * cbs, perm, seg, nu, nbr, ptr, col,
               out)
        return BlockSparseMatrix(nbr, nbc, rbs, cbs, ptr, col[:nu], out[:nu], _validate=False)


def multiply(a: BlockSparseMatrix, b: BlockSparseMatrix) -> BlockSparseMatrix:
    """Sparse block product a @ b (blockmat.py:337-353): block SpGEMM on the device in
    scipy csr_matmat's summation order, with its zero-drop (a block is kept iff one
    of its scalars is nonzero)."""
    from . import _lib

    if a.n_block_cols != b.n_block_rows or a.col_block_size != b.row_block_size:
        raise ValueError(
            f"block product mismatch: ({a.n_block_rows}x{a.n_block_cols} of {a.row_block_size}x{a.col_block_size})"
            f" @ ({b.n_block_rows}x{b.n_block_cols} of {b.row_block_size}x{b.col_block_size})")
    rbs, kbs, cbs = a.row_block_size, a.col_block_size, b.col_block_size
    nbr, nbc = a.n_block_rows, b.n_block_cols
    L = _lib.lib()
    s = D.stream()
    nu = ctypes.c_int64(0)
    h = L.bamg_spgemm_create(D.ctx(s), a._ptr.data_ptr(), a._col.data_ptr(), nbr, a.n_block_entries,
                             b._ptr.data_ptr(), b._col.data_ptr(), nbc, ctypes.byref(nu), s)
    if not h:
        raise _lib.NativeError(f"bamg_spgemm_create: {_lib.last_error()}")
    try:
        nk = ctypes.c_int64(0)
        _lib.call("bamg_spgemm_numeric", D.ctx(s), h, a.blocks, rbs, kbs, b.blocks, cbs, ctypes.byref(nk), s)
        nkeep = nk.value
        ptr = D.empty(nbr + 1, dtype=torch.int32)
        col = D.empty(max(nkeep, 1), dtype=torch.int32)
        out = D.empty(max(nkeep, 1), rbs, cbs)
        _lib.call("bamg_spgemm_finish", D.ctx(s), h, ptr, col, out, s)
        torch.cuda.current_stream().synchronize()  # before the handle's buffers are freed
    finally:
        L.bamg_spgemm_destroy(h)
    return BlockSparseMatrix(nbr, nbc, rbs, cbs, ptr, col[:nkeep], out[:nkeep], _validate=False)


def triple_product(r, a, p):
    """r @ a @ p as two successive sparse products (blockmat.py:356-360)."""
    return multiply(multiply(r, a), p)


def write_matrix_market(mat, path) -> None:
    """MatrixMarket coordinate file of the stored scalar entries (blockmat.py:363-372):
    every scalar of every stored block (explicit zeros included), blocks in storage
    order and row-major inside a block -- the order of scipy's bsr.tocoo()."""
    if isinstance(mat, BlockDiagMatrix):
        mat = mat.to_block_sparse()
    ptr, col, blk = D.host(mat.indptr), D.host(mat.indices), D.host(mat.blocks)
    R, C = mat.row_block_size, mat.col_block_size
    nnz = len(col)
    brow = np.repeat(np.arange(mat.n_block_rows, dtype=np.int64), np.diff(ptr))
    row = np.repeat(R * brow, R * C) + np.tile(np.repeat(np.arange(R), C), nnz)
    cols = np.repeat(C * col, R * C) + np.tile(np.arange(C), R * nnz)
    data = blk.reshape(-1)
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{mat.shape[0]} {mat.shape[1]} {len(data)}\n")
        fh.writelines(f"{i + 1} {j + 1} {v:.17g}\n" for i, j, v in zip(row.tolist(), cols.tolist(), data.tolist()))
