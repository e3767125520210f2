"""Damped normal equations and the reduced camera system on the device.

Drop-in for `bamg.schur` (`pkg/src/bamg/schur.py:1-188`). The point blocks are
eliminated per point (C^-1 by a batched 3x3 Cholesky), the explicit S is
assembled by the deterministic pair-list kernels of csrc/schur.cu, and the
implicit operator A x - W C^-1 W^T x runs as two segmented kernels. W is never
stored: every W block is F^T E of one observation; `SchurSystem.W` materialises
the reference-shaped BSR view on demand.
"""

from __future__ import annotations

import weakref

import torch

from . import _device as D
from .blockmat import BlockDiagMatrix, BlockSparseMatrix, IndefiniteBlockError
from .problem import CAMERA_SIZE, POINT_SIZE, JacobianBlocks

_DIAG_MIN = 1e-6  # schur.py:21
_DIAG_MAX = 1e32  # schur.py:22


class Damping:
    """Additive diagonal scaled by the trust radius (schur.py:25-55).

    The camera half is formed lazily: the explicit assembly's camera-major pass
    produces it alongside S_ii (no separate pass over the records); reading
    ``cam_diag`` before that runs a diagonal-only camera pass."""

    def __init__(self, radius, cam_diag, pt_diag, jac=None):
        self.radius = radius
        self._cam = cam_diag
        self.pt_diag = pt_diag
        self._jac = jac

    @property
    def cam_diag(self):
        if self._cam is None:
            jac, st = self._jac, self._jac._st
            dc = D.empty(jac.n_cameras, CAMERA_SIZE)
            D.call("bamg_camera_pass", st.cam_ptr, st.cm_list, jac._J, None, jac.n_cameras, float(self.radius), None,
                   None, None, dc, None)
            self._cam = dc
        return self._cam

    @cam_diag.setter
    def cam_diag(self, value):
        self._cam = value

    @staticmethod
    def from_jacobian(jac: JacobianBlocks, radius: float) -> "Damping":
        if not radius > 0:
            raise ValueError(f"trust radius must be positive, got {radius}")
        C, _ = jac.point_normal()
        dp = D.empty(jac.n_points, POINT_SIZE)
        D.call("bamg_damping", None, C, 0, jac.n_points, float(radius), None, dp)
        return Damping(radius, None, dp, jac)

    @staticmethod
    def zero(n_cameras: int, n_points: int) -> "Damping":
        return Damping(float("inf"), D.zeros(n_cameras, CAMERA_SIZE), D.zeros(n_points, POINT_SIZE))


class SchurSystem:
    """Block factors after point elimination (schur.py:58-96)."""

    def __init__(self, A, C, rhs_cam, grad_pt, jac, Cb, mode="implicit", damping=None):
        self._A = A  # None: A_raw + D formed on first use (the explicit path never needs it)
        self._damping = damping
        self.C = C
        self._rhs = rhs_cam  # None: formed on first use, or by the explicit assembly's diagonal pass
        self.grad_pt = grad_pt
        self.mode = mode
        self.S_explicit = None
        self._jac = jac
        self._Cb = Cb
        self._W = None
        self._qo = None

    @property
    def rhs_cam(self):
        """Reduced right-hand side b_c - W C^-1 b_p (schur.py:122). build_system defers
        it: the explicit assembly forms it in its camera-major diagonal pass (one
        sweep over the records instead of two); otherwise the standalone gather runs
        at first use."""
        if self._rhs is None:
            st = self._jac._st
            self._own_H()
            rhs = D.empty(self.n_cameras * CAMERA_SIZE)
            _, gc, _, _ = self._jac.normal_blocks()
            D.call("bamg_rhs_gather", st.cam_ptr, st.cm_list, self._jac._J, self._qo, gc, self.n_cameras, rhs)
            self._rhs = rhs
        return self._rhs

    @rhs_cam.setter
    def rhs_cam(self, value):
        self._rhs = value

    @property
    def A(self) -> BlockDiagMatrix:
        if self._A is None:
            A_raw, _, _, _ = self._jac.normal_blocks()
            A = D.empty(self.n_cameras, CAMERA_SIZE, CAMERA_SIZE)
            D.call("bamg_add_block_diag", A_raw, self._damping.cam_diag, self.n_cameras, CAMERA_SIZE, A)
            self._A = BlockDiagMatrix(A)
        return self._A

    @A.setter
    def A(self, value):
        self._A = value

    @property
    def n_cameras(self) -> int:
        return self._jac.n_cameras

    @property
    def n_points(self) -> int:
        return self.C.n_blocks

    @property
    def W(self) -> BlockSparseMatrix:
        """Reference-shaped coupling matrix (nc x np, 9x3 blocks, (cam, pt) order)."""
        if self._W is None:
            st = self._jac._st
            k = st.k
            blocks = D.empty(k, CAMERA_SIZE, POINT_SIZE)
            if k:
                D.call("bamg_materialize_W", st.cm_list, self._jac._J, k, blocks)
            cols = st.obs_pt_pm[st.cm_list.to(torch.int64)]
            self._W = BlockSparseMatrix(self.n_cameras, self.n_points, CAMERA_SIZE, POINT_SIZE, st.cam_ptr, cols,
                                        blocks)
        return self._W

    def implicit_matvec(self, x):
        """S x without materialising S: A x - W (C^-1 (W^T x)) (schur.py:84-86)."""
        x = D.f64(x).reshape(-1)
        st = self._jac._st
        if self._qo is None:
            self._qo = D.empty(max(st.k, 1), 2)
        y = D.empty(self.n_cameras * CAMERA_SIZE)
        D.call("bamg_implicit_matvec", st.cam_ptr, st.cm_list, st.pt_ptr, st.obs_cam_pm, self._jac._J,
               self.A.blocks, self.C._inv, x, self.n_cameras, self.n_points, self._qo, y)
        return y

    def matvec(self, x):
        if self.mode == "explicit":
            return self.ensure_explicit().matvec(x)
        return self.implicit_matvec(x)

    def _own_H(self):
        """Make the Jacobian's H slots (E C^-1) those of THIS system: another system
        built from the same Jacobian (e.g. a rejected LM trial re-damped) overwrites them."""
        owner = self._jac._h_owner() if self._jac._h_owner is not None else None
        if owner is not self:
            st = self._jac._st
            if self._qo is None:
                self._qo = D.empty(max(st.k, 1), 2)
            D.call("bamg_obs_H", st.obs_pt_pm, self.C._inv, self._Cb, st.k, self._jac._J, self._qo)
            self._jac._h_owner = weakref.ref(self)

    def ensure_explicit(self) -> BlockSparseMatrix:
        if self.S_explicit is None:
            self.S_explicit = schur_explicit(self, _VARIANT)
        return self.S_explicit


def build_system(jac: JacobianBlocks, damping: Damping) -> SchurSystem:
    """Assemble A, C (factored), rhs and the point gradient (schur.py:99-125)."""
    npt = jac.n_points
    st = jac._st
    C_raw, gp = jac.point_normal()
    C = D.empty(npt, 3, 3)
    Cinv = D.empty(npt, 3, 3)
    Cb = D.empty(npt, 3)
    qo = D.empty(max(st.k, 1), 2)
    bad = D.empty(1, dtype=torch.int32)
    # point half only: the damped camera blocks A are formed on demand (SchurSystem.A)
    D.call("bamg_build_system", st.cam_ptr, st.cm_list, st.pt_ptr, jac._J, st.k, None, C_raw, None, gp,
           None, damping.pt_diag, 0, npt, None, C, Cinv, Cb, qo, None, bad)
    b = int(bad.item())
    if b != 0x7FFFFFFF:
        raise IndefiniteBlockError(b)
    grad_pt = D.empty(npt * POINT_SIZE)
    D.call("bamg_negate", gp, grad_pt, npt * POINT_SIZE)
    Cm = BlockDiagMatrix(C, _inv=Cinv)
    s = SchurSystem(None, Cm, None, grad_pt, jac, Cb, damping=damping)
    s._qo = qo
    jac._h_owner = weakref.ref(s)  # weak: no jac <-> system reference cycle
    return s


def schur_explicit(sys: SchurSystem, variant: str = "pairs") -> BlockSparseMatrix:
    """S = A - W C^-1 W^T as a 9x9 BSR over the covisibility pattern (schur.py:128-144).

    ``variant`` "pairs" (default): block-owned accumulation over per-block
    point-pair lists (built once per problem); "rows": row-owned shared-memory
    accumulation. Both are deterministic; they differ only in summation order.
    """
    st = sys._jac._st
    S_ptr, S_col, nnz, _ = st.covis
    blocks = D.empty(nnz, CAMERA_SIZE, CAMERA_SIZE)
    J = sys._jac
    sys._own_H()
    # a materialised A is authoritative (the caller may have changed it): then the
    # assembly's own diagonal pass runs on it
    fused = sys._damping is not None and sys._A is None and variant in ("chunks", "pairs")
    if fused:  # diagonal blocks, right-hand side and camera damping in one camera-major pass
        _camera_pass(sys, st.pair_lists["dpos"] if variant == "pairs" else st.chunk_plan["dpos"], blocks)
    nc_diag = 0 if fused else sys.n_cameras  # otherwise the assembly's own diagonal pass (needs A)
    if variant == "chunks":
        ch = st.chunk_plan
        rhs = None
        gc = None
        if not fused:
            _, gc, _, _ = J.normal_blocks()
            if sys._rhs is None:
                rhs = D.empty(sys.n_cameras * CAMERA_SIZE)
        D.call("bamg_schur_numeric_chunked", st.cam_ptr, st.cm_list, J._J, None if fused else sys.A.blocks,
               ch["dpos"], nc_diag, ch["work"], ch["n_work"], ch["pair_a"], ch["pair_b"], ch["done"], nnz, sys._qo,
               gc, rhs, blocks)
        if rhs is not None:
            sys._rhs = rhs
    elif variant == "rows":
        sym = st.symbolic
        D.call("bamg_schur_numeric_rows", st.cam_ptr, st.cm_list, st.pt_ptr, st.obs_cam_pm, st.obs_pt_pm, J._J,
               sys.A.blocks, S_ptr, S_col, sym["dpos"], sym["up_off"], sym["up_tpos"], sys.n_cameras, blocks)
    else:  # off-diagonal blocks from the per-block pair lists
        sym = st.pair_lists
        rhs = None
        gc = None
        if not fused:
            _, gc, _, _ = J.normal_blocks()
            if sys._rhs is None:
                rhs = D.empty(sys.n_cameras * CAMERA_SIZE)
        D.call("bamg_schur_numeric", st.cam_ptr, st.cm_list, J._J, None if fused else sys.A.blocks, sym["dpos"],
               nc_diag, sym["up_blk"], sym["up_tpos"], sym["n_up"], sym["blk_ptr"], sym["pair_a"], sym["pair_b"],
               sys._qo, gc, rhs, blocks)
        if rhs is not None:
            sys._rhs = rhs
    S = BlockSparseMatrix(sys.n_cameras, sys.n_cameras, CAMERA_SIZE, CAMERA_SIZE, S_ptr, S_col, blocks,
                          _validate=False)
    if _SYMMETRIC:
        S._symop = st.symop  # S_ji == S_ij^T bit for bit: half-storage products
    return S


def _camera_pass(sys: SchurSystem, dpos, blocks):
    """Diagonal blocks S_ii, the right-hand side and (if still pending) the camera
    damping in one camera-major pass over the records (bamg_camera_pass)."""
    st, J, dmp = sys._jac._st, sys._jac, sys._damping
    rhs = D.empty(sys.n_cameras * CAMERA_SIZE) if sys._rhs is None else None
    dc = D.empty(sys.n_cameras, CAMERA_SIZE) if dmp is not None and dmp._cam is None else None
    D.call("bamg_camera_pass", st.cam_ptr, st.cm_list, J._J, sys._qo, sys.n_cameras, float(dmp.radius), dpos, blocks,
           rhs, dc, None)
    if rhs is not None:
        sys._rhs = rhs
    if dc is not None:
        dmp._cam = dc


_SYMMETRIC = __import__("os").environ.get("BAMG_SYM_SPMV", "1") == "1"
_VARIANT = __import__("os").environ.get("BAMG_SCHUR", "pairs")  # A/B: pairs | rows


def covisibility_block_count(sys: SchurSystem) -> int:
    """Camera-pair blocks S would store, with the reference's int8 pattern-product
    wrap (schur.py:147-159): pairs sharing a multiple of 256 points are not counted."""
    if sys.S_explicit is not None:
        return sys.S_explicit.n_block_entries
    return sys._jac._st.strength["wrapped"]


def choose_mode(sys: SchurSystem) -> str:
    """Cheaper matvec route by stored-entry flop count; ties explicit (schur.py:162-168)."""
    explicit_cost = 2 * covisibility_block_count(sys) * CAMERA_SIZE**2
    a_nnz = sys.n_cameras * CAMERA_SIZE**2  # sys.A.nnz_scalar() without forming A
    implicit_cost = 2 * (a_nnz + 2 * sys._jac._st.k * CAMERA_SIZE * POINT_SIZE + sys.C.nnz_scalar())
    return "explicit" if explicit_cost <= implicit_cost else "implicit"


def back_substitute(sys: SchurSystem, delta_cam):
    """Point update C^-1 (grad_pt - W^T dc) (schur.py:171-173)."""
    st = sys._jac._st
    dc = D.f64(delta_cam).reshape(-1)
    dp = D.empty(sys.n_points * POINT_SIZE)
    D.call("bamg_back_substitute", st.pt_ptr, st.obs_cam_pm, sys._jac._J, sys.C._inv, sys.grad_pt,
           dc, sys.n_cameras, sys.n_points, dp)
    return dp


def model_decrease(sys: SchurSystem, delta_cam) -> float:
    """Predicted decrease of the half-objective quadratic model (schur.py:176-188)."""
    dc = D.f64(delta_cam).reshape(-1)
    s_dc = sys.matvec(dc)
    a = D.dot(sys.rhs_cam, dc)
    b = D.dot(dc, s_dc)
    # grad_pt^T C^-1 grad_pt = sum_p b_p . (C^-1 b_p), Cb = C^-1 b_p from build_system
    c = D.dot(sys.grad_pt, sys._Cb.reshape(-1))
    return float(a - 0.5 * b + 0.5 * c)
