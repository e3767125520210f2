"""Bundle-adjustment problem on the device: structure, residuals, Jacobians, gauge.

Drop-in for `bamg.problem` (`pkg/src/bamg/problem.py`). Names, argument meaning and
error behaviour follow the reference; array-valued results are CUDA tensors
(float64 / int64) instead of numpy arrays -- inputs may be either. Observations
keep the caller's order at the API (`cam_index`, `pt_index`, `pixels`,
`JacobianBlocks.camera` ...); internally they are stored point-major (sorted by
(point, camera)) with a camera-major index list, see DESIGN.md.
"""

from __future__ import annotations

import warnings

import numpy as np
import torch

from . import _device as D
from .blockmat import DenseTall

CAMERA_SIZE = 9
POINT_SIZE = 3
_MIN_DEPTH = 1e-12  # problem.py:25


class BehindCameraError(Exception):
    """One or more observations project from behind the camera plane (problem.py:28-36)."""

    def __init__(self, observation_indices):
        self.observation_indices = np.atleast_1d(np.asarray(observation_indices, dtype=int))
        n = len(self.observation_indices)
        head = ", ".join(str(i) for i in self.observation_indices[:8])
        more = ", ..." if n > 8 else ""
        super().__init__(f"{n} observation(s) behind camera: [{head}{more}]")


# -- loss (problem.py:179-196), elementwise on tensors ---------------------------


def huber(s):
    s = torch.as_tensor(s, dtype=torch.float64)
    return torch.where(s <= 1.0, s, 2.0 * torch.sqrt(torch.clamp(s, min=1.0)) - 1.0)


def loss_value(s, kind: str):
    if kind == "trivial":
        return torch.as_tensor(s, dtype=torch.float64)
    return huber(s)


def loss_weight(s, kind: str):
    s = torch.as_tensor(s, dtype=torch.float64)
    if kind == "trivial":
        return torch.ones_like(s)
    return torch.where(s <= 1.0, torch.ones_like(s), torch.clamp(s, min=1.0) ** -0.25)


# -- observation structure --------------------------------------------------------


class ObsStructure:
    """Parameter-independent device layout of the observations.

    Built once per problem (the reference recomputes nothing structural either:
    `solver.py:221-230`). Holds the point-major order, the camera-major list, the
    covisibility (S) pattern, the visibility strength graph and the Schur pair lists.
    """

    def __init__(self, cam_index: torch.Tensor, pt_index: torch.Tensor, nc: int, npt: int,
                 pixels: torch.Tensor, pix_ready=None):
        k = int(cam_index.numel())
        self.k, self.nc, self.npt = k, nc, npt
        i32 = torch.int32
        self.pm_perm = D.empty(k, dtype=i32)
        self.obs_cam_pm = D.empty(k, dtype=i32)
        self.obs_pt_pm = D.empty(k, dtype=i32)
        self.pt_ptr = D.empty(npt + 1, dtype=i32)
        self.cm_list = D.empty(k, dtype=i32)
        self.cam_ptr = D.empty(nc + 1, dtype=i32)
        D.call("bamg_obs_orders", cam_index, pt_index, k, nc, npt, self.pm_perm, self.obs_cam_pm,
               self.obs_pt_pm, self.pt_ptr, self.cm_list, self.cam_ptr)
        # the point-major pixels are gathered on first use (evaluate): a pixel copy
        # still running on the copy stream then overlaps the structural passes
        # (covisibility, strength, pair lists) instead of stalling them
        self._pixels, self._pix_ready_ev, self._pix_pm = pixels, pix_ready, None
        self._covis = None
        self._strength = None
        self._symbolic = None
        self._wcache = None

    @property
    def pix_pm(self) -> torch.Tensor:
        if self._pix_pm is None:
            pm = D.empty(self.k, 2)
            if self._pix_ready_ev is not None:  # the pixel copy ran on a copy stream
                torch.cuda.current_stream().wait_event(self._pix_ready_ev)
            if self.k:
                D.call("bamg_gather_rows_f64", self._pixels, self.pm_perm, self.k, 2, pm)
            self._pix_pm, self._pixels = pm, None
        return self._pix_pm

    # point-major array (k, ...) -> caller order
    def to_input_order(self, a: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(a)
        if self.k:
            width = int(a[0].numel()) if a.dim() > 1 else 1
            D.call("bamg_scatter_rows_f64", a.reshape(self.k, -1), self.pm_perm, self.k, width,
                   out.reshape(self.k, -1))
        return out

    @property
    def covis(self):
        """(S_ptr, S_col, nnz, max_row): covisibility incl. the diagonal, sorted."""
        if self._covis is None:
            counts = D.empty(self.nc + 1, dtype=torch.int32)
            words = (self.nc + 31) // 32
            keep = self.nc * words * 4 <= _COVIS_KEEP_BYTES
            bm = D.empty(max(self.nc * words, 1), dtype=torch.int32) if keep else None
            if keep:  # the fill then compacts these bitmaps instead of sweeping the observations again
                D.call("bamg_covis_count_keep", self.cam_ptr, self.cm_list, self.obs_pt_pm, self.pt_ptr,
                       self.obs_cam_pm, self.nc, counts, bm)
            else:
                D.call("bamg_covis_count", self.cam_ptr, self.cm_list, self.obs_pt_pm, self.pt_ptr,
                       self.obs_cam_pm, self.nc, counts)
            max_row = int(counts[: self.nc].max().item()) if self.nc else 0
            total = D.empty(1, dtype=torch.int32)
            D.call("bamg_scan_exclusive_i32", counts, counts, self.nc + 1, total)
            nnz = int(counts[self.nc].item())
            S_col = D.empty(max(nnz, 1), dtype=torch.int32)
            if keep:
                D.call("bamg_covis_compact", bm, self.nc, counts, S_col)
                del bm
            else:
                D.call("bamg_covis_fill", self.cam_ptr, self.cm_list, self.obs_pt_pm, self.pt_ptr,
                       self.obs_cam_pm, self.nc, counts, S_col)
            self._covis = (counts, S_col[:nnz], nnz, max_row)
        return self._covis

    @property
    def strength(self):
        """Visibility strength CSR (multigrid.py:52-80) plus bookkeeping."""
        if self._strength is None:
            S_ptr, S_col, nnz, max_row = self.covis
            cnt = D.empty(max(nnz, 1), dtype=torch.int32)
            pl = getattr(self, "_pairs", None)
            if pl is not None:  # list lengths: no sweep of the observations
                D.call("bamg_shared_from_pairs", pl["up_blk"], pl["up_tpos"], pl["n_up"], pl["blk_ptr"], pl["dpos"],
                       self.cam_ptr, self.nc, cnt)
            else:
                D.call("bamg_shared_counts", self.cam_ptr, self.cm_list, self.obs_pt_pm, self.pt_ptr,
                       self.obs_cam_pm, self.nc, S_ptr, S_col, max_row, cnt)
            deg = D.empty(self.nc, dtype=torch.int32)
            G_ptr = D.empty(self.nc + 1, dtype=torch.int32)
            ng = nnz - self.nc
            G_col = D.empty(max(ng, 1), dtype=torch.int32)
            G_val = D.empty(max(ng, 1))
            flags = D.empty(2, dtype=torch.int32)
            D.call("bamg_visibility_strength", self.cam_ptr, S_ptr, S_col, cnt, self.nc, deg, G_ptr,
                   G_col, G_val, flags)
            f = flags.cpu().numpy()
            self._strength = dict(G_ptr=G_ptr, G_col=G_col[:ng], G_val=G_val[:ng], deg=deg,
                                  n_empty=int(f[0]), wrapped=int(f[1]), shared=cnt[:nnz])
        return self._strength

    def _schur_symbolic(self, with_pairs: bool):
        S_ptr, S_col, nnz, _ = self.covis
        pair_off = D.empty(max(self.npt, 1), dtype=torch.int32)
        dpos = D.empty(max(self.nc, 1), dtype=torch.int32)
        up_off = D.empty(max(self.nc, 1), dtype=torch.int32)
        sizes = np.zeros(2, dtype=np.int64)
        D.call("bamg_schur_symbolic_sizes", self.pt_ptr, S_ptr, S_col, self.nc, self.npt,
               pair_off, dpos, up_off, sizes.ctypes.data)
        n_pairs, n_up = int(sizes[0]), int(sizes[1])
        up_blk = D.empty(max(n_up, 1), dtype=torch.int32)
        up_row = D.empty(max(n_up, 1), dtype=torch.int32)
        up_tpos = D.empty(max(n_up, 1), dtype=torch.int32)
        out = dict(up_blk=up_blk, up_row=up_row, up_tpos=up_tpos, dpos=dpos, up_off=up_off, n_up=n_up,
                   n_pairs=n_pairs)
        if with_pairs:
            out["pair_a"] = D.empty(max(n_pairs, 1), dtype=torch.int32)
            out["pair_b"] = D.empty(max(n_pairs, 1), dtype=torch.int32)
            out["blk_ptr"] = D.empty(nnz + 1, dtype=torch.int32)
        D.call("bamg_schur_symbolic", self.pt_ptr, self.obs_cam_pm, self.obs_pt_pm, S_ptr, S_col, self.nc, self.npt,
               nnz, pair_off, n_pairs, dpos, up_off, out.get("pair_a"), out.get("pair_b"), out.get("blk_ptr"),
               up_blk, up_row, up_tpos)
        return out

    @property
    def symbolic(self):
        """Upper-triangle block list of S: diagonal slots, per-row offsets, transposed
        positions (schur.cu, row-owned numeric assembly)."""
        if self._symbolic is None:
            self._symbolic = self._schur_symbolic(False)
        return self._symbolic

    @property
    def symop(self):
        """Half-storage view of S's pattern for the solve-phase products (blockmat.SymmetricPattern)."""
        if getattr(self, "_symop", None) is None:
            from .blockmat import SymmetricPattern

            S_ptr, S_col, nnz, _ = self.covis
            p = getattr(self, "_pairs", None) or self.symbolic
            self._symop = SymmetricPattern(S_ptr, S_col, p["dpos"], p["up_blk"], p["up_tpos"], p["n_up"], self.nc)
        return self._symop

    @property
    def chunk_plan(self):
        """Point-chunk phased pair lists (schur.cu, bamg_schur_chunk_*): pairs sorted by
        (chunk, S block), one work item per (chunk, block) segment."""
        if getattr(self, "_chunks", None) is None:
            S_ptr, S_col, nnz, _ = self.covis
            sym = getattr(self, "_pairs", None) or self.symbolic
            pair_off = D.empty(max(self.npt, 1), dtype=torch.int32)
            dpos = D.empty(max(self.nc, 1), dtype=torch.int32)
            up_off = D.empty(max(self.nc, 1), dtype=torch.int32)
            sizes = np.zeros(4, dtype=np.int64)
            D.call("bamg_schur_symbolic_sizes", self.pt_ptr, S_ptr, S_col, self.nc, self.npt,
                   pair_off, dpos, up_off, sizes.ctypes.data)
            n_pairs = int(sizes[0])
            pair_a = D.empty(max(n_pairs, 1), dtype=torch.int32)
            pair_b = D.empty(max(n_pairs, 1), dtype=torch.int32)
            skey = D.empty(max(n_pairs, 1), dtype=torch.int32)
            D.call("bamg_schur_chunk_pairs", self.pt_ptr, self.obs_cam_pm, S_ptr, S_col, self.nc, self.npt, nnz,
                   self.k, pair_off, n_pairs, _CHUNK_RECORDS, pair_a, pair_b, skey, sizes.ctypes.data)
            n_seg, n_chunks, blk_bits = int(sizes[0]), int(sizes[1]), int(sizes[2])
            cap = n_seg + 10 * n_chunks
            work = D.empty(max(cap, 1), 4, dtype=torch.int32)
            out = np.zeros(1, dtype=np.int64)
            D.call("bamg_schur_chunk_work", S_ptr, S_col, self.nc, skey, n_pairs, n_seg, n_chunks, blk_bits,
                   _CHUNK_GROUP_ROWS, work, cap, out.ctypes.data)
            del skey
            self._chunks = dict(pair_a=pair_a, pair_b=pair_b, work=work, n_work=int(out[0]), n_seg=n_seg,
                                n_chunks=n_chunks, dpos=sym["dpos"], done=D.empty(max(nnz, 1), dtype=torch.int32))
        return self._chunks

    @property
    def pair_lists(self):
        """Per-block point-pair lists (the block-owned alternative assembly)."""
        if getattr(self, "_pairs", None) is None:
            p = self._schur_symbolic(True)
            D.call("bamg_schur_order_upper", p["up_blk"], p["up_row"], p["up_tpos"], p["n_up"], p["blk_ptr"],
                   p["pair_a"])
            self._pairs = p
        return self._pairs


# -- problem ----------------------------------------------------------------------


def _pinned(x) -> bool:
    return isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned()


_COPY_STREAMS = {}


def _copy_stream():
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = torch.cuda.Stream()
    return _COPY_STREAMS[dev]


_EAGER_STRUCTURE = __import__("os").environ.get("BAMG_EAGER_STRUCTURE", "1") == "1"
_COVIS_KEEP_BYTES = 256 << 20  # row bitmaps kept between the covisibility count and fill passes
_CHUNK_RECORDS = int(__import__("os").environ.get("BAMG_SCHUR_CHUNK", "150000"))  # observations per point chunk
_CHUNK_GROUP_ROWS = int(__import__("os").environ.get("BAMG_SCHUR_CHUNK_ROWS", "1"))


class BundleProblem:
    """Cameras, points and pixel observations (problem.py:81-173), device resident."""

    def __init__(self, camera_params, points, cam_index, pt_index, pixels, loss: str = "trivial",
                 _structure: ObsStructure | None = None):
        cams = D.f64(camera_params).clone()
        pinned = (_structure is None and _pinned(points) and _pinned(cam_index) and _pinned(pt_index)
                  and _pinned(pixels))
        if pinned:
            # pinned host inputs: the index copies go first on the current stream (the
            # orders sort needs them); points and pixels follow on a copy stream, and
            # every consumer waits on `_pix_ready` (points / pixels properties, the
            # point-major pixel gather in front of evaluate)
            ci = cam_index.to(D.dev(), non_blocking=True).to(torch.int64).reshape(-1)
            pi = pt_index.to(D.dev(), non_blocking=True).to(torch.int64).reshape(-1)
            main = torch.cuda.current_stream()
            cs = _copy_stream()
            cs.wait_stream(main)
            with torch.cuda.stream(cs):
                pts = points.to(D.dev(), dtype=torch.float64, non_blocking=True)
                pix = pixels.to(D.dev(), dtype=torch.float64, non_blocking=True).reshape(-1, 2)
            pts.record_stream(main)
            pix.record_stream(main)
            self._pix_ready = torch.cuda.Event()
            self._pix_ready.record(cs)
        else:
            pts = D.f64(points).clone()
        if cams.dim() != 2 or cams.shape[1] != CAMERA_SIZE:
            raise ValueError(f"camera_params must be (n, 9), got {tuple(cams.shape)}")
        if pts.dim() != 2 or pts.shape[1] != POINT_SIZE:
            raise ValueError(f"points must be (m, 3), got {tuple(pts.shape)}")
        if loss not in ("trivial", "huber"):
            raise ValueError(f"unknown loss {loss!r}")
        self.loss = loss
        self._cams, self._pts = cams, pts
        if cams.shape[0]:
            D.call("bamg_canonicalize", self._cams, cams.shape[0], CAMERA_SIZE)  # problem.py:106
        if _structure is not None:
            self._ci, self._pi, self._pix, self._st = _structure._ci, _structure._pi, _structure._pix, _structure
            return
        if pinned:
            pass  # copies issued above
        else:
            ci = torch.as_tensor(cam_index, device=D.dev()).to(torch.int64).reshape(-1)
            pi = torch.as_tensor(pt_index, device=D.dev()).to(torch.int64).reshape(-1)
            pix = D.f64(pixels).reshape(-1, 2) if np.size(pixels) else D.empty(0, 2)
            self._pix_ready = None
        if not (ci.numel() == pi.numel() == pix.shape[0]):
            raise ValueError("observation arrays disagree on length")
        k, nc, npt = ci.numel(), cams.shape[0], pts.shape[0]
        if k:
            lo_hi = torch.stack([ci.min(), ci.max(), pi.min(), pi.max()]).cpu().numpy()
            if lo_hi[0] < 0 or lo_hi[1] >= nc:
                raise ValueError("camera index out of range")
            if lo_hi[2] < 0 or lo_hi[3] >= npt:
                raise ValueError("point index out of range")
        st = ObsStructure(ci.to(torch.int32), pi.to(torch.int32), nc, npt, pix, self._pix_ready)
        st._ci, st._pi, st._pix = ci, pi, pix
        if k > 1:
            dup = ((st.obs_pt_pm[1:] == st.obs_pt_pm[:-1]) & (st.obs_cam_pm[1:] == st.obs_cam_pm[:-1])).any()
            if bool(dup.item()):
                raise ValueError("duplicate (camera, point) observation")
        cam_cnt = (st.cam_ptr[1:] - st.cam_ptr[:-1]) if nc else st.cam_ptr[:0]
        pt_cnt = (st.pt_ptr[1:] - st.pt_ptr[:-1]) if npt else st.pt_ptr[:0]
        n_empty = int((cam_cnt < 1).sum().item()) if nc else 0
        n_weak = int((pt_cnt < 2).sum().item()) if npt else 0
        if n_empty:
            warnings.warn(f"{n_empty} camera(s) observe no points", stacklevel=2)
        if n_weak:
            warnings.warn(f"{n_weak} point(s) observed by fewer than 2 cameras", stacklevel=2)
        self._ci, self._pi, self._pix, self._st = ci, pi, pix, st
        if self._pix_ready is not None and k and nc > 1 and not n_empty and _EAGER_STRUCTURE:
            # pinned inputs: the pixel upload is still running on the copy stream, so
            # the parameter-independent passes every linear solve needs anyway run now,
            # in its shadow -- covisibility, visibility strength, the level-0
            # aggregation scan (side stream) and the Schur pair lists
            from . import multigrid

            st.pair_lists  # first: the strength pass then reads the shared counts off its lists
            G = multigrid.visibility_strength(self)
            multigrid._aggregate_prefetch(G, 20)

    # -- reference attributes (device tensors, caller order) --
    @property
    def camera_params(self) -> torch.Tensor:
        return self._cams

    @property
    def points(self) -> torch.Tensor:
        ev = getattr(self, "_pix_ready", None)
        if ev is not None:  # pinned inputs: the copy-stream upload must be complete
            torch.cuda.current_stream().wait_event(ev)
        return self._pts

    @property
    def cam_index(self) -> torch.Tensor:
        return self._ci

    @property
    def pt_index(self) -> torch.Tensor:
        return self._pi

    @property
    def pixels(self) -> torch.Tensor:
        ev = getattr(self, "_pix_ready", None)
        if ev is not None:  # the copy-stream upload must be complete for the caller's stream
            torch.cuda.current_stream().wait_event(ev)
        return self._pix

    @property
    def structure(self) -> ObsStructure:
        return self._st

    @property
    def n_cameras(self) -> int:
        return self._cams.shape[0]

    @property
    def n_points(self) -> int:
        return self._pts.shape[0]

    @property
    def n_observations(self) -> int:
        return int(self._ci.numel())

    def copy(self) -> "BundleProblem":
        return BundleProblem(self._cams, self.points, None, None, None, self.loss, _structure=self._st)

    def with_params(self, camera_params, points) -> "BundleProblem":
        return BundleProblem(camera_params, points, None, None, None, self.loss, _structure=self._st)

    def __eq__(self, other) -> bool:
        if not isinstance(other, BundleProblem):
            return NotImplemented
        return (self.loss == other.loss and self._cams.shape == other._cams.shape
                and self._pts.shape == other._pts.shape
                and bool(torch.equal(self._cams, other._cams)) and bool(torch.equal(self.points, other.points))
                and bool(torch.equal(self._ci, other._ci)) and bool(torch.equal(self._pi, other._pi))
                and bool(torch.equal(self.pixels, other.pixels)))


# -- Jacobian blocks --------------------------------------------------------------


class JacobianBlocks:
    """Loss-weighted residuals and Jacobian blocks (problem.py:237-269).

    Device storage is point-major, one 256-byte record per observation
    ``_J[o] = [F (2x9) | E (2x3) | H (2x3) | r (2)]`` (H = E C^-1 is written by
    `build_system`); ``camera``/``point``/``residual``/``weight`` give
    caller-order tensors (k,2,9)/(k,2,3)/(k,2)/(k,). The per-camera and per-point
    reductions (J^T J blocks, gradient, diagonal) are computed once by one
    deterministic kernel pass and shared by `gradient`, `normal_diagonal`,
    `Damping.from_jacobian` and `build_system`.
    """

    REC = 32

    def __init__(self, camera, point, residual, weight, cam_index, pt_index, n_cameras, n_points):
        """Reference constructor (problem.py:237-253): caller-order blocks, e.g. a
        fabricated Jacobian; packed here into the device record layout."""
        ci = torch.as_tensor(cam_index, device=D.dev()).to(torch.int64).reshape(-1)
        pi = torch.as_tensor(pt_index, device=D.dev()).to(torch.int64).reshape(-1)
        k = ci.numel()
        st = ObsStructure(ci.to(torch.int32), pi.to(torch.int32), int(n_cameras), int(n_points), D.zeros(k, 2))
        J = D.zeros(max(k, 1), self.REC)[:k]
        if k:
            for a, lo, hi in ((camera, 0, 18), (point, 18, 24), (residual, 30, 32)):
                src = D.f64(a).reshape(k, hi - lo)
                tmp = D.empty(k, hi - lo)
                D.call("bamg_gather_rows_f64", src, st.pm_perm, k, hi - lo, tmp)
                J[:, lo:hi] = tmp
        w = D.empty(k)
        if k:
            D.call("bamg_gather_rows_f64", D.f64(weight).reshape(k, 1), st.pm_perm, k, 1, w.reshape(k, 1))
        self._init(st, J, w, int(n_cameras), int(n_points), ci, pi)

    @classmethod
    def _from_records(cls, st, J, w, n_cameras, n_points, cam_index, pt_index):
        obj = cls.__new__(cls)
        obj._init(st, J, w, n_cameras, n_points, cam_index, pt_index)
        return obj

    def _init(self, st: ObsStructure, J, w, n_cameras, n_points, cam_index, pt_index):
        self._st = st
        self._J, self._w = J, w
        self.n_cameras, self.n_points = n_cameras, n_points
        self.cam_index, self.pt_index = cam_index, pt_index
        self._normal = None
        self._pnormal = None
        self._h_owner = None  # weakref to the SchurSystem whose C^-1 produced the H slots

    @property
    def camera(self):
        return self._st.to_input_order(self._J[:, 0:18].contiguous()).reshape(-1, 2, CAMERA_SIZE)

    @property
    def point(self):
        return self._st.to_input_order(self._J[:, 18:24].contiguous()).reshape(-1, 2, POINT_SIZE)

    @property
    def residual(self):
        return self._st.to_input_order(self._J[:, 30:32].contiguous()).reshape(-1, 2)

    @property
    def weight(self):
        return self._st.to_input_order(self._w.reshape(-1, 1)).reshape(-1)

    def point_normal(self):
        """(C_raw (np,3,3), g_pt (np,3)): the point half of normal_blocks (point-major pass)."""
        if self._pnormal is None:
            npt = self.n_points
            C = D.empty(npt, 3, 3)
            gp = D.empty(npt, 3)
            st = self._st
            D.call("bamg_normal_blocks", st.cam_ptr, st.cm_list, st.pt_ptr, self._J, 0, npt, None, None, C, gp)
            self._pnormal = (C, gp)
        return self._pnormal

    def normal_blocks(self):
        """(A_raw (nc,9,9), g_cam (nc,9), C_raw (np,3,3), g_pt (np,3)) -- undamped. The
        linear solve does not need the camera blocks themselves (its camera-major pass
        forms D, S_ii and the right-hand side directly); they are formed here on demand."""
        if self._normal is None:
            nc = self.n_cameras
            A = D.empty(nc, 9, 9)
            gc = D.empty(nc, 9)
            C, gp = self.point_normal()
            st = self._st
            D.call("bamg_normal_blocks", st.cam_ptr, st.cm_list, st.pt_ptr, self._J, nc, 0, A, gc, None, None)
            self._normal = (A, gc, C, gp)
        return self._normal

    def gradient(self):
        """Gradient of half the objective: (per-camera (n,9), per-point (m,3))."""
        _, gc, _, gp = self.normal_blocks()
        return gc, gp

    def normal_diagonal(self):
        """Diagonal of J^T J: (per-camera (n,9), per-point (m,3))."""
        A, _, C, _ = self.normal_blocks()
        return torch.diagonal(A, dim1=1, dim2=2), torch.diagonal(C, dim1=1, dim2=2)


def _params(problem: BundleProblem, camera_params, points):
    cams = problem._cams if camera_params is None else D.f64(camera_params).reshape(-1, CAMERA_SIZE)
    pts = problem._pts if points is None else D.f64(points).reshape(-1, POINT_SIZE)
    return cams, pts


def evaluate(problem: BundleProblem, camera_params=None, points=None, with_jacobian: bool = True):
    """Objective and (optionally) Jacobian blocks (problem.py:272-326).

    Raises BehindCameraError with ascending caller-order indices when any
    observation has z >= -1e-12 in its camera frame.
    """
    cams, pts = _params(problem, camera_params, points)
    st = problem._st
    k = st.k
    huber = 1 if problem.loss == "huber" else 0
    # objective (f64) and behind-camera count (i32) share one 16 B buffer: one readback
    res = D.empty(2)
    obj = res[:1]
    nb = res[1:].view(torch.int32)[:1]
    behind = D.empty(max(k, 1), dtype=torch.uint8)
    if with_jacobian:
        J, w = D.empty(max(k, 1), JacobianBlocks.REC)[:k], D.empty(k)
    else:
        J = w = None
    jac = None
    if k:
        D.call("bamg_evaluate", cams, cams.shape[0], pts, st.obs_cam_pm, st.obs_pt_pm, st.pix_pm, k, huber,
               1 if with_jacobian else 0, J, w, behind, obj, nb)
        if with_jacobian:
            # the points' normal blocks depend on the Jacobian alone: queued ahead of the
            # objective readback so the device works through the host round trip
            jac = JacobianBlocks._from_records(st, J, w, problem.n_cameras, problem.n_points, problem._ci,
                                               problem._pi)
            jac.point_normal()
        host = res.cpu()
        n_behind = int(host[1:].view(torch.int32)[0])
        objective = float(host[0])
    else:
        n_behind, objective = 0, 0.0
    if n_behind:
        flagged = st.pm_perm[behind[:k].bool()].to(torch.int64)
        idx = torch.sort(flagged).values.cpu().numpy()
        raise BehindCameraError(idx)
    if not with_jacobian:
        return objective, None
    if jac is None:
        jac = JacobianBlocks._from_records(st, J, w, problem.n_cameras, problem.n_points, problem._ci, problem._pi)
    return objective, jac


def _objective_dev(problem: BundleProblem, cams, pts, obj_out, n_behind_out) -> None:
    """Objective-only evaluation into device slots (no readback): the LM driver's
    candidate step (solver.py:282-286) decides on the device (bamg_lm_trial)."""
    st = problem._st
    k = st.k
    if not k:
        obj_out.zero_()
        n_behind_out.zero_()
        return
    huber = 1 if problem.loss == "huber" else 0
    behind = D.empty(k, dtype=torch.uint8)
    D.call("bamg_evaluate", cams, cams.shape[0], pts, st.obs_cam_pm, st.obs_pt_pm, st.pix_pm, k, huber, 0, None, None, behind,
           obj_out, n_behind_out)


def gauge_nullspace(problem: BundleProblem, camera_params=None) -> DenseTall:
    """Camera-space near-nullspace basis, (9 n_cameras) x 16 (problem.py:332-352)."""
    cams, _ = _params(problem, camera_params, None)
    n = cams.shape[0]
    K = D.empty(n * CAMERA_SIZE, 16)
    if n:
        D.call("bamg_gauge_nullspace", cams, n, K)
    return DenseTall(K)
