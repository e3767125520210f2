"""CPU oracle: a numpy / scipy restatement of the reference LM linear-solve path.

TEST INFRASTRUCTURE ONLY. Nothing in the product package imports this module;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may call it, and then only as the checker or the timed CPU
baseline.

The reference (`/root/reference/pkg/src/bamg`, Python + numpy + scipy) is
restated here function by function; every function names the reference lines it
follows. The arithmetic building blocks are the same third-party libraries the
reference calls (numpy ufuncs / einsum, scipy.sparse CSR/BSR kernels, LAPACK via
numpy.linalg and scipy.linalg), so the restatement is also a faithful CPU timing
baseline. Parity of this restatement with the reference itself is pinned by
``tests/test_oracle_golden.py`` against fixtures produced by
``oracle/make_golden.py`` (which imports the real reference in the build
container).

Conventions: cameras (nc, 9) = [angle-axis(3), t(3), f, k1, k2]; points (np, 3);
observation arrays in the problem's own order; block matrices are
(indptr, indices, blocks) triples with int64 indices, columns sorted per row.
"""

from __future__ import annotations

import dataclasses
import time

import numpy as np
import scipy.linalg
import scipy.sparse as sp

CAM = 9
PT = 3
NS = 16  # multigrid.py:25 NULLSPACE_DIM
RANK_TOL = 1e-10  # multigrid.py:26
LANCZOS_SEED = 20210607  # multigrid.py:27
LANCZOS_STEPS = 5  # multigrid.py:28
CHEB_HI, CHEB_LO = 1.1, 0.3  # multigrid.py:29-30
DIAG_MIN, DIAG_MAX = 1e-6, 1e32  # schur.py:21-22
MIN_DEPTH = 1e-12  # problem.py:25
SMALL = 1e-4  # rotation.py:16


class BehindCamera(Exception):
    """problem.py:28-36 -- carries ascending observation indices."""

    def __init__(self, idx):
        self.observation_indices = np.asarray(idx, dtype=np.int64)
        super().__init__(f"{len(self.observation_indices)} behind camera")


class Indefinite(Exception):
    """blockmat.py:25-39 -- first non-PD block."""

    def __init__(self, i):
        self.block_index = int(i)
        super().__init__(f"block {i} is not positive definite")


class NotSPD(Exception):
    """solver.py:30-31."""


class Diverged(Exception):
    """solver.py:34-35."""


# -- rotation (rotation.py:19-137) -------------------------------------------


def skew(v):
    z = np.zeros(v.shape[:-1])
    return np.stack([
        np.stack([z, -v[..., 2], v[..., 1]], -1),
        np.stack([v[..., 2], z, -v[..., 0]], -1),
        np.stack([-v[..., 1], v[..., 0], z], -1),
    ], -2)


def _angle_coeffs(aa):
    th2 = np.einsum("ni,ni->n", aa, aa)
    th = np.sqrt(th2)
    tiny = th < SMALL
    s = np.where(tiny, 1.0, th)
    return th2, th, tiny, s


def rotate(aa, X):
    """rotation.py:36-58 (Rodrigues on vectors, series below 1e-4)."""
    th2, th, tiny, s = _angle_coeffs(aa)
    with np.errstate(invalid="ignore", divide="ignore"):
        a = np.where(tiny, 1.0 - th2 / 6.0, np.sin(th) / s)
        b = np.where(tiny, 0.5 - th2 / 24.0, (1.0 - np.cos(th)) / np.where(tiny, 1.0, th2))
    u = np.cross(aa, X)
    return X + a[:, None] * u + b[:, None] * np.cross(aa, u)


def rotmat(aa):
    """rotation.py:61-71."""
    th2, th, tiny, s = _angle_coeffs(aa)
    a = np.where(tiny, 1.0 - th2 / 6.0, np.sin(th) / s)
    b = np.where(tiny, 0.5 - th2 / 24.0, (1.0 - np.cos(th)) / s**2)
    K = skew(aa)
    return np.eye(3) + a[:, None, None] * K + b[:, None, None] * (K @ K)


def right_jac(aa):
    """rotation.py:74-88."""
    th2, th, tiny, s = _angle_coeffs(aa)
    c1 = np.where(tiny, 0.5 - th2 / 24.0, (1.0 - np.cos(th)) / s**2)
    c2 = np.where(tiny, 1.0 / 6.0 - th2 / 120.0, (th - np.sin(th)) / s**3)
    K = skew(aa)
    return np.eye(3) - c1[:, None, None] * K + c2[:, None, None] * (K @ K)


def right_jac_inv(aa):
    """rotation.py:91-107."""
    th2, th, tiny, s = _angle_coeffs(aa)
    with np.errstate(invalid="ignore", divide="ignore"):
        cot = np.cos(s / 2.0) / np.sin(s / 2.0)
    d2 = np.where(tiny, 1.0 / 12.0 + th2 / 720.0, 1.0 / s**2 - cot / (2.0 * s))
    K = skew(aa)
    return np.eye(3) + 0.5 * K + d2[:, None, None] * (K @ K)


def d_rotate(aa, X):
    """rotation.py:110-114: -R [X]x Jr."""
    return -rotmat(aa) @ skew(X) @ right_jac(aa)


def canonicalize(aa):
    """rotation.py:124-137."""
    aa = np.array(np.atleast_2d(aa), dtype=float, copy=True)
    while True:
        th = np.linalg.norm(aa, axis=-1)
        big = th > np.pi
        if not big.any():
            return aa
        aa[big] *= (1.0 - 2.0 * np.pi / th[big])[:, None]


# -- problem (problem.py:179-352) ---------------------------------------------


@dataclasses.dataclass
class Problem:
    cams: np.ndarray
    pts: np.ndarray
    ci: np.ndarray
    pi: np.ndarray
    pix: np.ndarray
    loss: str = "trivial"

    @property
    def nc(self):
        return self.cams.shape[0]

    @property
    def npt(self):
        return self.pts.shape[0]

    @staticmethod
    def of(scene, loss="trivial"):
        cams = np.array(scene.camera_params, dtype=float, copy=True)
        cams[:, :3] = canonicalize(cams[:, :3])  # problem.py:106
        return Problem(cams, np.array(scene.points, float), np.asarray(scene.cam_index, np.int64),
                       np.asarray(scene.pt_index, np.int64), np.array(scene.pixels, float), loss)


@dataclasses.dataclass
class Jac:
    """problem.py:237-269 -- loss-weighted blocks in observation order."""

    F: np.ndarray
    E: np.ndarray
    r: np.ndarray
    w: np.ndarray
    ci: np.ndarray
    pi: np.ndarray
    nc: int
    npt: int

    def gradient(self):
        """problem.py:255-261."""
        gc = np.zeros((self.nc, CAM))
        gp = np.zeros((self.npt, PT))
        np.add.at(gc, self.ci, np.einsum("kij,ki->kj", self.F, self.r))
        np.add.at(gp, self.pi, np.einsum("kij,ki->kj", self.E, self.r))
        return gc, gp

    def normal_diag(self):
        """problem.py:263-269."""
        dc = np.zeros((self.nc, CAM))
        dp = np.zeros((self.npt, PT))
        np.add.at(dc, self.ci, np.einsum("kij,kij->kj", self.F, self.F))
        np.add.at(dp, self.pi, np.einsum("kij,kij->kj", self.E, self.E))
        return dc, dp


def loss_rho(s, kind):
    """problem.py:179-188."""
    if kind == "trivial":
        return s
    return np.where(s <= 1.0, s, 2.0 * np.sqrt(np.maximum(s, 1.0)) - 1.0)


def loss_sqrt_drho(s, kind):
    """problem.py:191-196."""
    if kind == "trivial":
        return np.ones_like(s)
    return np.where(s <= 1.0, 1.0, np.maximum(s, 1.0) ** -0.25)


def evaluate(prob: Problem, cams=None, pts=None, with_jacobian=True):
    """problem.py:202-219 (projection) + 272-326 (residual, F, E, weights)."""
    cams = prob.cams if cams is None else cams
    pts = prob.pts if pts is None else pts
    c = cams[prob.ci]
    X = pts[prob.pi]
    pc = rotate(c[:, :3], X) + c[:, 3:6]
    z = pc[:, 2]
    behind = z >= -MIN_DEPTH
    if behind.any():
        raise BehindCamera(np.flatnonzero(behind))
    p = -pc[:, :2] / z[:, None]
    n2 = np.einsum("ki,ki->k", p, p)
    f, k1, k2 = c[:, 6], c[:, 7], c[:, 8]
    dist = 1.0 + k1 * n2 + k2 * n2 * n2
    res = (f * dist)[:, None] * p - prob.pix
    s = np.einsum("ki,ki->k", res, res)
    obj = float(np.sum(loss_rho(s, prob.loss)))
    if not with_jacobian:
        return obj, None
    k = len(z)
    dp = np.zeros((k, 2, 3))
    dp[:, 0, 0] = dp[:, 1, 1] = -1.0 / z
    dp[:, 0, 2] = pc[:, 0] / z**2
    dp[:, 1, 2] = pc[:, 1] / z**2
    g = f * (2.0 * k1 + 4.0 * k2 * n2)
    dpix = (f * dist)[:, None, None] * np.eye(2) + g[:, None, None] * (p[:, :, None] * p[:, None, :])
    D = dpix @ dp
    F = np.empty((k, 2, CAM))
    F[:, :, 0:3] = D @ d_rotate(c[:, :3], X)
    F[:, :, 3:6] = D
    F[:, :, 6] = dist[:, None] * p
    F[:, :, 7] = (f * n2)[:, None] * p
    F[:, :, 8] = (f * n2 * n2)[:, None] * p
    E = D @ rotmat(c[:, :3])
    w = loss_sqrt_drho(s, prob.loss)
    return obj, Jac(F * w[:, None, None], E * w[:, None, None], res * w[:, None], w,
                    prob.ci, prob.pi, prob.nc, prob.npt)


def gauge_nullspace(cams):
    """problem.py:332-352: (9 nc, 16) near-nullspace."""
    n = cams.shape[0]
    K = np.zeros((n, CAM, NS))
    K[:, 3:6, 0:3] = -rotmat(cams[:, :3])
    K[:, 0:3, 3:6] = -right_jac_inv(cams[:, :3])
    K[:, 3:6, 6] = cams[:, 3:6]
    K[:, np.arange(CAM), 7 + np.arange(CAM)] = 1.0
    return K.reshape(n * CAM, NS)


# -- block containers ---------------------------------------------------------


@dataclasses.dataclass
class BSR:
    """blockmat.py:152-193 layout."""

    nbr: int
    nbc: int
    indptr: np.ndarray
    indices: np.ndarray
    blocks: np.ndarray

    @property
    def rbs(self):
        return self.blocks.shape[1]

    @property
    def cbs(self):
        return self.blocks.shape[2]

    def scipy(self):
        return sp.bsr_matrix((self.blocks, self.indices, self.indptr),
                             shape=(self.nbr * self.rbs, self.nbc * self.cbs))

    def matvec(self, x):
        return self.scipy() @ x

    def rmatvec(self, x):
        return self.scipy().T @ x

    def dense(self):
        return self.scipy().toarray()

    def rows(self):
        return np.repeat(np.arange(self.nbr), np.diff(self.indptr))

    def diag_blocks(self):
        """blockmat.py:270-282."""
        out = np.zeros((self.nbr, self.rbs, self.cbs))
        r = self.rows()
        on = r == self.indices
        out[r[on]] = self.blocks[on]
        return out

    @staticmethod
    def from_scipy(m, rbs, cbs):
        """blockmat.py:232-245 (csr -> bsr, sorted)."""
        b = m.tobsr(blocksize=(rbs, cbs))
        b.sort_indices()
        return BSR(b.shape[0] // rbs, b.shape[1] // cbs, b.indptr.astype(np.int64),
                   b.indices.astype(np.int64), np.ascontiguousarray(b.data, float))

    @staticmethod
    def from_triplets(nbr, nbc, r, c, blocks):
        """blockmat.py:195-230: lexsort + duplicate summation."""
        order = np.lexsort((c, r))
        r, c, blocks = r[order], c[order], blocks[order]
        first = np.ones(len(r), bool)
        first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        st = np.flatnonzero(first)
        summed = np.add.reduceat(blocks, st, axis=0) if len(st) else blocks[:0]
        ptr = np.zeros(nbr + 1, np.int64)
        np.cumsum(np.bincount(r[st], minlength=nbr), out=ptr[1:])
        return BSR(nbr, nbc, ptr, c[st].astype(np.int64), summed)


def chol_inv(blocks):
    """blockmat.py:95-115: batched Cholesky, first failing index, L^-T L^-1."""
    try:
        L = np.linalg.cholesky(blocks)
    except np.linalg.LinAlgError:
        for i, b in enumerate(blocks):
            try:
                np.linalg.cholesky(b)
            except np.linalg.LinAlgError:
                raise Indefinite(i) from None
        raise
    Li = np.linalg.inv(L)
    return np.einsum("nki,nkj->nij", Li, Li)


def bdiag_apply(blocks, x):
    b = blocks.shape[1]
    return np.einsum("nij,nj->ni", blocks, x.reshape(-1, b)).ravel()


# -- reduced system (schur.py) ------------------------------------------------


@dataclasses.dataclass
class System:
    A: np.ndarray
    C: np.ndarray
    Cinv: np.ndarray
    W: BSR
    rhs: np.ndarray
    gpt: np.ndarray
    S: BSR | None = None
    mode: str = "implicit"

    def matvec(self, x):
        """schur.py:84-91."""
        if self.mode == "explicit":
            return self.explicit().matvec(x)
        return bdiag_apply(self.A, x) - self.W.matvec(bdiag_apply(self.Cinv, self.W.rmatvec(x)))

    def explicit(self):
        if self.S is None:
            self.S = schur_explicit(self)
        return self.S


def damping(jac: Jac, radius):
    """schur.py:38-47."""
    if not radius > 0:
        raise ValueError("trust radius must be positive")
    dc, dp = jac.normal_diag()
    return (np.clip(dc, DIAG_MIN, DIAG_MAX) / radius, np.clip(dp, DIAG_MIN, DIAG_MAX) / radius)


def build_system(jac: Jac, damp):
    """schur.py:99-125."""
    dc, dp = damp
    A = np.zeros((jac.nc, CAM, CAM))
    np.add.at(A, jac.ci, np.einsum("kij,kil->kjl", jac.F, jac.F))
    A[:, np.arange(CAM), np.arange(CAM)] += dc
    C = np.zeros((jac.npt, PT, PT))
    np.add.at(C, jac.pi, np.einsum("kij,kil->kjl", jac.E, jac.E))
    C[:, np.arange(PT), np.arange(PT)] += dp
    W = BSR.from_triplets(jac.nc, jac.npt, jac.ci, jac.pi, np.einsum("kij,kil->kjl", jac.F, jac.E))
    gc, gp = jac.gradient()
    bc, bp = -gc.ravel(), -gp.ravel()
    Cinv = chol_inv(C)
    rhs = bc - W.matvec(bdiag_apply(Cinv, bp))
    return System(A, C, Cinv, W, rhs, bp)


def schur_explicit(s: System) -> BSR:
    """schur.py:128-144 (+ blockmat.py:308-353): symmetrised A - (W C^-1) W^T."""
    W = s.W
    Y = BSR(W.nbr, W.nbc, W.indptr, W.indices,
            np.einsum("nij,njk->nik", W.blocks, s.Cinv[W.indices]))
    Wt = BSR.from_triplets(W.nbc, W.nbr, W.indices, W.rows(), W.blocks.transpose(0, 2, 1))
    off = Y.scipy().tocsr() @ Wt.scipy().tocsr()
    Abs = BSR(s.A.shape[0], s.A.shape[0], np.arange(s.A.shape[0] + 1), np.arange(s.A.shape[0]), s.A)
    raw = Abs.scipy().tocsr() - BSR.from_scipy(off, CAM, CAM).scipy().tocsr()
    sym = (raw + raw.T).tocsr()
    sym.data *= 0.5
    return BSR.from_scipy(sym, CAM, CAM)


def covisible_blocks(s: System) -> int:
    """schur.py:147-159, including the int8 pattern-product wrap."""
    if s.S is not None:
        return len(s.S.indices)
    pat = sp.csr_matrix((np.ones(len(s.W.indices), np.int8), s.W.indices, s.W.indptr),
                        shape=(s.W.nbr, s.W.nbc))
    return int((pat @ pat.T).nnz)


def choose_mode(s: System) -> str:
    """schur.py:162-168."""
    nc, npt = s.A.shape[0], s.C.shape[0]
    exp = 2 * covisible_blocks(s) * CAM * CAM
    imp = 2 * (nc * CAM * CAM + 2 * len(s.W.indices) * CAM * PT + npt * PT * PT)
    return "explicit" if exp <= imp else "implicit"


def back_substitute(s: System, dc):
    """schur.py:171-173."""
    return bdiag_apply(s.Cinv, s.gpt - s.W.rmatvec(dc))


def model_decrease(s: System, dc):
    """schur.py:176-188."""
    return float(s.rhs @ dc - 0.5 * dc @ s.matvec(dc) + 0.5 * s.gpt @ bdiag_apply(s.Cinv, s.gpt))


# -- multigrid (multigrid.py) -------------------------------------------------


def visibility_strength(ci, pi, nc, npt):
    """multigrid.py:52-80: cosine of visibility sets, CSR without diagonal."""
    deg = np.bincount(ci, minlength=nc).astype(float)
    if np.any(deg == 0):
        raise ValueError("camera(s) observe no points; visibility strength undefined")
    inc = sp.csr_matrix((np.ones(len(ci)), (ci, pi)), shape=(nc, npt))
    cnt = (inc @ inc.T).tocoo()
    off = cnt.row != cnt.col
    r, c, v = cnt.row[off], cnt.col[off], cnt.data[off]
    return sp.csr_matrix((np.minimum(v / np.sqrt(deg[r] * deg[c]), 1.0), (r, c)), shape=(nc, nc))


def operator_strength(op: BSR):
    """multigrid.py:83-98."""
    nrm = np.sqrt(np.einsum("nij,nij->n", op.blocks, op.blocks))
    r = op.rows()
    on = r == op.indices
    dn = np.zeros(op.nbr)
    dn[r[on]] = nrm[on]
    if np.any(dn == 0):
        raise ValueError("operator has a structurally zero diagonal block")
    off = ~on
    v = np.minimum(nrm[off] / np.sqrt(dn[r[off]] * dn[op.indices[off]]), 1.0)
    return sp.csr_matrix((v, (r[off], op.indices[off])), shape=(op.nbr, op.nbc))


def aggregate(G, max_size=20):
    """multigrid.py:127-176 (Alg. 2): greedy scan, then leftover post-pass.

    The in-scan choice is the first neighbour, ordered by (-strength,
    already-aggregated, index), that is unaggregated (pair) or sits in an
    aggregate smaller than ``max_size`` (join). Leftovers join the neighbour with
    the largest (strength, -index) whose aggregate has at most ``max_size``.
    """
    G = sp.csr_matrix(G)
    n = G.shape[0]
    ip, ix, gv = G.indptr, G.indices, G.data
    agg = np.full(n, -1, np.int64)
    size = []
    for i in range(n):
        if agg[i] >= 0:
            continue
        cols, vals = ix[ip[i]:ip[i + 1]], gv[ip[i]:ip[i + 1]]
        if len(cols) == 0:
            continue
        order = np.lexsort((cols, agg[cols] >= 0, -vals))
        for j in cols[order]:
            if agg[j] < 0:
                agg[i] = agg[j] = len(size)
                size.append(2)
                break
            if size[agg[j]] < max_size:
                agg[i] = agg[j]
                size[agg[j]] += 1
                break
    for i in np.flatnonzero(agg < 0):
        cols, vals = ix[ip[i]:ip[i + 1]], gv[ip[i]:ip[i + 1]]
        best = None
        for v, c in zip(vals, cols):
            if size[agg[c]] <= max_size and (best is None or (v, -c) > (best[0], -best[1])):
                best = (v, c)
        if best is None:
            agg[i] = len(size)
            size.append(1)
        else:
            agg[i] = agg[best[1]]
            size[agg[i]] += 1
    return agg, len(size)


def members_of(agg, n_agg):
    """multigrid.py:121-124 (stable grouping, ascending members)."""
    order = np.argsort(agg, kind="stable")
    cuts = np.searchsorted(agg[order], np.arange(n_agg + 1))
    return [order[cuts[a]:cuts[a + 1]] for a in range(n_agg)]


def prolongation(agg, n_agg, K, bs):
    """multigrid.py:179-237: per-aggregate QR of the near-nullspace rows.

    Returns (P as BSR, K_coarse (16 n_agg, 16), padded dofs, info) where info
    records (pivoted?, rank) per aggregate.
    """
    n = len(agg)
    Kc = np.zeros((n_agg * NS, NS))
    Pb = np.zeros((n, bs, NS))
    padded, info = [], []
    for a, mem in enumerate(members_of(agg, n_agg)):
        rows = (mem[:, None] * bs + np.arange(bs)).ravel()
        loc = K[rows]
        m = loc.shape[0]
        keep = min(m, NS)
        done = False
        if m >= NS:
            q, r = scipy.linalg.qr(loc, mode="economic")
            d = np.diag(r)
            if np.min(np.abs(d)) > RANK_TOL * np.max(np.abs(d)):
                sg = np.where(d < 0, -1.0, 1.0)
                blk = q * sg
                Kc[a * NS:(a + 1) * NS] = r * sg[:, None]
                info.append((False, NS))
                done = True
        if not done:
            q, r, piv = scipy.linalg.qr(loc, mode="full", pivoting=True)
            d = np.abs(np.diag(r))
            rank = int(np.sum(d > RANK_TOL * d[0])) if d.size and d[0] > 0 else 0
            ru = np.zeros((NS, NS))
            ru[:rank, piv] = r[:rank, :]
            Kc[a * NS:(a + 1) * NS] = ru
            blk = np.zeros((m, NS))
            blk[:, :keep] = q[:, :keep]
            padded.extend(a * NS + c for c in range(keep, NS))
            info.append((True, rank))
        Pb[mem] = blk.reshape(len(mem), bs, NS)
    P = BSR(n, n_agg, np.arange(n + 1, dtype=np.int64), agg.astype(np.int64), Pb)
    return P, Kc, np.asarray(padded, np.int64), info


def galerkin(P: BSR, A: BSR, padded):
    """multigrid.py:409-411 + 444-471: sym(P^T A P) with decoupled-dof patch."""
    Pt = BSR.from_triplets(P.nbc, P.nbr, P.indices, P.rows(), P.blocks.transpose(0, 2, 1))
    pta = BSR.from_scipy(Pt.scipy().tocsr() @ A.scipy().tocsr(), NS, A.cbs)
    ac = BSR.from_scipy(pta.scipy().tocsr() @ P.scipy().tocsr(), NS, NS)
    raw = ac.scipy().tocsr()
    sym = (raw + raw.T).tocsr()
    sym.data *= 0.5
    out = BSR.from_scipy(sym, NS, NS)
    r = out.rows()
    for dof in padded:
        blk, loc = divmod(int(dof), NS)
        hit = np.flatnonzero((r == blk) & (out.indices == blk))
        if len(hit):
            out.blocks[hit[0], loc, loc] += 1.0
    return out


def lambda_max(matvec, Dblocks, Dinv, n, steps=LANCZOS_STEPS, seed=LANCZOS_SEED, v0=None):
    """multigrid.py:243-284: D-inner-product Lanczos with full reorthogonalisation."""
    v = np.random.default_rng(seed).standard_normal(n) if v0 is None else v0
    Dm = lambda x: bdiag_apply(Dblocks, x)  # noqa: E731
    q = v / np.sqrt(v @ Dm(v))
    qprev = np.zeros(n)
    basis = [q]
    al, be = [], []
    bprev = 0.0
    for _ in range(steps):
        u = matvec(q)
        a = float(q @ u)
        z = bdiag_apply(Dinv, u) - a * q - bprev * qprev
        for qb in basis:
            z = z - qb * (qb @ Dm(z))
        al.append(a)
        b2 = float(z @ Dm(z))
        if not np.isfinite(b2):
            raise FloatingPointError("Lanczos iteration produced a non-finite value")
        if b2 <= 0 or np.sqrt(b2) < 1e-12 * abs(a):
            break
        b = np.sqrt(b2)
        be.append(b)
        qprev, q = q, z / b
        basis.append(q)
        bprev = b
    be = be[:len(al) - 1]
    return float(scipy.linalg.eigh_tridiagonal(np.asarray(al), np.asarray(be), eigvals_only=True)[-1])


@dataclasses.dataclass
class Cheb:
    """multigrid.py:287-336."""

    Dinv: np.ndarray
    lam: float
    lo: float
    hi: float
    its: int = 2

    def apply(self, matvec, x, b):
        th = 0.5 * (self.hi + self.lo)
        de = 0.5 * (self.hi - self.lo)
        sg = th / de
        rho = 1.0 / sg
        if x is None:
            r, x = b.copy(), np.zeros_like(b)
        else:
            x = x.copy()
            r = b - matvec(x)
        d = bdiag_apply(self.Dinv, r) / th
        x += d
        for _ in range(self.its - 1):
            r = b - matvec(x)
            rn = 1.0 / (2.0 * sg - rho)
            d = rn * rho * d + (2.0 * rn / de) * bdiag_apply(self.Dinv, r)
            x += d
            rho = rn
        return x


@dataclasses.dataclass
class Level:
    matvec: object
    dim: int
    op: BSR
    smoother: Cheb | None = None
    P: BSR | None = None
    agg: np.ndarray | None = None
    n_agg: int = 0
    K: np.ndarray | None = None
    info: list | None = None
    padded: np.ndarray | None = None
    coarse: object = None


def hierarchy(s: System, K, G, max_coarse=400, max_ratio=0.7, max_agg=20, seed=LANCZOS_SEED,
              level0_agg=None):
    """multigrid.py:371-441."""
    S = s.explicit()
    levels = [Level(s.matvec, S.nbr * CAM, S, K=K)]
    while levels[-1].dim > max_coarse:
        cur = levels[-1]
        first = len(levels) == 1
        if first and level0_agg is not None:
            agg, na = level0_agg
        else:
            agg, na = aggregate(G if first else operator_strength(cur.op), max_agg)
        if na * NS / cur.dim > max_ratio:
            break
        bs = CAM if first else NS
        P, Kc, pad, info = prolongation(agg, na, cur.K, bs)
        Ac = galerkin(P, cur.op, pad)
        cur.P, cur.agg, cur.n_agg, cur.info, cur.padded = P, agg, na, info, pad
        levels.append(Level(Ac.matvec, na * NS, Ac, K=Kc))
    for li, L in enumerate(levels[:-1]):
        D = L.op.diag_blocks()
        Dinv = chol_inv(D)
        lam = lambda_max(L.matvec, D, Dinv, L.dim, seed=seed + li)
        if not lam > 0:
            raise ValueError(f"nonpositive spectral estimate {lam}")
        L.smoother = Cheb(Dinv, lam, CHEB_LO * lam, CHEB_HI * lam)
    last = levels[-1]
    dense = last.op.dense()
    try:
        last.coarse = scipy.linalg.cho_factor(0.5 * (dense + dense.T))
    except scipy.linalg.LinAlgError as e:
        raise ValueError("coarsest-level operator is not positive definite") from e
    return levels


def vcycle(levels, l, x, b):
    """multigrid.py:474-483."""
    L = levels[l]
    if L.coarse is not None:
        return scipy.linalg.cho_solve(L.coarse, b)
    x = L.smoother.apply(L.matvec, x, b)
    r = b - L.matvec(x)
    xc = vcycle(levels, l + 1, None, L.P.rmatvec(r))
    x = x + L.P.matvec(xc)
    return L.smoother.apply(L.matvec, x, b)


def pbj(s: System):
    """precond.py:24-56 (explicit-S branch or point-accumulated diagonal)."""
    if s.S is not None:
        blocks = s.S.diag_blocks()
    else:
        blocks = s.A.copy()
        Y = np.einsum("nij,njk->nik", s.W.blocks, s.Cinv[s.W.indices])
        np.add.at(blocks, s.W.rows(), -np.einsum("nij,nkj->nik", Y, s.W.blocks))
    try:
        Dinv = chol_inv(blocks)
    except Indefinite as e:
        raise Indefinite(e.block_index) from None
    return lambda r: bdiag_apply(Dinv, r)


VJ_CLUSTER_CAP = 100  # precond.py:21


def visibility_cluster(G, max_cluster=VJ_CLUSTER_CAP):
    """precond.py:59-62: the MG aggregation with a larger cap -> (assignment, n)."""
    return aggregate(G, max_cluster)


def vj(s: System, agg, n_agg):
    """precond.py:82-144 vj_setup + VisibilityJacobi.apply (69-78).

    Per cluster, the principal submatrix of S over the members (ascending): copied
    from the assembled S when present (96-111), else A's diagonal blocks minus the
    in-cluster point contributions W_a C^-1 W_b^T (112-136); scipy cho_factor, and
    cho_solve per cluster in the apply. Indefinite(cid) on a failed factor.
    """
    agg = np.asarray(agg)
    if len(agg) != s.A.shape[0]:
        raise ValueError(f"partition covers {len(agg)} cameras, system has {s.A.shape[0]}")
    members = members_of(agg, n_agg)
    factors = []
    wrows = s.W.rows()
    for cid, mem in enumerate(members):
        m = len(mem)
        local = np.zeros((m * CAM, m * CAM))
        pos = {int(c): k for k, c in enumerate(mem)}
        if s.S is not None:
            S = s.S
            for k, cam in enumerate(mem):
                for q in range(S.indptr[cam], S.indptr[cam + 1]):
                    o = pos.get(int(S.indices[q]))
                    if o is not None:
                        local[k * CAM:(k + 1) * CAM, o * CAM:(o + 1) * CAM] = S.blocks[q]
        else:
            for k, cam in enumerate(mem):
                local[k * CAM:(k + 1) * CAM, k * CAM:(k + 1) * CAM] = s.A[cam]
            inc = agg[wrows] == cid
            for pt in np.unique(s.W.indices[inc]):
                sel = np.flatnonzero((s.W.indices == pt) & inc)
                cams_p = wrows[sel]
                wk = s.W.blocks[sel]
                y = wk @ s.Cinv[pt]
                contrib = np.einsum("aij,bkj->aibk", y, wk)
                for a, ca in enumerate(cams_p):
                    for b, cb in enumerate(cams_p):
                        ia, ib = pos[int(ca)], pos[int(cb)]
                        local[ia * CAM:(ia + 1) * CAM, ib * CAM:(ib + 1) * CAM] -= contrib[a, :, b, :]
        try:
            factors.append(scipy.linalg.cho_factor(local))
        except scipy.linalg.LinAlgError:
            raise Indefinite(cid) from None

    def apply(r):
        out = np.empty_like(r)
        rb, ob = r.reshape(-1, CAM), out.reshape(-1, CAM)
        for mem, f in zip(members, factors):
            ob[mem] = scipy.linalg.cho_solve(f, rb[mem].ravel()).reshape(-1, CAM)
        return out

    return apply


# -- solver (solver.py) ---------------------------------------------------------


@dataclasses.dataclass
class CgOut:
    iterations: int
    stop_reason: str
    relative_residual: float
    q_history: list


def pcg(A, M, b, tau, max_iterations=500, residual_tolerance=1e-12):
    """solver.py:38-128."""
    qh = [0.0]
    bn = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    if bn == 0.0:
        return x, CgOut(0, "residual_tol", 0.0, qh)
    r = b.copy()
    z = M(r)
    rz = float(r @ z)
    if not np.isfinite(rz):
        raise Diverged("preconditioner produced a non-finite value")
    if rz <= 0.0:
        raise NotSPD(f"<r, M r> = {rz:.3e} at iteration 0")
    p = z.copy()
    qv, rel = 0.0, 1.0
    for i in range(1, max_iterations + 1):
        ap = A(p)
        pap = float(p @ ap)
        if not np.isfinite(pap):
            raise Diverged("operator produced a non-finite value")
        if pap <= 0.0:
            raise Diverged(f"nonpositive curvature {pap:.3e}")
        al = rz / pap
        x += al * p
        r -= al * ap
        qv -= 0.5 * al * rz
        qh.append(qv)
        rel = float(np.linalg.norm(r)) / bn
        if not np.isfinite(rel):
            raise Diverged("residual became non-finite")
        if rel <= residual_tolerance:
            return x, CgOut(i, "residual_tol", rel, qh)
        if len(qh) >= 2 and qh[-1] != 0.0 and (len(qh) - 1) * (qh[-1] - qh[-2]) / qh[-1] <= tau:
            return x, CgOut(i, "forcing", rel, qh)
        z = M(r)
        rzn = float(r @ z)
        if not np.isfinite(rzn):
            raise Diverged("preconditioner produced a non-finite value")
        if rzn <= 0.0:
            raise NotSPD(f"<r, M r> = {rzn:.3e} at iteration {i}")
        p = z + (rzn / rz) * p
        rz = rzn
    return x, CgOut(max_iterations, "max_iterations", rel, qh)


@dataclasses.dataclass
class StepRecord:
    """solver.py:173-184."""

    iteration: int
    objective: float
    cg_iterations: int
    setup_seconds: float
    solve_seconds: float
    radius: float
    accepted: bool
    step_norm: float = 0.0
    rho: float = 0.0
    cg_stop_reason: str = ""


def lm_solve(prob: Problem, preconditioner="multigrid", tau=1e-30, max_iterations=10,
             cg_max_iterations=20000, initial_radius=1e4, cg_residual_tolerance=1e-6,
             min_rho=1e-3, function_tolerance=0.0, gradient_tolerance=0.0,
             parameter_tolerance=0.0, mg_max_coarse_dim=400, mg_max_ratio=0.7,
             mg_max_aggregate=20, timings=None):
    """solver.py:205-319 with the BASELINE settings of SURVEY 8(d) as defaults.

    The CG residual tolerance is forwarded (the reference needs a patch for it,
    SURVEY TL;DR hazard 4). Rejected trials reuse the Jacobian.
    """
    cams, pts = prob.cams.copy(), prob.pts.copy()
    radius = initial_radius
    obj, jac = evaluate(prob, cams, pts)
    recs = [StepRecord(0, obj, 0, 0.0, 0.0, radius, True)]
    G = None
    l0 = None
    clusters = None
    if preconditioner in ("multigrid", "visibility"):
        G = visibility_strength(prob.ci, prob.pi, prob.nc, prob.npt)
    if preconditioner == "visibility":
        clusters = visibility_cluster(G)
    it = 0
    termination = "max_iterations"
    while it < max_iterations:
        gc, gp = jac.gradient()
        gmax = max(float(np.max(np.abs(gc))) if gc.size else 0.0,
                   float(np.max(np.abs(gp))) if gp.size else 0.0)
        if gmax < gradient_tolerance:
            termination = "gradient_tolerance"
            break
        it += 1
        t0 = time.perf_counter()
        s = build_system(jac, damping(jac, radius))
        s.mode = choose_mode(s)
        if preconditioner == "multigrid":
            if l0 is None:
                l0 = aggregate(G, mg_max_aggregate)
            levels = hierarchy(s, gauge_nullspace(cams), G, mg_max_coarse_dim, mg_max_ratio,
                               mg_max_aggregate, level0_agg=l0)
            M = lambda r: vcycle(levels, 0, None, r)  # noqa: E731
        elif preconditioner == "visibility":
            M = vj(s, *clusters)
        else:
            if s.mode == "explicit":
                s.explicit()
            M = pbj(s)
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        dc, cg = pcg(s.matvec, M, s.rhs, tau, cg_max_iterations, cg_residual_tolerance)
        dp = back_substitute(s, dc)
        t_solve = time.perf_counter() - t0
        if timings is not None:
            timings.append((t_setup, t_solve))
        dec = model_decrease(s, dc)
        ncams = cams + dc.reshape(-1, CAM)
        npts = pts + dp.reshape(-1, PT)
        snorm = float(np.sqrt(dc @ dc + dp @ dp))
        try:
            nobj, _ = evaluate(prob, ncams, npts, with_jacobian=False)
            rho = 0.5 * (obj - nobj) / dec if dec > 0 else -np.inf
        except BehindCamera:
            nobj, rho = obj, -np.inf
        if rho > min_rho:
            cams, pts = ncams, npts
            cams[:, :3] = canonicalize(cams[:, :3])
            prev = obj
            obj, jac = evaluate(prob, cams, pts)
            radius /= max(1.0 / 3.0, 1.0 - (2.0 * rho - 1.0) ** 3)
            recs.append(StepRecord(it, obj, cg.iterations, t_setup, t_solve, radius, True,
                                   snorm, rho, cg.stop_reason))
            if prev - obj < function_tolerance * prev:
                termination = "function_tolerance"
                break
            pn = float(np.sqrt(np.sum(cams**2) + np.sum(pts**2)))
            if snorm < parameter_tolerance * (pn + parameter_tolerance):
                termination = "parameter_tolerance"
                break
        else:
            radius /= 2.0
            recs.append(StepRecord(it, obj, cg.iterations, t_setup, t_solve, radius, False,
                                   snorm, rho, cg.stop_reason))
            if radius < 1e-32:
                termination = "radius_underflow"
                break
    return cams, pts, recs, termination


def linear_solve(prob: Problem, radius=1e4, preconditioner="multigrid", tau=1e-30,
                 cg_max_iterations=20000, cg_residual_tolerance=1e-6, l0=None, G=None, jac=None):
    """One LM linear solve at the initial point (solver.py:244-274), for timing.

    The parameter-independent strength graph G and its level-0 aggregation may be
    passed in (computed once per problem, as lm_solve does: solver.py:221-230).
    """
    if jac is None:
        obj, jac = evaluate(prob)
    t0 = time.perf_counter()
    s = build_system(jac, damping(jac, radius))
    s.mode = choose_mode(s)
    if preconditioner == "multigrid":
        if G is None:
            G = visibility_strength(prob.ci, prob.pi, prob.nc, prob.npt)
        if l0 is None:
            l0 = aggregate(G)
        levels = hierarchy(s, gauge_nullspace(prob.cams), G, level0_agg=l0)
        M = lambda r: vcycle(levels, 0, None, r)  # noqa: E731
    elif preconditioner == "visibility":
        if G is None:
            G = visibility_strength(prob.ci, prob.pi, prob.nc, prob.npt)
        M = vj(s, *visibility_cluster(G))
    else:
        s.explicit()
        M = pbj(s)
    t1 = time.perf_counter()
    dc, cg = pcg(s.matvec, M, s.rhs, tau, cg_max_iterations, cg_residual_tolerance)
    dp = back_substitute(s, dc)
    t2 = time.perf_counter()
    return dict(dc=dc, dp=dp, cg=cg, setup=t1 - t0, solve=t2 - t1, system=s)
