"""Plain-text problem file I/O (drop-in for `bamg.balio`, balio.py:1-97).

Layout: a header line ``n_cameras n_points n_observations``; one line per
observation ``camera point x y``; then nine lines per camera and three per point,
one scalar per line, written with 17 significant digits so a write/read round trip
reproduces every float bit-exactly. Blank lines are skipped on reading.

The parsing and formatting run in libbamg_b200 (multi-threaded C++ over a mapped
file: two passes, line counts then per-chunk parsing), with the reference's error
classes, messages and 1-based line numbers. ``read_bal_arrays`` / ``write_bal_arrays``
work on host numpy arrays (no GPU needed); ``read_bal`` / ``write_bal`` take and give
a BundleProblem.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib


class BalFormatError(Exception):
    """Malformed problem file; carries the 1-based line number (balio.py:17-22)."""

    def __init__(self, lineno: int, message: str):
        self.lineno = lineno
        super().__init__(f"line {lineno}: {message}")


_FORMAT = 5  # BAMG_ERR_FORMAT


def _path(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _check(rc: int, line: np.ndarray, msg, path) -> None:
    if rc == 0:
        return
    text = msg.value.decode(errors="replace")
    if rc == _FORMAT:
        raise BalFormatError(int(line[0]), text)
    raise OSError(text or f"cannot access {os.fspath(path)}")


def read_bal_arrays(path, n_threads: int = 0):
    """(camera_params (nc,9), points (np,3), cam_index, pt_index (k,) int64, pixels (k,2)) as numpy."""
    L = _lib.lib()
    p = _path(path)
    counts = np.zeros(3, dtype=np.int64)
    line = np.zeros(1, dtype=np.int64)
    msg = ctypes.create_string_buffer(512)
    _check(L.bamg_bal_read_header(p, counts.ctypes.data, line.ctypes.data, msg, 512), line, msg, path)
    nc, npt, k = (int(v) for v in counts)
    cams = np.zeros((nc, 9))
    pts = np.zeros((npt, 3))
    ci = np.zeros(k, dtype=np.int64)
    pi = np.zeros(k, dtype=np.int64)
    pix = np.zeros((k, 2))
    rc = L.bamg_bal_read(p, nc, npt, k, ci.ctypes.data, pi.ctypes.data, pix.ctypes.data, cams.ctypes.data,
                         pts.ctypes.data, int(n_threads), line.ctypes.data, msg, 512)
    _check(rc, line, msg, path)
    return cams, pts, ci, pi, pix


def write_bal_arrays(path, camera_params, points, cam_index, pt_index, pixels, n_threads: int = 0) -> None:
    cams = np.ascontiguousarray(camera_params, dtype=np.float64).reshape(-1, 9)
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    ci = np.ascontiguousarray(cam_index, dtype=np.int64).reshape(-1)
    pi = np.ascontiguousarray(pt_index, dtype=np.int64).reshape(-1)
    pix = np.ascontiguousarray(pixels, dtype=np.float64).reshape(-1, 2)
    rc = _lib.lib().bamg_bal_write(_path(path), cams.shape[0], pts.shape[0], ci.shape[0], ci.ctypes.data,
                                   pi.ctypes.data, pix.ctypes.data, cams.ctypes.data, pts.ctypes.data,
                                   int(n_threads))
    if rc != 0:
        raise OSError(f"cannot write {os.fspath(path)}")


def _host(a):
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def write_bal(path, problem) -> None:
    """balio.py:25-35."""
    write_bal_arrays(path, _host(problem.camera_params), _host(problem.points), _host(problem.cam_index),
                     _host(problem.pt_index), _host(problem.pixels))


def read_bal(path, loss: str = "trivial"):
    """balio.py:38-97: parse, validate, and build the BundleProblem (device arrays)."""
    from .problem import BundleProblem

    cams, pts, ci, pi, pix = read_bal_arrays(path)
    return BundleProblem(cams, pts, ci, pi, pix, loss)
