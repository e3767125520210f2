import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def relerr(got, want):
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    d = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (d if d else 1.0))


def max_entry_rel(got, want, floor=0.0):
    """max |got-want| / max(|want|, floor) over entries (per-entry relative)."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    den = np.maximum(np.abs(want), floor)
    mask = den > 0
    if not mask.any():
        return float(np.max(np.abs(got - want))) if got.size else 0.0
    return float(np.max(np.abs(got - want)[mask] / den[mask]))


def block_rel(got, want):
    """per-entry error normalised by each block's max-abs entry."""
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    if want.size == 0:
        return 0.0
    scale = np.max(np.abs(want.reshape(want.shape[0], -1)), axis=1)
    scale = np.where(scale > 0, scale, 1.0)
    diff = np.max(np.abs((got - want).reshape(want.shape[0], -1)), axis=1)
    return float(np.max(diff / scale))


@pytest.fixture(scope="session")
def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


VJ_CASES = ["ring", "r1003", "r1004", "r1008"]


def vj_inputs(tag, g):
    """(cams, pts, ci, pi, pix) of a visibility-Jacobi golden case (tests/golden/vj_cases.npz)."""
    from paper_2007_01941_b200 import scenes

    if tag == "ring":
        sc = scenes.ring()
        assert sc.digest() == str(g["ring_digest"]), "scene generator drifted from the golden"
        return sc.camera_params, sc.points, sc.cam_index, sc.pt_index, sc.pixels
    return g[f"{tag}_cams"], g[f"{tag}_pts"], g[f"{tag}_ci"], g[f"{tag}_pi"], g[f"{tag}_pix"]
