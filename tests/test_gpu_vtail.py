"""Coarse V-cycle tail as one persistent cooperative kernel (vcycle.cuh k_vcycle_tail):
the recorded op list replays exactly what the per-level launches compute. Levels
the launched plan runs with k_row16_cta are bit-identical; a level the launched plan
runs through the half-storage pair differs only by summation order."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P
    from paper_2007_01941_b200 import scenes

    sc = scenes.large(n_clusters=1, n_points=60_000, threads=4)
    prob = P.BundleProblem(*sc.arrays())
    obj, jac = P.evaluate(prob)
    s = P.build_system(jac, P.Damping.from_jacobian(jac, 1e4))
    s.mode = P.choose_mode(s)
    h = P.build_hierarchy(s, P.gauge_nullspace(prob), P.visibility_strength(prob), max_coarse_dim=60)
    return P, s, h


def H(t):
    from paper_2007_01941_b200 import _device

    return _device.host(t)


def _apply(P, h, v, mb):
    from paper_2007_01941_b200 import _lib

    _lib.call("bamg_mg_set_tail", h._plan.handle, mb)
    h._plan.prepare()
    kinds = [int(_lib.lib().bamg_mg_level_kind(h._plan.handle, li)) for li in range(h.n_levels)]
    return H(h.apply(P._device.f64(v))), kinds


def test_tail_matches_launched_levels(setup):
    P, s, h = setup
    assert h._plan is not None and h.n_levels >= 3
    rng = np.random.default_rng(5)
    v = rng.normal(size=h.levels[0].scalar_dim)
    off, k_off = _apply(P, h, v, 0)
    assert 5 not in k_off
    # only the levels the launched plan runs with the row-CTA kernel: bit-identical
    rowcta_mb = 32
    on, k_on = _apply(P, h, v, rowcta_mb)
    if 5 in k_on:
        assert all(k_off[li] in (1, 4) for li, k in enumerate(k_on) if k == 5)
        np.testing.assert_array_equal(on, off)
    # every 16x16 level in the tail (half-storage levels included): summation order only
    big, k_big = _apply(P, h, v, 4096)
    assert 5 in k_big and k_big[0] != 5
    assert np.max(np.abs(big - off)) <= 1e-11 * np.max(np.abs(off))
    # repeated applications are deterministic
    again, _ = _apply(P, h, v, 4096)
    np.testing.assert_array_equal(again, big)
    _apply(P, h, v, -1)


def test_tail_pcg(setup):
    P, s, h = setup
    from paper_2007_01941_b200 import _lib

    its = []
    for mb in (0, 4096):
        _lib.call("bamg_mg_set_tail", h._plan.handle, mb)
        x, rep = P.pcg(s.matvec, h.apply, s.rhs_cam, tau=1e-30, max_iterations=2000, residual_tolerance=1e-6)
        its.append((rep.iterations, H(x)))
    _lib.call("bamg_mg_set_tail", h._plan.handle, -1)
    assert abs(its[0][0] - its[1][0]) <= 1
    assert np.linalg.norm(its[0][1] - its[1][1]) <= 1e-6 * np.linalg.norm(its[0][1])
