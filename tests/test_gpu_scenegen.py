"""Device-side scene generation for configs 3-5 (csrc/scenegen.cu).

The device generator draws from its own counter-based streams, so it is checked by
what the model fixes rather than by digests: determinism in the seed, the structural
rules of `scenes._finish` (point-major order, >= 2 cameras per point, no empty camera,
depth / field-of-view limits at the truth, in front at the start), the pixel model
(residuals at the truth are the N(0, 1) noise, through the CPU oracle's projection),
the perturbation scales, the visibility rules of each config, and the same per-point
statistics as the numpy generator on the same parameters.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SMALL = {
    3: dict(n_cameras=400, n_points=20_000, side=63.0),
    4: dict(n_cameras=800, n_points=40_000, n_clusters=4, side=300.0),
    5: dict(n_cameras=800, n_points=50_000),
}


@pytest.fixture(scope="module", params=[3, 4, 5], ids=lambda n: f"c{n}")
def gen(request):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_01941_b200 import scenes

    n = request.param
    return n, scenes.device_config(n, seed=3, **SMALL[n]).to_host()


def test_deterministic_in_seed(gen):
    from paper_2007_01941_b200 import scenes

    n, a = gen
    b = scenes.device_config(n, seed=3, **SMALL[n]).to_host()
    c = scenes.device_config(n, seed=4, **SMALL[n]).to_host()
    assert a.digest() == b.digest()
    assert a.digest() != c.digest()


def test_structure_rules(gen):
    _, sc = gen
    ci, pi = sc.cam_index, sc.pt_index
    assert ci.dtype == np.int64 and pi.dtype == np.int64
    assert sc.n_observations > 2 * sc.n_points >= 2
    # point-major, cameras strictly increasing inside a point (no duplicates)
    key = pi * sc.n_cameras + ci
    assert np.all(np.diff(key) > 0)
    assert np.bincount(pi, minlength=sc.n_points).min() >= 2
    assert np.bincount(ci, minlength=sc.n_cameras).min() >= 1
    assert pi.max() == sc.n_points - 1 and ci.max() == sc.n_cameras - 1


def test_pixels_are_truth_projection_plus_unit_noise(gen):
    from oracle import bamg_oracle as O  # checker only

    _, sc = gen
    truth = O.Problem(sc.truth_cameras.copy(), sc.truth_points, sc.cam_index, sc.pt_index, sc.pixels)
    c = sc.truth_cameras[sc.cam_index]
    pc = O.rotate(c[:, :3], sc.truth_points[sc.pt_index]) + c[:, 3:6]
    depth = -pc[:, 2]
    assert depth.min() >= 1.0  # scenes._finish: depth >= 1, |p| <= 2 at the truth
    assert np.max(np.sum((pc[:, :2] / depth[:, None]) ** 2, axis=1)) <= 4.0 + 1e-9
    obj, jac = O.evaluate(truth, with_jacobian=True)[:2]
    r = np.asarray(jac.r).reshape(-1)
    assert abs(r.mean()) < 0.02
    assert abs(r.std() - 1.0) < 0.02
    assert np.isclose(obj, np.sum(r * r), rtol=1e-12)  # problem.py:179-188 trivial loss
    assert np.all(sc.truth_cameras[:, 6] == 500.0)
    assert 0.007 < sc.truth_cameras[:, 7].std() < 0.013 and 0.007 < sc.truth_cameras[:, 8].std() < 0.013


def test_start_is_a_small_centre_preserving_perturbation(gen):
    from scipy.spatial.transform import Rotation

    from oracle import bamg_oracle as O

    _, sc = gen
    Rt = Rotation.from_rotvec(sc.truth_cameras[:, :3])
    R0 = Rotation.from_rotvec(sc.camera_params[:, :3])
    ang = (R0 * Rt.inv()).magnitude()
    assert 0.012 < ang.mean() < 0.020  # |N(0, 1e-2 I_3)| has mean 1.6e-2
    c_t = -Rt.inv().apply(sc.truth_cameras[:, 3:6])
    c_0 = -R0.inv().apply(sc.camera_params[:, 3:6])
    d = c_0 - c_t
    assert 0.008 < d.std() < 0.012
    dp = sc.points - sc.truth_points
    assert 0.048 < dp.std() < 0.052
    assert np.all(np.linalg.norm(sc.camera_params[:, :3], axis=1) <= np.pi + 1e-12)
    # the start evaluates: nothing behind a camera (problem.py:211-213)
    O.evaluate(O.Problem.of(sc), with_jacobian=False)


def test_visibility_model(gen):
    from scipy.spatial.transform import Rotation

    n, sc = gen
    cnt = np.bincount(sc.pt_index, minlength=sc.n_points)
    centres = -Rotation.from_rotvec(sc.truth_cameras[:, :3]).inv().apply(sc.truth_cameras[:, 3:6])
    d_xy = np.linalg.norm(centres[sc.cam_index, :2] - sc.truth_points[sc.pt_index, :2], axis=1)
    if n == 3:
        assert d_xy.max() <= 15.0
        assert 3.0 < cnt.mean() < 6.5  # 2 + Poisson(4), cut by the candidate filters
    elif n == 4:
        assert d_xy.max() <= 60.0
        assert 5.5 < cnt.mean() < 6.7  # 2 + Poisson(4.5) = 6.5 requested
        assert cnt.max() <= 32
    else:
        # runs of consecutive cameras 7-10 behind the point, plus ~0.5% bridges 51-100 behind
        first = np.r_[0, np.cumsum(cnt)[:-1]]
        span = np.empty(sc.n_points, np.int64)
        for p in range(0, sc.n_points, max(1, sc.n_points // 2000)):
            cams = np.sort(sc.cam_index[first[p]:first[p] + cnt[p]])
            gaps = np.diff(np.r_[cams, cams[0] + sc.n_cameras])
            span[p] = sc.n_cameras - gaps.max()  # shortest arc holding all of them
        sampled = span[::max(1, sc.n_points // 2000)]
        assert np.mean(sampled <= 40) > 0.98
        assert 2.5 < cnt.mean() < 4.5  # 2 + geometric(0.5), mean 4, cut by the filters


def test_matches_numpy_generator_statistics():
    """Same parameters through scenes.city (numpy) and the device generator: the
    per-point camera counts agree in distribution (different random streams)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2007_01941_b200 import scenes

    host = scenes.city(seed=1, n_cameras=400, n_points=20_000, side=63.0)
    dev = scenes.device_config(3, seed=1, **SMALL[3]).to_host()
    ch = np.bincount(host.pt_index)
    cd = np.bincount(dev.pt_index)
    assert abs(ch.mean() - cd.mean()) < 0.06 * ch.mean()
    assert abs(host.n_points - dev.n_points) < 0.03 * host.n_points
    hh = np.bincount(ch, minlength=20)[:20] / len(ch)
    hd = np.bincount(cd, minlength=20)[:20] / len(cd)
    assert np.abs(hh - hd).max() < 0.02


def test_config4_full_size_on_device_solves():
    """BASELINE config 4 generated in HBM and fed to the solver without a host copy:
    ~4.5 M points, ~29 M observations, S inside the [2 M, 3 M] block band, and the
    multigrid PCG of one LM linear solve converges like on the numpy scene."""
    import time

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P
    from paper_2007_01941_b200 import scenes

    scenes.device_config(3, seed=0, **SMALL[3])  # warm the library
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sc = scenes.device_config(4, seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"config 4 on device: {sc.n_cameras} cameras, {sc.n_points} points, {sc.n_observations} obs in {dt:.3f} s")
    assert sc.n_cameras == 13_000
    assert 4.4e6 < sc.n_points <= 4.5e6
    assert 27e6 < sc.n_observations < 31e6
    assert dt < 5.0  # the numpy generator takes ~25 s
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, cg_max_iterations=200, cg_residual_tolerance=1e-6)
    obj, jac = P.evaluate(prob)
    dc, dp, cg, sys_, *_ = P.solver.linear_solve(prob, jac, 1e4, cfg)
    S = sys_.ensure_explicit()
    assert 2.0e6 < S.blocks.shape[0] < 3.0e6
    assert cg.iterations <= 30 and cg.relative_residual <= 1e-6


@pytest.mark.parametrize("n, pts_band, obs_band", [(3, (0.93e6, 1.0e6), (4.6e6, 5.7e6)), (5, (1.95e6, 2.0e6), (7.5e6, 8.5e6))])
def test_configs_3_and_5_full_size_on_device_solve(n, pts_band, obs_band):
    """BASELINE configs 3 and 5 at full size from the device generator: sizes next to the
    numpy scenes' (977 k points / 5.12 M observations; 2.0 M / 8.0 M) and the multigrid
    PCG of the first LM linear solve converges within the numpy scenes' counts + 3."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P
    from paper_2007_01941_b200 import scenes

    sc = scenes.device_config(n, seed=0)
    assert pts_band[0] < sc.n_points <= pts_band[1], sc.n_points
    assert obs_band[0] < sc.n_observations < obs_band[1], sc.n_observations
    prob = P.BundleProblem(*sc.arrays())
    cfg = P.SolveConfig(preconditioner="multigrid", tau=1e-30, cg_max_iterations=200, cg_residual_tolerance=1e-6)
    obj, jac = P.evaluate(prob)
    dc, dp, cg, *_ = P.solver.linear_solve(prob, jac, 1e4, cfg)
    assert cg.relative_residual <= 1e-6
    assert cg.iterations <= {3: 15, 5: 27}[n] + 3, cg.iterations
