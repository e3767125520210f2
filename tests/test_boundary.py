"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/bamg_b200.h declares; the product never touches the oracle;
the package mirrors the reference's hot-path names."""

import ast
import ctypes
import os
import re

import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2007_01941_b200")


def test_library_exports_every_header_symbol():
    from paper_2007_01941_b200 import _lib

    protos = _lib.parse_header()
    assert len(protos) >= 50
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in protos if not hasattr(L, n)]
    assert not missing, missing
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (bamg_\w+)", out))
    assert exported == set(protos), exported ^ set(protos)


def test_library_loads_and_reports_version():
    from paper_2007_01941_b200 import _lib

    assert _lib.lib().bamg_version() == 1
    assert isinstance(_lib.last_error(), str)


def test_tridiagonal_eigen_host_helper():
    import numpy as np
    import scipy.linalg

    from paper_2007_01941_b200 import _lib

    rng = np.random.default_rng(0)
    for n in range(1, 6):
        a = rng.normal(size=n) + 3
        b = rng.uniform(0.1, 1, size=max(n - 1, 1))
        got = _lib.lib().bamg_tridiag_max_eig(a.ctypes.data, b.ctypes.data, n)
        want = scipy.linalg.eigh_tridiagonal(a, b[: n - 1], eigvals_only=True)[-1]
        assert abs(got - want) <= 1e-13 * max(1.0, abs(want))


def test_product_does_not_import_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    names = [a.name for a in node.names]
                elif isinstance(node, ast.ImportFrom):
                    names = [node.module or ""]
                else:
                    continue
                assert not any(n.split(".")[0] == "oracle" for n in names), (f, names)
                assert not any("bamg" == n.split(".")[0] for n in names), (f, names)


def test_reference_names_mirrored():
    import paper_2007_01941_b200 as P

    for name in ["BundleProblem", "evaluate", "gauge_nullspace", "Damping", "build_system", "schur_explicit",
                 "choose_mode", "back_substitute", "model_decrease", "visibility_strength", "operator_strength",
                 "aggregate", "build_prolongation", "estimate_lambda_max", "build_hierarchy", "mgcycle",
                 "pbj_setup", "pcg", "lm_solve", "SolveConfig", "BlockSparseMatrix", "BlockDiagMatrix",
                 "IndefiniteBlockError", "BehindCameraError", "PreconditionerNotSPD", "CgDivergence"]:
        assert name in P.__all__, name


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2007_01941_b200 import _lib, problem

    with pytest.raises(_lib.NativeError):
        problem.BundleProblem([[0.0] * 9], [[0.0, 0.0, 1.0]], [0], [0], [[0.0, 0.0]])


def test_device_scene_arguments_checked_before_any_gpu_work():
    """scenes.device_config validates the configuration number and parameter names on
    the host (no CUDA needed for that), and the scene entry points are exported."""
    import ctypes

    import pytest

    from paper_2007_01941_b200 import _lib, scenes

    with pytest.raises(ValueError):
        scenes.device_config(2)
    with pytest.raises(TypeError):
        scenes.device_config(4, n_camera=10)
    L = _lib.lib()
    for name in ("bamg_scene_grid_cells", "bamg_scene_layout", "bamg_scene_visibility", "bamg_scene_emit"):
        assert hasattr(L, name)
    # the grid-size helper is pure host code: city defaults -> ceil(200 / 15) + 1 cells a side
    p = (ctypes.c_double * 8)(200.0, 1, 0, 0, 20.0, 4.0, 15.0, 0.0)
    assert L.bamg_scene_grid_cells(3, 4000, 1_000_000, ctypes.addressof(p)) == 15 * 15
    assert L.bamg_scene_grid_cells(7, 4000, 1_000_000, ctypes.addressof(p)) == -1
