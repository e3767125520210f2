"""B200-native LM linear-solve path of arXiv 2007.01941 (multigrid bundle adjustment).

Drop-in for the hot-path names of the reference package `bamg`
(`pkg/src/bamg/__init__.py:3-95`): problem / schur / blockmat / multigrid /
precond / solver, with the arithmetic in hand-written sm_100a kernels
(libbamg_b200.so, C ABI in include/bamg_b200.h). Array results are CUDA tensors.
Submodules import lazily so that `import paper_2007_01941_b200` works on a host
without a GPU (the build check); any compute call then fails loudly.
"""

from __future__ import annotations

import importlib

_EXPORTS = {
    "balio": ["BalFormatError", "read_bal", "write_bal", "read_bal_arrays", "write_bal_arrays"],
    "blockmat": ["BlockDiagMatrix", "BlockSparseMatrix", "DenseTall", "IndefiniteBlockError", "multiply",
                 "triple_product", "write_matrix_market"],
    "multigrid": ["Aggregation", "ChebyshevSmoother", "MgHierarchy", "StrengthMatrix", "aggregate", "build_hierarchy",
                  "build_prolongation", "estimate_lambda_max", "hierarchy_stats", "mgcycle", "operator_strength",
                  "visibility_strength", "make_smoother"],
    "precond": ["DEFAULT_CLUSTER_CAP", "PointBlockJacobi", "pbj_setup", "VisibilityJacobi", "visibility_cluster",
                "vj_setup"],
    "problem": ["CAMERA_SIZE", "POINT_SIZE", "BehindCameraError", "BundleProblem", "JacobianBlocks", "evaluate",
                "gauge_nullspace", "huber", "loss_value", "loss_weight"],
    "schur": ["Damping", "SchurSystem", "back_substitute", "build_system", "choose_mode",
              "covisibility_block_count", "model_decrease", "schur_explicit"],
    "solver": ["CgDivergence", "CgReport", "ForcingCriterion", "IterationRecord", "NonlinearReport",
               "PreconditionerNotSPD", "SolveConfig", "TrustRegion", "lm_solve", "pcg"],
}
_WHERE = {name: mod for mod, names in _EXPORTS.items() for name in names}

__all__ = sorted(_WHERE) + list(_EXPORTS)
__version__ = "0.1.0"


def __getattr__(name):
    if name in _WHERE:
        return getattr(importlib.import_module(f".{_WHERE[name]}", __name__), name)
    if name in _EXPORTS or name in ("scenes", "build", "_lib", "_device"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
