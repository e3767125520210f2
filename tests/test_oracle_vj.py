"""Pin the oracle's visibility block-Jacobi restatement (precond.py:59-144) against
fixtures from the real reference (oracle/make_golden_vj.py). CPU only."""

import numpy as np
import pytest

from conftest import VJ_CASES, golden, relerr, vj_inputs
from oracle import bamg_oracle as O


@pytest.fixture(scope="module")
def g():
    return golden("vj_cases")


@pytest.mark.parametrize("tag", VJ_CASES)
def test_vj_oracle_matches_reference(g, tag):
    prob = O.Problem(*[np.array(a, copy=True) for a in vj_inputs(tag, g)])
    prob.cams[:, :3] = O.canonicalize(prob.cams[:, :3])
    obj, jac = O.evaluate(prob)
    s = O.build_system(jac, O.damping(jac, 1e4))
    s.mode = O.choose_mode(s)
    G = O.visibility_strength(prob.ci, prob.pi, prob.nc, prob.npt)
    for cap in (100, 6):
        agg, n = O.visibility_cluster(G, cap)
        np.testing.assert_array_equal(agg, g[f"{tag}_cap{cap}_assign"])
        assert n == int(g[f"{tag}_cap{cap}_n"])
        M = O.vj(s, agg, n)  # S not assembled: the accumulated route
        for v, want in zip(g[f"{tag}_vin"], g[f"{tag}_cap{cap}_vout"]):
            assert relerr(M(v), want) <= 1e-10
        x, rep = O.pcg(s.matvec, M, s.rhs, 1e-30, 20000, 1e-6)
        assert abs(rep.iterations - int(g[f"{tag}_cap{cap}_pcg_its"])) <= 1
    s.explicit()
    agg, n = O.visibility_cluster(G)
    M = O.vj(s, agg, n)  # assembled route
    assert relerr(M(g[f"{tag}_vin"][0]), g[f"{tag}_cap100_vout"][0]) <= 1e-10


def test_vj_oracle_lm(g):
    tag = "r1003"
    prob = O.Problem(*[np.array(a, copy=True) for a in vj_inputs(tag, g)])
    prob.cams[:, :3] = O.canonicalize(prob.cams[:, :3])
    cams, pts, recs, term = O.lm_solve(prob, preconditioner="visibility")
    cg = np.array([r.cg_iterations for r in recs])
    assert np.all(np.abs(cg - g[f"{tag}_lm_cg"]) <= 1)
    np.testing.assert_array_equal([r.accepted for r in recs], g[f"{tag}_lm_accepted"])
    assert abs(recs[-1].objective - g[f"{tag}_lm_obj"][-1]) <= 1e-8 * abs(g[f"{tag}_lm_obj"][-1])
