"""Side-by-side parity of the B200 solver against the CPU oracle (same
problem, same alpha): per-iteration ||r||_M traces, branch sequences and final
iterates.  GPU only."""
import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_2505_12078_b200.problem import ScenarioTree
from support import TinyOpts, make_tiny

pytestmark = pytest.mark.gpu


def _pair(p, **kw):
    from paper_2505_12078_b200.solver import SpockSolver
    g = SpockSolver(p, **kw)
    o = OracleSolver(p, alpha=g.alpha, **kw)
    return g, o


@pytest.mark.parametrize("k", [1, 2, 5, 30])
def test_cp_iterates_match_oracle(k):
    p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 31, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    g, o = _pair(p, max_iters=k, eps_abs=1e-14, eps_rel=1e-14)
    a, b = g.solve_cp(), o.solve_cp()
    assert a.status["iterations"] == b.status["iterations"] == k
    np.testing.assert_allclose(a.status["rnorm_history"], b.status["rnorm_history"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(a.z_scaled, b.z_scaled, rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(a.eta, b.eta, rtol=1e-9, atol=1e-10)
    assert a.status["xi1_inf"] == pytest.approx(b.status["xi1_inf"], rel=1e-7)
    assert a.status["xi2_inf"] == pytest.approx(b.status["xi2_inf"], rel=1e-7)


@pytest.mark.parametrize("k", [1, 3, 6, 20])
def test_supermann_iterates_match_oracle(k):
    p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 31, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    g, o = _pair(p, max_iters=k, eps_abs=1e-14, eps_rel=1e-14)
    a, b = g.solve(), o.solve()
    assert a.status["branches"] == b.status["branches"]
    np.testing.assert_allclose(a.status["rnorm_history"], b.status["rnorm_history"], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(a.z_scaled, b.z_scaled, rtol=1e-7, atol=1e-9)
