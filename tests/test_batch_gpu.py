"""Concurrent multi-x_init solves (BatchSolver): every result is
bitwise the sequential SpockSolver result for the same x_init (and warm
start), with the fused T launch capped to a share of the SMs.  GPU only."""
import numpy as np
import pytest

from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.problem import ScenarioTree
from support import TinyOpts, make_tiny

pytestmark = pytest.mark.gpu


def _x_inits(p, n, seed=5):
    rng = np.random.default_rng(seed)
    return [p.x_init * (1.0 + 0.3 * rng.standard_normal(p.x_init.shape)) for _ in range(n)]


def _same(a, b):
    assert a.status["iterations"] == b.status["iterations"]
    assert a.status["reason"] == b.status["reason"]
    assert a.status["branches"] == b.status["branches"]
    np.testing.assert_array_equal(a.z, b.z)
    np.testing.assert_array_equal(a.eta, b.eta)


@pytest.mark.parametrize("algo", ["solve", "solve_cp"])
@pytest.mark.parametrize("name,streams", [("tiny", 3), ("c2p", 2)])
def test_batch_matches_sequential(name, streams, algo):
    from paper_2505_12078_b200.solver import BatchSolver, SpockSolver
    if name == "tiny":
        p = make_tiny(ScenarioTree.from_branching([2, 2, 1]), 3, 2, 7, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    else:
        p = make_config(name, seed=2)
    kw = dict(max_iters=300, eps_abs=1e-9, eps_rel=1e-9)
    xs = _x_inits(p, 5)
    b = BatchSolver(p, streams=streams, **kw)
    assert len(b.solvers) == streams
    got = getattr(b, algo)(xs)
    ref = SpockSolver(p, **kw)
    full = ref.grid
    if b.solvers[0].t_path == "fused" and streams > 1:
        assert 0 < b.solvers[0].grid <= max(16, full // streams)
    for x, g in zip(xs, got):
        _same(g, getattr(ref, algo)(x))


def test_batch_warm_start():
    from paper_2505_12078_b200.solver import BatchSolver, SpockSolver
    p = make_tiny(ScenarioTree.from_branching([3, 1]), 2, 1, 11, TinyOpts(gamma=0.4, box_halfwidth=2.0))
    kw = dict(max_iters=200, eps_abs=1e-8, eps_rel=1e-8)
    ref = SpockSolver(p, **kw)
    xs = _x_inits(p, 4, seed=9)
    warm = [(r.z_scaled, r.eta) for r in (ref.solve(x) for x in xs)]
    b = BatchSolver(p, streams=2, **kw)
    got = b.solve(xs[::-1], warm=warm[::-1])
    for x, w, g in zip(xs[::-1], warm[::-1], got):
        _same(g, ref.solve(x, warm=w))


def test_grid_cap_after_solve_rejected():
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_tiny(ScenarioTree.from_branching([2]), 2, 1, 3, TinyOpts())
    s = SpockSolver(p, max_iters=5)
    s.set_grid_cap(8)
    s.solve()
    with pytest.raises(ValueError):
        s.set_grid_cap(4)


@pytest.mark.parametrize("algo", ["solve", "solve_cp"])
def test_batch_matches_oracle(algo):
    """Every x_init of a batch against the CPU oracle's solve from the same
    x_init (solver.cpp:176-187): same branch string and iteration count over a
    short run, traces and iterates to rounding."""
    from oracle.oracle import OracleSolver
    from paper_2505_12078_b200.solver import BatchSolver
    p = make_tiny(ScenarioTree.from_branching([2, 2, 1]), 3, 2, 7, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    kw = dict(max_iters=25, eps_abs=1e-14, eps_rel=1e-14)
    xs = _x_inits(p, 4, seed=13)
    b = BatchSolver(p, streams=2, **kw)
    got = getattr(b, algo)(xs)
    o = OracleSolver(p, alpha=b.solvers[0].alpha, **kw)
    for x, g in zip(xs, got):
        r = getattr(o, algo)(x)
        assert g.status["branches"] == r.status["branches"]
        assert g.status["iterations"] == r.status["iterations"]
        np.testing.assert_allclose(g.status["rnorm_history"], r.status["rnorm_history"], rtol=1e-8, atol=1e-12)
        np.testing.assert_allclose(g.z, r.z, rtol=1e-7, atol=1e-9)
