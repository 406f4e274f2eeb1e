"""The three device schedules of T -- CTA-granular dataflow ("fused"), warp-
granular streaming dataflow ("wide") and per-stage launches ("stages") -- each
against the CPU oracle's apply_T (proj/src/solver.cpp:148-164) on the same
problem, alpha and random (z, eta).  GPU only."""
import contextlib
import os

import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.rng import Philox
from support import TinyOpts, make_tiny

pytestmark = pytest.mark.gpu

_ENV = {
    "fused": {"SPOCK_T_FUSED": "1"},
    "wide": {"SPOCK_T_UNFUSED": "1", "SPOCK_T_WIDE": "1"},
    "stages": {"SPOCK_T_UNFUSED": "1", "SPOCK_T_WIDE": "0"},
}
_KEYS = ("SPOCK_T_FUSED", "SPOCK_T_UNFUSED", "SPOCK_T_WIDE", "SPOCK_WIDE_WARPS", "SPOCK_WIDE_SLOTS",
         "SPOCK_WIDE_CHUNK")


@contextlib.contextmanager
def path_env(path, **extra):
    old = {k: os.environ.get(k) for k in _KEYS}
    try:
        for k in _KEYS:
            os.environ.pop(k, None)
        os.environ.update(_ENV[path])
        os.environ.update({k: str(v) for k, v in extra.items()})
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _solver(p, path, params=None, **extra):
    from paper_2505_12078_b200.solver import SpockSolver
    with path_env(path, **extra):
        s = SpockSolver(p, **(params or {}))
    assert s.t_path == path, (s.t_path, path)
    return s


def _rand(n, seed):
    return -1.0 + 2.0 * Philox(seed).uniform_array(n)


def _problems():
    yield "binary-2x2", make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 31, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    yield "mixed-3-1-2", make_tiny(ScenarioTree.from_branching([3, 1, 2]), 3, 2, 5, TinyOpts(gamma=0.3))
    yield "expectation", make_tiny(ScenarioTree.from_branching([2, 3]), 3, 2, 7, TinyOpts(gamma=1.0))
    yield "avar-at-one", make_tiny(ScenarioTree.from_branching([2, 2]), 2, 2, 9,
                                   TinyOpts(gamma=1.0, avar_form_at_one=True))
    yield "rank-deficient-Q", make_tiny(ScenarioTree.from_branching([2, 2, 2]), 4, 2, 11,
                                        TinyOpts(gamma=0.7, q_rank_deficient_prob=0.6, box_halfwidth=0.5))
    yield "fan-out-40", make_tiny(ScenarioTree.from_branching([40, 1]), 3, 2, 13, TinyOpts(gamma=0.4))
    yield "c1", make_config("c1", seed=1)


PROBLEMS = list(_problems())


@pytest.mark.parametrize("path", ["fused", "wide", "stages"])
@pytest.mark.parametrize("name,p", PROBLEMS, ids=[n for n, _ in PROBLEMS])
def test_T_matches_oracle(path, name, p):
    g = _solver(p, path)
    o = OracleSolver(p, alpha=g.alpha)
    for seed in (3, 4):
        z = _rand(g.nz, seed)
        e = _rand(g.neta, seed + 100)
        zg, eg = g.apply_T(z, e)
        zo, eo = o.apply_T(z, e)
        sz = max(1.0, float(np.abs(zo).max()))
        se = max(1.0, float(np.abs(eo).max()))
        assert float(np.abs(zg - zo).max()) <= 1e-11 * sz, name
        assert float(np.abs(eg - eo).max()) <= 1e-11 * se, name


@pytest.mark.parametrize("warps,slots,chunk", [(4, 3, 2048), (1, 1, 512), (8, 2, 1024), (3, 5, 600)])
def test_wide_ring_configurations(warps, slots, chunk):
    """Chunking across item boundaries, single-slot rings and odd chunk sizes
    give the same T (the ring is pure data movement)."""
    p = make_config("c2", seed=2)
    g = _solver(p, "wide", SPOCK_WIDE_WARPS=warps, SPOCK_WIDE_SLOTS=slots, SPOCK_WIDE_CHUNK=chunk)
    o = OracleSolver(p, alpha=g.alpha)
    z = _rand(g.nz, 21)
    e = _rand(g.neta, 22)
    zg, eg = g.apply_T(z, e)
    zo, eo = o.apply_T(z, e)
    assert float(np.abs(zg - zo).max()) <= 1e-10 * max(1.0, float(np.abs(zo).max()))
    assert float(np.abs(eg - eo).max()) <= 1e-10 * max(1.0, float(np.abs(eo).max()))


def test_wide_bitwise_deterministic_and_equal_to_stages_on_c2p():
    p = make_config("c2p", seed=1)
    w = _solver(p, "wide")
    s = _solver(p, "stages")
    assert w.alpha == s.alpha
    z = _rand(w.nz, 5)
    e = _rand(w.neta, 6)
    a1 = w.apply_T(z, e)
    a2 = w.apply_T(z, e)
    assert np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1])
    b = s.apply_T(z, e)
    np.testing.assert_allclose(a1[0], b[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a1[1], b[1], rtol=1e-12, atol=1e-12)


def test_wide_cp_trace_matches_oracle():
    p = make_tiny(ScenarioTree.from_branching([3, 2]), 3, 2, 17, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    g = _solver(p, "wide", params=dict(max_iters=25, eps_abs=1e-14, eps_rel=1e-14))
    o = OracleSolver(p, alpha=g.alpha, max_iters=25, eps_abs=1e-14, eps_rel=1e-14)
    a, b = g.solve(), o.solve()
    assert a.status["branches"] == b.status["branches"]
    np.testing.assert_allclose(a.status["rnorm_history"], b.status["rnorm_history"], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(a.z_scaled, b.z_scaled, rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("lop", ["wide", "lop", "cta"])
@pytest.mark.parametrize("name,p", PROBLEMS[:3] + PROBLEMS[-2:], ids=[n for n, _ in PROBLEMS[:3] + PROBLEMS[-2:]])
def test_standalone_L_Lt_all_schedules(lop, name, p):
    """TreeOperator::apply / apply_adjoint (tree_operator.cpp:20-114) on the
    streaming kernel (wide.cu), the one-shot CTA-per-node kernels (lop.cu) and
    narrow.cu's CTA-per-node kernels."""
    from paper_2505_12078_b200.solver import SpockSolver
    env = {"wide": {"SPOCK_LOP_WIDE": "1"}, "lop": {"SPOCK_LOP_WIDE": "0"},
           "cta": {"SPOCK_LOP_WIDE": "0", "SPOCK_LOP_NARROW": "0"}}[lop]
    old = {k: os.environ.get(k) for k in ("SPOCK_LOP_WIDE", "SPOCK_LOP_NARROW")}
    os.environ.update(env)
    try:
        g = SpockSolver(p)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    o = OracleSolver(p, alpha=g.alpha)
    for seed in (8, 11):
        z = _rand(g.nz, seed)
        e = _rand(g.neta, seed + 1)
        le, lo_ = g.apply_L(z), o.apply_L(z)
        te, to_ = g.apply_Lt(e), o.apply_Lt(e)
        assert float(np.abs(le - lo_).max()) <= 1e-12 * max(1.0, float(np.abs(lo_).max()))
        assert float(np.abs(te - to_).max()) <= 1e-12 * max(1.0, float(np.abs(to_).max()))
