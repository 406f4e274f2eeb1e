"""Default-schedule T, L and L* against the CPU oracle on the configurations
that carry the bench numbers: c2 and c2p on the CTA
dataflow kernel, c3 and c4 on the streaming kernel, and two ~1e5-node shapes of
the tree-structure sweep (BASELINE configs[3]) -- a 100-way fan-out (12, 100, 2)
and a 100-stage horizon (100, 10, 3).  Every instance is per-node perturbed
(SURVEY §8d): each node's A, B, Q, R differ, so a kernel reading another node's
block of the same event cannot pass.  GPU only; the oracle's setup dominates the
run time (minutes at 1e5 nodes)."""
import os

import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.rng import Philox

pytestmark = pytest.mark.gpu

CASES = [
    ("c2", "c2", {}, "fused"),
    ("c2p", "c2p", {}, "fused"),
    ("c3", "c3", {}, "wide"),
    ("c4", "c4", {}, "wide"),
    ("shape-12-100-2", "c4", dict(N=12, nw=100, nb=2), "wide"),
    ("shape-100-10-3", "c4", dict(N=100, nw=10, nb=3), "wide"),
    ("c5p", "c5p", {}, "wide"),  # n_x = 100, n_u = 50 (the c5 state size): 5 row groups per lane
]
TOL = 1e-10  # relative to the output's max |entry|: fp64, different (fixed) summation orders


def _rand(n, seed):
    return -1.0 + 2.0 * Philox(seed).uniform_array(n)


def _close(got, ref, what):
    sc = max(1.0, float(np.abs(ref).max()))
    err = float(np.abs(got - ref).max())
    assert err <= TOL * sc, f"{what}: max |diff| {err:.3e} (scale {sc:.3e})"
    return err / sc


@pytest.mark.parametrize("name,cfg,over,path", CASES, ids=[c[0] for c in CASES])
def test_default_schedule_matches_oracle(name, cfg, over, path):
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config(cfg, seed=1, **over)
    assert p.meta["perturb"] > 0.0
    g = SpockSolver(p)
    assert g.t_path == path, (name, g.t_path)
    os.environ["ORACLE_SKIP_NORM"] = "1"  # alpha is given: the oracle's power iteration is not read
    try:
        o = OracleSolver(p, alpha=g.alpha)
    finally:
        os.environ.pop("ORACLE_SKIP_NORM", None)
    z = _rand(g.nz, 41)
    e = _rand(g.neta, 42)
    zg, eg = g.apply_T(z, e)
    zo, eo = o.apply_T(z, e)
    rz = _close(zg, zo, f"{name} T z")
    re_ = _close(eg, eo, f"{name} T eta")
    _close(g.apply_L(z), o.apply_L(z), f"{name} L")
    _close(g.apply_Lt(e), o.apply_Lt(e), f"{name} L*")
    # a second application from the first's output (iterates, not random data)
    zg2, eg2 = g.apply_T(zo, eo)
    zo2, eo2 = o.apply_T(zo, eo)
    _close(zg2, zo2, f"{name} T^2 z")
    _close(eg2, eo2, f"{name} T^2 eta")
    print(f"{name}: nodes {p.tree.num_nodes()} path {g.t_path} rel err z {rz:.1e} eta {re_:.1e}")


def test_pooled_blocks_bitwise_equal_per_node():
    """Shared-matrix instance (the generator's per-event A, B, Q, R, perturbation
    off): the streaming kernel's records point every node at its class
    representative's blocks (Engine::compute_pool).  T, L and L* are bitwise
    those of the per-node records (SPOCK_POOL=0) and match the oracle."""
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config("c2p", seed=1, perturb=0.0)
    env = {"SPOCK_T_UNFUSED": "1", "SPOCK_T_WIDE": "1", "SPOCK_LOP_WIDE": "1"}
    out = {}
    for pool in ("1", "0"):
        old = {k: os.environ.get(k) for k in list(env) + ["SPOCK_POOL"]}
        os.environ.update(env)
        os.environ["SPOCK_POOL"] = pool
        try:
            g = SpockSolver(p)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        assert g.t_path == "wide"
        z = _rand(g.nz, 41)
        e = _rand(g.neta, 42)
        out[pool] = (g.apply_T(z, e), g.apply_L(z), g.apply_Lt(e), g.alpha, z, e)
    (za, ea), la, lta, alpha, z, e = out["1"]
    (zb, eb), lb, ltb, _, _, _ = out["0"]
    assert np.array_equal(za, zb) and np.array_equal(ea, eb)
    assert np.array_equal(la, lb) and np.array_equal(lta, ltb)
    os.environ["ORACLE_SKIP_NORM"] = "1"
    try:
        o = OracleSolver(p, alpha=alpha)
    finally:
        os.environ.pop("ORACLE_SKIP_NORM", None)
    zo, eo = o.apply_T(z, e)
    _close(za, zo, "pooled T z")
    _close(ea, eo, "pooled T eta")


@pytest.mark.parametrize("method", ["solve", "solve_cp"])
def test_nx100_solve_trace_matches_oracle(method):
    """The c5 state size (n_x 100, n_u 50; c5p, 9 557 nodes) through a whole
    device-resident solve against the oracle's: branch strings, iteration
    counts and ||r||_M traces over a short run (solver.cpp:189-350, 182-187)."""
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config("c5p", seed=1)
    kw = dict(max_iters=8, eps_abs=1e-14, eps_rel=1e-14)
    g = SpockSolver(p, **kw)
    assert g.t_path == "wide" and g.loop_path == "graph"
    os.environ["ORACLE_SKIP_NORM"] = "1"
    try:
        o = OracleSolver(p, alpha=g.alpha, **kw)
    finally:
        os.environ.pop("ORACLE_SKIP_NORM", None)
    a, b = getattr(g, method)(p.x_init), getattr(o, method)(p.x_init)
    assert a.status["branches"] == b.status["branches"]
    assert a.status["iterations"] == b.status["iterations"] == 8
    np.testing.assert_allclose(a.status["rnorm_history"], b.status["rnorm_history"], rtol=1e-9, atol=1e-12)
    sc = max(1.0, float(np.abs(b.z).max()))
    assert float(np.abs(a.z - b.z).max()) <= 1e-8 * sc
