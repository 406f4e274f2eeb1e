"""Setup KATs: SOC epigraph data and preconditioning (proj/tests/test_problem.cpp)."""
import numpy as np
import pytest

from oracle import oracle
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.rng import Philox
from support import TinyOpts, make_tiny


def _G(d, z, tau):
    p = d["p"]
    g = np.zeros(p + 2)
    if p > 0:
        g[:p] = d["head_map"] @ z
    row = 0.5 * tau - 0.5 * d["q_kernel"] @ z
    g[p] = g[p + 1] = row
    return g


def _member(d, z, tau, tol=0.0):
    v = _G(d, z, tau) - d["a"]
    p = d["p"]
    return np.linalg.norm(v[:p + 1]) <= v[p + 1] + tol


def test_scalar_q1():  # test_problem.cpp:22-33
    d = oracle.soc_data_quadlin(np.ones((1, 1)), np.zeros(1))
    assert d["p"] == 1
    np.testing.assert_allclose(d["a"], [0.0, 0.5, -0.5], atol=1e-15)
    g = _G(d, np.ones(1), 1.0) - d["a"]
    assert np.linalg.norm(g[:2]) == pytest.approx(g[2], rel=1e-14)
    assert _member(d, np.ones(1), 1.0, 1e-12)
    assert not _member(d, np.ones(1), 1.0 - 1e-6)


def test_vanishing_linear_term():  # test_problem.cpp:35-48
    rng = Philox(5)
    for _ in range(10):
        n = rng.uniform_int(1, 4)
        M = rng.normal_matrix(n, n, 0.0, 1.0)
        d = oracle.soc_data_quadlin(M @ M.T + 0.1 * np.eye(n), np.zeros(n))
        assert d["p"] == n
        assert np.abs(d["a"][:n]).max() < 1e-14
        assert d["a"][n] == pytest.approx(0.5) and d["a"][n + 1] == pytest.approx(-0.5)


def test_q4_q2():  # test_problem.cpp:50-63
    d = oracle.soc_data_quadlin(4.0 * np.ones((1, 1)), 2.0 * np.ones(1))
    assert d["sqrt_factor"][0, 0] == pytest.approx(2.0)
    np.testing.assert_allclose(d["a"], [-0.5, 0.375, -0.625])
    g = _G(d, np.zeros(1), 0.0) - d["a"]
    np.testing.assert_allclose(g, [0.5, -0.375, 0.625])
    assert np.linalg.norm(g[:2]) == pytest.approx(g[2], rel=1e-14)


def test_zero_q_linear_epigraph():  # test_problem.cpp:65-70
    d = oracle.soc_data_quadlin(np.zeros((2, 2)), np.array([1.0, -1.0]))
    assert d["p"] == 0
    assert _member(d, np.array([1.0, 2.0]), -0.999, 1e-9)
    assert not _member(d, np.array([1.0, 2.0]), -1.001)


def test_epigraph_membership_500_samples():  # test_problem.cpp:72-88
    rng = Philox(9)
    checked = 0
    for _ in range(500):
        n = rng.uniform_int(1, 4)
        deficient = rng.uniform() < 0.4
        M = rng.normal_matrix(n, n, 0.0, 1.0)
        if deficient and n > 1:
            drop = rng.uniform_int(1, n - 1)
            M[:, n - drop:] = 0.0
        Q = M @ M.T
        q = rng.uniform_vector(n, -2.0, 2.0)
        d = oracle.soc_data_quadlin(Q, q)
        z = rng.uniform_vector(n, -2.0, 2.0)
        tau = rng.uniform(-3.0, 8.0)
        ell = z @ Q @ z + q @ z
        if abs(ell - tau) <= 1e-9 * max(1.0, abs(tau)):
            continue
        assert _member(d, z, tau, 1e-9) == (ell <= tau)
        checked += 1
    assert checked > 450


def test_identity_problem_unchanged_by_preconditioning():  # test_problem.cpp:151-170
    tree = ScenarioTree.from_branching([1, 1])
    p = make_tiny(tree, 2, 1, 42, TinyOpts(box_halfwidth=1.0))
    p.Q[:] = np.eye(2)
    p.R[:] = np.eye(1)
    p.QN[0] = np.eye(2)
    o = oracle.OracleSolver(p)
    pc = o.precond()
    assert pc["c_hat"] == 1.0
    assert np.all(pc["sx"] == 1.0) and np.all(pc["su"] == 1.0) and np.all(pc["sxN"] == 1.0)
    for i in range(1, tree.num_nodes()):
        assert np.abs(o.scaled_mat(0, i - 1, (2, 2)) - p.A[i - 1]).max() == 0.0
    assert np.all(pc["cstr_scale"] == 1.0)


def test_scalar_diagonal_scaling():  # test_problem.cpp:172-184
    tree = ScenarioTree.from_branching([4, 1])
    p = make_tiny(tree, 1, 1, 43)
    p.Q[:] = 4.0
    p.R[:] = 1.0
    o = oracle.OracleSolver(p)
    pc = o.precond()
    assert pc["c_hat"] == pytest.approx(2.0)
    assert pc["sx"][0] == pytest.approx(4.0)
    assert pc["su"][0] == pytest.approx(2.0)
    assert o.scaled_mat(2, 0, (1, 1))[0, 0] == pytest.approx(4.0 / 16.0)


def test_preconditioned_costs_value_preserving():  # test_problem.cpp:199-211
    tree = ScenarioTree.from_branching([2, 1])
    p = make_tiny(tree, 2, 2, 45)
    o = oracle.OracleSolver(p)
    pc = o.precond()
    rng = Philox(1)
    for i in range(1, tree.num_nodes()):
        x = rng.uniform_vector(2, -1.0, 1.0)
        u = rng.uniform_vector(2, -1.0, 1.0)
        Qs = o.scaled_mat(2, i - 1, (2, 2))
        Rs = o.scaled_mat(3, i - 1, (2, 2))
        xs, us = pc["sx"] * x, pc["su"] * u
        orig = x @ p.Q[i - 1] @ x + u @ p.R[i - 1] @ u + p.q[i - 1] @ x + p.r[i - 1] @ u
        qs, rs = p.q[i - 1] / pc["sx"], p.r[i - 1] / pc["su"]
        scal = xs @ Qs @ xs + us @ Rs @ us + qs @ xs + rs @ us
        assert orig == pytest.approx(scal, rel=1e-12)
