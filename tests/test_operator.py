"""L / L* / M-norm / ||L|| KATs and properties (proj/tests/test_oper.cpp)."""
import numpy as np
import pytest

from conftest import make_solver
from oracle import oracle
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.rng import Philox
from support import TinyOpts, make_tiny, materialize, random_vec, small_trees


def _raw(impl, p, **kw):
    return make_solver(impl, p, use_preconditioner=False, **kw)


def test_zero_and_linearity(impl):  # test_oper.cpp:39-55
    s = _raw(impl, make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 1))
    assert np.abs(s.apply_L(np.zeros(s.nz))).max() == 0.0
    rng = Philox(2)
    z1, z2 = random_vec(rng, s.nz), random_vec(rng, s.nz)
    e1, e2, e3 = s.apply_L(z1), s.apply_L(z2), s.apply_L(1.75 * z1 - 0.5 * z2)
    lin = 1.75 * e1 - 0.5 * e2
    assert np.abs(e3 - lin).max() <= 1e-12 * max(1.0, np.abs(lin).max())


def test_identity_weight_chain_segments(impl):  # test_oper.cpp:57-87
    tree = ScenarioTree.from_branching([1])
    p = make_tiny(tree, 1, 1, 3, TinyOpts(affine_c=False, linear_cost=False))
    p.A[0] = 1.0
    p.B[0] = 1.0
    p.Q[0] = 1.0
    p.R[0] = 1.0
    p.QN[0] = 1.0
    s = _raw(impl, p)
    el = oracle.OracleSolver(p, use_preconditioner=False).dual_layout()
    rng = Philox(4)
    z = random_vec(rng, s.nz)
    eta = s.apply_L(z)
    x0, x1, u0 = z[1], z[2], z[3]
    y0 = 4  # y_off[0]
    tau1, s1 = z[4 + p.risk[0].rows()], z[5 + p.risk[0].rows()]
    so = el["seg2_off"][0]
    assert eta[so + 0] == pytest.approx(x0, rel=1e-14)
    assert eta[so + 1] == pytest.approx(u0, rel=1e-14)
    assert eta[so + 2] == pytest.approx(0.5 * tau1, rel=1e-14)
    assert eta[so + 3] == pytest.approx(0.5 * tau1, rel=1e-14)
    lo = el["seg3_off"][0] + el["seg3_nc"][0]
    assert eta[lo + 0] == pytest.approx(x1, rel=1e-14)
    assert eta[lo + 1] == pytest.approx(0.5 * s1, rel=1e-14)
    rs = el["seg1_off"][0] + el["seg1_ydim"][0]
    ny = p.risk[0].rows()
    assert eta[rs] == pytest.approx(z[0] - p.risk[0].b @ z[y0:y0 + ny], rel=1e-14)


def test_adjoint_identity(impl):  # test_oper.cpp:89-107
    rng = Philox(5)
    for tree in small_trees():
        p = make_tiny(tree, 3, 2, rng.next_u64(), TinyOpts(gamma=0.6, q_rank_deficient_prob=0.3))
        s = _raw(impl, p)
        for _ in range(100):
            z, e = random_vec(rng, s.nz), random_vec(rng, s.neta)
            a, b = s.apply_L(z) @ e, z @ s.apply_Lt(e)
            assert abs(a - b) <= 1e-10 * max(1.0, abs(a))


def test_risk_scalar_adjoint_scatter(impl):  # test_oper.cpp:109-123
    p = make_tiny(ScenarioTree.from_branching([2]), 1, 1, 6)
    s = _raw(impl, p)
    el = oracle.OracleSolver(p, use_preconditioner=False).dual_layout()
    e = np.zeros(s.neta)
    e[el["seg1_off"][0] + el["seg1_ydim"][0]] = 1.0
    z = s.apply_Lt(e)
    assert z[0] == 1.0
    y0 = 1 + 3 * 1 + 1 * 1
    ny = p.risk[0].rows()
    assert np.abs(z[y0:y0 + ny] + p.risk[0].b).max() == 0.0
    z[0] = 0.0
    z[y0:y0 + ny] = 0.0
    assert np.abs(z).max() == 0.0


def test_operator_deterministic(impl):  # test_oper.cpp:125-141
    p = make_tiny(ScenarioTree.from_branching([3, 2, 1]), 3, 2, 7)
    s = _raw(impl, p)
    rng = Philox(8)
    z, e = random_vec(rng, s.nz), random_vec(rng, s.neta)
    if impl == "oracle":
        oracle.set_num_threads(4)
    a1, b1 = s.apply_L(z), s.apply_Lt(e)
    if impl == "oracle":
        oracle.set_num_threads(1)
    a2, b2 = s.apply_L(z), s.apply_Lt(e)
    if impl == "oracle":
        oracle.set_num_threads(2)
    assert np.abs(a1 - a2).max() == 0.0 and np.abs(b1 - b2).max() == 0.0


def test_power_iteration_matches_svd(impl):  # test_oper.cpp:143-157
    rng = Philox(9)
    for tree in small_trees():
        if tree.num_nodes() > 10:
            continue
        p = make_tiny(tree, 2, 1, rng.next_u64())
        s = _raw(impl, p)
        o = oracle.OracleSolver(p, use_preconditioner=False)
        L = materialize(s.nz, s.apply_L)
        sv = np.linalg.svd(L, compute_uv=False)[0]
        est = 0.99 / s.alpha
        assert est == pytest.approx(sv, rel=1e-6)
        nrm = o.op_norm()
        assert nrm["converged"]
        assert nrm["estimate"] <= nrm["analytic_bound"] * (1 + 1e-6)


def test_power_iteration_identity():  # test_oper.cpp:159-163
    assert oracle.estimate_norm_identity(10) == pytest.approx(1.0, rel=1e-6)


def test_scaling_cost_block_scales_norm(impl):  # test_oper.cpp:165-181
    tree = ScenarioTree.from_branching([1, 1])
    p = make_tiny(tree, 2, 1, 10, TinyOpts(linear_cost=False))
    for g in p.Gx:
        g[:] = 0.0
    for g in p.Gu:
        g[:] = 0.0
    for g in p.GN:
        g[:] = 0.0
    p.Q[:] = 100.0 * np.eye(2)
    n1 = 0.99 / _raw(impl, p).alpha
    p.Q *= 4.0
    n2 = 0.99 / _raw(impl, p).alpha
    assert n2 == pytest.approx(2.0 * n1, rel=1e-3)


def test_analytic_bound_dominates():  # test_oper.cpp:183-197
    rng = Philox(11)
    for _ in range(10):
        nx, nu = rng.uniform_int(1, 4), rng.uniform_int(1, 3)
        o = TinyOpts(gamma=rng.uniform(), q_rank_deficient_prob=0.3)
        for tree in small_trees():
            s = oracle.OracleSolver(make_tiny(tree, nx, nu, rng.next_u64(), o), use_preconditioner=False)
            n = s.op_norm()
            assert n["estimate"] <= n["analytic_bound"] * (1 + 1e-6)


def test_block_sparsity(impl):  # test_oper.cpp:199-235
    tree = ScenarioTree.from_branching([2, 1])
    p = make_tiny(tree, 2, 1, 12)
    s = _raw(impl, p)
    o = oracle.OracleSolver(p, use_preconditioner=False)
    zl, el = o.primal_layout(), o.dual_layout()
    L = materialize(s.nz, s.apply_L)
    nx, nu = 2, 1
    allowed = np.zeros_like(L)

    def allow(r0, rn, c0, cn):
        allowed[r0:r0 + rn, c0:c0 + cn] = 1

    xo = lambda i: 1 + i * nx
    uo = lambda i: zl["u_base"] + i * nu
    so = lambda i: 0 if i == 0 else zl["s_base"] + i - 1
    for i in range(tree.num_nonleaf()):
        yd, yo = zl["y_dim"][i], zl["y_off"][i]
        s1 = el["seg1_off"][i]
        allow(s1, yd, yo, yd)
        allow(s1 + yd, 1, yo, yd)
        allow(s1 + yd, 1, so(i), 1)
        allow(s1 + yd + 1, el["seg1_nc"][i], xo(i), nx)
        allow(s1 + yd + 1, el["seg1_nc"][i], uo(i), nu)
    for i in range(1, tree.num_nodes()):
        a = tree.anc[i]
        o2, d = el["seg2_off"][i - 1], el["seg2_dim"][i - 1]
        allow(o2, d, xo(a), nx)
        allow(o2, d, uo(a), nu)
        allow(o2, d, zl["tau_base"] + i - 1, 1)
    for j in range(tree.num_leaves()):
        node = tree.num_nonleaf() + j
        o3, nc, d = el["seg3_off"][j], el["seg3_nc"][j], el["seg3_socdim"][j]
        allow(o3, nc, xo(node), nx)
        allow(o3 + nc, d, xo(node), nx)
        allow(o3 + nc, d, so(node), 1)
    assert np.all(L[allowed == 0] == 0.0)


def test_m_norm_cases_and_bounds(impl):  # test_oper.cpp:237-274
    p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 13)
    s = _raw(impl, p)
    rng = Philox(14)
    z, e = random_vec(rng, s.nz), random_vec(rng, s.neta)
    assert s.m_norm(z, np.zeros(s.neta), 0.3) == pytest.approx(np.linalg.norm(z), rel=1e-14)
    assert s.m_norm(z, e, 0.0) == pytest.approx(np.sqrt(z @ z + e @ e), rel=1e-14)
    nL = 0.99 / s.alpha
    alpha = 0.99 / nL
    for _ in range(50):
        zz, ee = random_vec(rng, s.nz), random_vec(rng, s.neta)
        m2 = s.m_norm(zz, ee, alpha) ** 2
        v2 = zz @ zz + ee @ ee
        assert m2 >= (1 - alpha * nL) * v2 - 1e-9
        assert m2 <= (1 + alpha * nL) * v2 + 1e-9
    prng = Philox(1)
    zdom = prng.normal_array(s.nz)
    for _ in range(200):
        back = s.apply_Lt(s.apply_L(zdom))
        zdom = back / np.linalg.norm(back)
    Lz = s.apply_L(zdom)
    with pytest.raises(RuntimeError):
        s.m_norm(zdom, Lz / np.linalg.norm(Lz), 10.0 / nL)
