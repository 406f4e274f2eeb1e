"""Projection KATs and properties, restated from proj/tests/test_proj.cpp.

Each test runs against the oracle (CPU restatement) and, on a GPU box, against
the B200 solver through the C-ABI (``impl`` fixture), so the parity suite reads
like the reference's own tests.  Problems are built unpreconditioned where the
reference calls the projections on the raw problem.
"""
import numpy as np
import pytest

from conftest import make_solver
from oracle import oracle
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.rng import Philox
from support import (TinyOpts, dense_dynamics_constraints, make_scalar_chain, make_tiny, proj_affine_kkt,
                     random_vec, small_trees)


def test_soc_closed_forms():  # test_proj.cpp:38-45
    assert np.array_equal(oracle.proj_soc([1, 2]), [1, 2])
    assert np.linalg.norm(oracle.proj_soc([1, -2])) == 0.0
    r = oracle.proj_soc([3, 4, 0])
    np.testing.assert_allclose(r, [1.5, 2.0, 2.5])


def test_translated_soc_variational_inequality():  # test_proj.cpp:47-63
    rng = Philox(2)
    for _ in range(100):
        d = rng.uniform_int(2, 6)
        a = random_vec(rng, d)
        v = 3.0 * random_vec(rng, d)
        r = oracle.proj_soc(v - a) + a
        rc = r - a
        assert np.linalg.norm(rc[:-1]) <= rc[-1] + 1e-12
        for _ in range(20):
            w = random_vec(rng, d)
            w[-1] = np.linalg.norm(w[:-1]) + rng.uniform(0.0, 2.0)
            w = w + a
            assert (v - r) @ (w - r) <= 1e-9


def _raw(impl, p, **kw):
    return make_solver(impl, p, use_preconditioner=False, **kw)


def _z1(s, z):
    nn, nnl = s.problem.tree.num_nodes(), s.problem.tree.num_nonleaf()
    return z[1:1 + nn * s.problem.nx + nnl * s.problem.nu]


def test_dynamics_factorization_scalar_chain():  # test_proj.cpp:73-81
    s = oracle.OracleSolver(make_scalar_chain(), use_preconditioner=False)
    assert s.cache_mat(0, 1)[0, 0] == pytest.approx(1.0)
    assert s.cache_mat(1, 0)[0, 0] == pytest.approx(-0.5)
    assert s.cache_mat(3, 0)[0, 0] == pytest.approx(0.5)
    assert s.cache_mat(0, 0)[0, 0] == pytest.approx(1.5)


def test_zero_input_matrix_reduces_factorization():  # test_proj.cpp:83-96
    tree = ScenarioTree.from_branching([2, 1])
    p = make_tiny(tree, 2, 1, 4)
    p.B[:] = 0.0
    s = oracle.OracleSolver(p, use_preconditioner=False)
    for i in range(tree.num_nonleaf()):
        assert np.abs(s.cache_mat(1, i)).max() == 0.0
        np.testing.assert_array_equal(s.cache_mat(2, i), np.eye(1))
    for i in range(1, tree.num_nodes()):
        assert np.abs(s.cache_mat(3, i - 1) - p.A[i - 1]).max() == 0.0


def test_identical_children_double_riccati_sum():  # test_proj.cpp:98-108
    tree = ScenarioTree.from_branching([2])
    p = make_tiny(tree, 2, 2, 5)
    p.A[1] = p.A[0]
    p.B[1] = p.B[0]
    s = oracle.OracleSolver(p, use_preconditioner=False)
    want = np.eye(2) + 2.0 * p.B[0].T @ p.B[0]
    assert np.abs(s.cache_mat(2, 0) - want).max() < 1e-12


def test_scalar_chain_projection_example(impl):  # test_proj.cpp:110-122
    p = make_scalar_chain(0.0)
    s = _raw(impl, p)
    z = np.zeros(s.nz)
    z[1 + 1] = 2.0  # x(1)
    out = s.proj_s1(z)
    u0 = 1 + 2 * 1  # u_base
    assert out[1] == pytest.approx(0.0)
    assert out[2] == pytest.approx(1.0)
    assert out[u0] == pytest.approx(1.0)


def test_feasible_points_fixed(impl):  # test_proj.cpp:124-145
    rng = Philox(6)
    for tree in small_trees():
        p = make_tiny(tree, 2, 1, rng.next_u64())
        s = _raw(impl, p)
        nx, nu, nn = 2, 1, tree.num_nodes()
        ub = 1 + nn * nx
        z = np.zeros(s.nz)
        z[1:1 + nx] = p.x_init
        for i in range(tree.num_nonleaf()):
            z[ub + i * nu: ub + (i + 1) * nu] = random_vec(rng, nu)
            for ip in tree.children(i):
                z[1 + ip * nx: 1 + (ip + 1) * nx] = (p.A[ip - 1] @ z[1 + i * nx: 1 + (i + 1) * nx]
                                                    + p.B[ip - 1] @ z[ub + i * nu: ub + (i + 1) * nu] + p.c[ip - 1])
        out = s.proj_s1(z)
        assert np.abs(out - z).max() < 1e-10


def test_dynamics_projection_matches_dense_kkt(impl):  # test_proj.cpp:147-164
    rng = Philox(7)
    for tree in small_trees():
        p = make_tiny(tree, 2, 1, rng.next_u64())
        s = _raw(impl, p)
        G, h = dense_dynamics_constraints(p, p.x_init)
        for _ in range(25):
            z = random_vec(rng, s.nz, 3.0)
            got = _z1(s, s.proj_s1(z))
            want = proj_affine_kkt(G, h, _z1(s, z))
            assert np.abs(got - want).max() < 1e-8
            assert np.abs(G @ got - h).max() < 1e-10


def _s2_groups(p, zl_y_off, tau_base, s_base):
    tr = p.tree
    for i in range(tr.num_nonleaf()):
        ny = p.risk[i].rows()
        nch = tr.child_count[i]
        cf = tr.child_first[i]
        M = np.zeros((nch, ny + 2 * nch))
        M[:, :ny] = p.risk[i].E.T
        M[:, ny:ny + nch] = -np.eye(nch)
        M[:, ny + nch:] = -np.eye(nch)
        idx = list(range(zl_y_off[i], zl_y_off[i] + ny))
        idx += [tau_base + (cf + k - 1) for k in range(nch)]
        idx += [(0 if cf + k == 0 else s_base + (cf + k - 1)) for k in range(nch)]
        yield M, np.array(idx)


def test_kernel_projection_matches_dense_kkt(impl):  # test_proj.cpp:166-205
    rng = Philox(8)
    for tree in small_trees():
        p = make_tiny(tree, 2, 1, rng.next_u64(), TinyOpts(gamma=0.7))
        s = _raw(impl, p)
        lay = oracle.OracleSolver(p, use_preconditioner=False).primal_layout()
        for _ in range(25):
            z0 = random_vec(rng, s.nz, 3.0)
            z = s.proj_s2(z0)
            for M, idx in _s2_groups(p, lay["y_off"], lay["tau_base"], lay["s_base"]):
                want = proj_affine_kkt(M, np.zeros(M.shape[0]), z0[idx])
                assert np.abs(z[idx] - want).max() < 1e-9
                assert np.abs(M @ z[idx]).max() < 1e-9
            nz1 = tree.num_nodes() * 2 + tree.num_nonleaf()
            assert np.array_equal(z[:1 + nz1], z0[:1 + nz1])


def test_kernel_projectors_idempotent_symmetric():  # test_proj.cpp:207-217
    tree = ScenarioTree.from_branching([3, 2])
    p = make_tiny(tree, 2, 1, 9, TinyOpts(gamma=0.3))
    s = oracle.OracleSolver(p, use_preconditioner=False)
    for i in range(tree.num_nonleaf()):
        N = s.cache_mat(4, i)
        assert np.abs(N @ N - N).max() < 1e-10
        assert np.abs(N - N.T).max() < 1e-12


def test_image_projection_feasible_unchanged(impl):  # test_proj.cpp:219-268
    rng = Philox(10)
    tree = ScenarioTree.from_branching([2, 2])
    p = make_tiny(tree, 2, 1, 11, TinyOpts(gamma=0.5, box_halfwidth=1.0))
    s = _raw(impl, p)
    o = oracle.OracleSolver(p, use_preconditioner=False)
    el = o.dual_layout()
    nnl, nn = tree.num_nonleaf(), tree.num_nodes()
    eta = np.zeros(s.neta)
    for i in range(nnl):
        ny, nc, off = el["seg1_ydim"][i], el["seg1_nc"][i], el["seg1_off"][i]
        eta[off:off + ny] = np.abs(random_vec(rng, ny))
        eta[off + ny] = rng.uniform(0.0, 1.0)
        eta[off + ny + 1: off + ny + 1 + nc] = np.clip(random_vec(rng, nc, 2.0), p.C[i].lo, p.C[i].hi)
    for i in range(1, nn):
        d, off = el["seg2_dim"][i - 1], el["seg2_off"][i - 1]
        w = random_vec(rng, d)
        w[-1] = np.linalg.norm(w[:-1]) + rng.uniform(0.0, 2.0)
        eta[off:off + d] = w + o.soc(0, i - 1)["a"]
    for j in range(tree.num_leaves()):
        nc, off, d = el["seg3_nc"][j], el["seg3_off"][j], el["seg3_socdim"][j]
        eta[off:off + nc] = np.clip(random_vec(rng, nc, 2.0), p.CN[j].lo, p.CN[j].hi)
        w = random_vec(rng, d)
        w[-1] = np.linalg.norm(w[:-1]) + rng.uniform(0.0, 2.0)
        eta[off + nc: off + nc + d] = w + o.soc(1, j)["a"]
    out = s.proj_s3(eta)
    assert np.abs(out - eta).max() < 1e-12
    eta[el["seg1_off"][0] + el["seg1_ydim"][0]] = -1.0
    out = s.proj_s3(eta)
    assert out[el["seg1_off"][0] + el["seg1_ydim"][0]] == 0.0
    e1 = random_vec(rng, s.neta, 3.0)
    if impl == "oracle":
        oracle.set_num_threads(4)
        a = s.proj_s3(e1)
        oracle.set_num_threads(1)
        b = s.proj_s3(e1)
        oracle.set_num_threads(2)
    else:
        a = s.proj_s3(e1)
        b = s.proj_s3(e1)
    assert np.abs(a - b).max() == 0.0


def test_projections_idempotent_nonexpansive(impl):  # test_proj.cpp:270-299
    rng = Philox(12)
    tree = ScenarioTree.from_branching([2, 2, 1])
    p = make_tiny(tree, 2, 2, 13, TinyOpts(gamma=0.4, box_halfwidth=0.8))
    s = _raw(impl, p)
    for _ in range(20):
        a = random_vec(rng, s.nz, 3.0)
        b = random_vec(rng, s.nz, 3.0)
        pa, pb = s.proj_s1(a), s.proj_s1(b)
        assert np.abs(s.proj_s1(pa) - pa).max() < 1e-10
        za, zb, pza, pzb = _z1(s, a), _z1(s, b), _z1(s, pa), _z1(s, pb)
        assert np.linalg.norm(pza - pzb) <= np.linalg.norm(za - zb) + 1e-12
        assert (pza - pzb) @ (pza - pzb) <= (za - zb) @ (pza - pzb) + 1e-9
        pa, pb = s.proj_s2(a), s.proj_s2(b)
        assert np.abs(s.proj_s2(pa) - pa).max() < 1e-10
        assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) + 1e-12
        ea = random_vec(rng, s.neta, 3.0)
        eb = random_vec(rng, s.neta, 3.0)
        qa, qb = s.proj_s3(ea), s.proj_s3(eb)
        assert np.abs(s.proj_s3(qa) - qa).max() < 1e-10
        assert np.linalg.norm(qa - qb) <= np.linalg.norm(ea - eb) + 1e-12
