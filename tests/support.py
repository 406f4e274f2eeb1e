"""Test fixtures restated from the reference suite (proj/tests/support.hpp:10-130)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2505_12078_b200.problem import Box, Raocp, ScenarioTree, avar_spec, expectation_spec
from paper_2505_12078_b200.rng import Philox


@dataclass
class TinyOpts:  # support.hpp:12-21
    gamma: float = 1.0
    box_halfwidth: float = 1e6
    affine_c: bool = True
    linear_cost: bool = True
    q_rank_deficient_prob: float = 0.0
    avar_form_at_one: bool = False


def make_tiny(tree: ScenarioTree, nx: int, nu: int, seed: int, o: TinyOpts = None) -> Raocp:
    """make_tiny, support.hpp:24-88 (same Philox draw order)."""
    o = o or TinyOpts()
    rng = Philox(seed)
    nn, nnl, nl = tree.num_nodes(), tree.num_nonleaf(), tree.num_leaves()
    A = np.zeros((nn - 1, nx, nx))
    B = np.zeros((nn - 1, nx, nu))
    c = np.zeros((nn - 1, nx))
    Q = np.zeros((nn - 1, nx, nx))
    R = np.zeros((nn - 1, nu, nu))
    q = np.zeros((nn - 1, nx))
    r = np.zeros((nn - 1, nu))
    for i in range(1, nn):
        A[i - 1] = 0.8 * np.eye(nx) + rng.normal_matrix(nx, nx, 0.0, 0.1)
        B[i - 1] = rng.normal_matrix(nx, nu, 0.0, 0.5)
        if o.affine_c:
            c[i - 1] = rng.normal_matrix(nx, 1, 0.0, 0.1)[:, 0]
        M = rng.normal_matrix(nx, nx, 0.0, 1.0)
        if rng.uniform() < o.q_rank_deficient_prob and nx > 1:
            M[:, 0] = 0.0
        Q[i - 1] = M @ M.T / nx
        Mr = rng.normal_matrix(nu, nu, 0.0, 0.3)
        R[i - 1] = np.eye(nu) + Mr @ Mr.T
        if o.linear_cost:
            q[i - 1] = rng.normal_matrix(nx, 1, 0.0, 0.1)[:, 0]
            r[i - 1] = rng.normal_matrix(nu, 1, 0.0, 0.1)[:, 0]
    QN = np.zeros((nl, nx, nx))
    qN = np.zeros((nl, nx))
    for j in range(nl):
        M = rng.normal_matrix(nx, nx, 0.0, 1.0)
        QN[j] = M @ M.T / nx
        if o.linear_cost:
            qN[j] = rng.normal_matrix(nx, 1, 0.0, 0.1)[:, 0]
    Gx = np.zeros((nx + nu, nx))
    Gx[:nx] = np.eye(nx)
    Gu = np.zeros((nx + nu, nu))
    Gu[nx:] = np.eye(nu)
    bh = np.full(nx + nu, o.box_halfwidth)
    risk = []
    for i in range(nnl):
        if o.gamma == 1.0 and not o.avar_form_at_one:
            risk.append(expectation_spec(tree.child_probs(i)))
        else:
            risk.append(avar_spec(o.gamma, tree.child_probs(i)))
    x_init = rng.normal_matrix(nx, 1, 0.0, 1.0)[:, 0]
    return Raocp(tree=tree, nx=nx, nu=nu, A=A, B=B, c=c, Q=Q, R=R, q=q, r=r, QN=QN, qN=qN,
                 Gx=[Gx.copy() for _ in range(nnl)], Gu=[Gu.copy() for _ in range(nnl)],
                 C=[Box(-bh.copy(), bh.copy()) for _ in range(nnl)], risk=risk,
                 GN=[np.eye(nx) for _ in range(nl)],
                 CN=[Box(np.full(nx, -o.box_halfwidth), np.full(nx, o.box_halfwidth)) for _ in range(nl)],
                 x_init=x_init)


def make_scalar_chain(x_init: float = 1.0) -> Raocp:
    """make_scalar_chain, support.hpp:92-105."""
    tree = ScenarioTree.from_branching([1])
    p = make_tiny(tree, 1, 1, 0, TinyOpts(affine_c=False, linear_cost=False))
    p.A[0] = 1.0
    p.B[0] = 1.0
    p.Q[0] = 1.0
    p.R[0] = 1.0
    p.QN[0] = 1.0
    p.x_init = np.array([x_init])
    return p


def small_trees():
    """small_trees, support.hpp:108-130."""
    out = [ScenarioTree.from_branching([1, 1, 1]), ScenarioTree.from_branching([2, 1]),
           ScenarioTree.from_branching([2, 2]), ScenarioTree.from_branching([3, 2, 1])]
    cp = [np.array([0.5, 0.3, 0.2]), np.array([0.5, 0.5]), np.array([0.25, 0.75]), np.array([0.9, 0.1])]
    cp += [np.ones(1)] * 6
    out.append(ScenarioTree.from_branching([3, 2, 1], cp))
    tm = np.array([[0.9, 0.1], [0.4, 0.6]])
    out.append(ScenarioTree.from_markov(tm, np.array([0.7, 0.3]), 3, 2))
    return out


def random_vec(rng: Philox, n: int, scale: float = 2.0) -> np.ndarray:
    """random_vec of the reference tests: uniform(-scale, scale) per entry."""
    return -scale + 2.0 * scale * rng.uniform_array(n)


# ---- dense oracles restated from proj/src/reference.cpp (numpy) ----
def materialize(n_in: int, apply) -> np.ndarray:
    """reference.cpp:247-258."""
    cols = []
    e = np.zeros(n_in)
    for k in range(n_in):
        e[k] = 1.0
        cols.append(np.asarray(apply(e.copy()), dtype=np.float64))
        e[k] = 0.0
    return np.stack(cols, axis=1)


def proj_affine_kkt(A: np.ndarray, b: np.ndarray, v: np.ndarray) -> np.ndarray:
    """min ||w - v|| s.t. A w = b (reference.cpp:260-272), via lstsq on the KKT system."""
    n, m = A.shape[1], A.shape[0]
    K = np.zeros((n + m, n + m))
    K[:n, :n] = np.eye(n)
    K[:n, n:] = A.T
    K[n:, :n] = A
    rhs = np.concatenate([v, b])
    sol = np.linalg.lstsq(K, rhs, rcond=None)[0]
    return sol[:n]


def dense_dynamics_constraints(p: Raocp, x_init: np.ndarray):
    """reference.cpp:274-296; columns: x for all nodes, then u for non-leaves."""
    tr = p.tree
    nn, nnl, nx, nu = tr.num_nodes(), tr.num_nonleaf(), p.nx, p.nu
    nz1 = nn * nx + nnl * nu
    G = np.zeros((nn * nx, nz1))
    h = np.zeros(nn * nx)
    G[:nx, :nx] = np.eye(nx)
    h[:nx] = x_init
    for i in range(1, nn):
        a = tr.anc[i]
        G[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx] = np.eye(nx)
        G[i * nx:(i + 1) * nx, a * nx:(a + 1) * nx] = -p.A[i - 1]
        G[i * nx:(i + 1) * nx, nn * nx + a * nu: nn * nx + (a + 1) * nu] = -p.B[i - 1]
        h[i * nx:(i + 1) * nx] = p.c[i - 1]
    return G, h


def riccati_tree_solve(p: Raocp, x_init: np.ndarray) -> float:
    """Risk-neutral DP optimum value (reference.cpp:24-81)."""
    tr = p.tree
    nn, nnl = tr.num_nodes(), tr.num_nonleaf()
    W, w, w0 = [None] * nn, [None] * nn, [0.0] * nn
    for j in range(nnl, nn):
        W[j] = p.QN[j - nnl]
        w[j] = p.qN[j - nnl]
    for i in range(nnl - 1, -1, -1):
        Hxx = np.zeros((p.nx, p.nx))
        Huu = np.zeros((p.nu, p.nu))
        Hxu = np.zeros((p.nx, p.nu))
        hx = np.zeros(p.nx)
        hu = np.zeros(p.nu)
        h0 = 0.0
        for ip in tr.children(i):
            pr = tr.cond_prob[ip]
            A, B, c = p.A[ip - 1], p.B[ip - 1], p.c[ip - 1]
            Wc = W[ip]
            wc = 2.0 * Wc @ c + w[ip]
            Hxx += pr * (p.Q[ip - 1] + A.T @ Wc @ A)
            Huu += pr * (p.R[ip - 1] + B.T @ Wc @ B)
            Hxu += pr * (A.T @ Wc @ B)
            hx += pr * (p.q[ip - 1] + A.T @ wc)
            hu += pr * (p.r[ip - 1] + B.T @ wc)
            h0 += pr * (c @ Wc @ c + w[ip] @ c + w0[ip])
        Wi = Hxx - Hxu @ np.linalg.solve(Huu, Hxu.T)
        W[i] = 0.5 * (Wi + Wi.T)
        w[i] = hx - Hxu @ np.linalg.solve(Huu, hu)
        w0[i] = h0 - 0.25 * hu @ np.linalg.solve(Huu, hu)
    return float(x_init @ W[0] @ x_init + w[0] @ x_init + w0[0])


def _soc_proj_local(v: np.ndarray) -> np.ndarray:
    """reference.cpp:300-312 (axis last)."""
    t, hn = v[-1], np.linalg.norm(v[:-1])
    if hn <= t:
        return v.copy()
    r = np.zeros_like(v)
    if hn <= -t:
        return r
    r[:-1] = (hn + t) / (2.0 * hn) * v[:-1]
    r[-1] = 0.5 * (hn + t)
    return r


def _soc_face_distance(w, eta, a, tolc):
    """reference.cpp:314-331: sup-norm distance from w to the support face of
    SOC + a at eta (the face ray's sign corrected, see below); also returns the
    polar-cone violation of eta."""
    u = w - a
    ph, pt = np.linalg.norm(eta[:-1]), eta[-1]
    dv = ph + pt
    if np.abs(eta).max(initial=0.0) <= tolc:
        return float(np.abs(u - _soc_proj_local(u)).max()), dv
    if ph + pt < -tolc:
        return float(np.abs(u).max()), dv
    # Deviation from reference.cpp:325-327, documented: the reference builds the
    # ray along (-eta_head, |eta_head|).  For eta = c (d, -1) in the polar cone
    # (the normal cone of SOC at the boundary point s (d, 1), which is what
    # eta+ = p - alpha Pi(p / alpha) is, solver.cpp:148-164) the support face is the
    # ray along (+eta_head, |eta_head|); with the reference's sign the check fails
    # at every active SOC, also on the oracle's own converged solutions.
    d = np.concatenate([eta[:-1], [ph]])
    dn2 = d @ d
    s = max(0.0, (u @ d) / dn2) if dn2 > 0.0 else 0.0
    return float(np.abs(u - s * d).max()), dv


def kkt_check(sp, soc, L, zl, el, z, eta, tol1, tol2):
    """eps-KKT report of reference.cpp:335-494 (ref::kkt_check), numpy.

    sp: the scaled problem; soc(which, idx) -> dict with the translation "a"
    (0: stage, idx = node-1; 1: leaf); L: materialised operator (n_eta x n_z);
    zl / el: primal / dual layouts.  COD solves are min-norm least squares: the
    least-squares residual is the same for every minimiser."""
    from paper_2505_12078_b200.problem import CONE_FREE, CONE_NONNEG, CONE_SOC, CONE_ZERO, dual_cone
    tr = sp.tree
    nn, nnl, nx, nu = tr.num_nodes(), tr.num_nonleaf(), sp.nx, sp.nu
    Lte, Lz = L.T @ eta, L @ z
    tolc = 1e-8 * (1.0 + np.abs(eta).max())
    primal = abs(1.0 + Lte[0]) / tol1[0]
    membership = dual = 0.0
    nz1 = nn * nx + nnl * nu
    G, h = dense_dynamics_constraints(sp, sp.x_init)
    membership = max(membership, float(np.abs(G @ z[1:1 + nz1] - h).max()))
    w = -Lte[1:1 + nz1]
    lam = np.linalg.lstsq(G.T, w, rcond=None)[0]
    primal = max(primal, float((np.abs(w - G.T @ lam) / tol1[1:1 + nz1]).max()))
    for i in range(nnl):
        rk = sp.risk[i]
        ny, nch, cf = int(zl["y_dim"][i]), int(tr.child_count[i]), int(tr.child_first[i])
        nnu = rk.F.shape[1]
        dim = ny + 2 * nch
        M = np.zeros((nch + nnu, dim))
        M[:nch, :ny] = rk.E.T
        M[:nch, ny:ny + nch] = -np.eye(nch)
        M[:nch, ny + nch:] = -np.eye(nch)
        if nnu:
            M[nch:, :ny] = rk.F.T
        idx = np.array(list(range(zl["y_off"][i], zl["y_off"][i] + ny))
                       + [zl["tau_base"] + cf + k - 1 for k in range(nch)]
                       + [zl["s_base"] + cf + k - 1 for k in range(nch)])
        membership = max(membership, float(np.abs(M @ z[idx]).max()))
        w2 = -Lte[idx]
        lam = np.linalg.lstsq(M.T, w2, rcond=None)[0]
        primal = max(primal, float((np.abs(w2 - M.T @ lam) / tol1[idx]).max()))

    def box_dist(e, wv, lo, hi):
        if e > tolc:
            return abs(wv - hi)
        if e < -tolc:
            return abs(wv - lo)
        return max(0.0, lo - wv, wv - hi)

    for i in range(nn):
        if i < nnl:
            off = int(el["seg1_off"][i])
            for part in dual_cone(sp.risk[i].cone):
                if part.kind == CONE_SOC:
                    d, dv = _soc_face_distance(Lz[off:off + part.dim], eta[off:off + part.dim],
                                               np.zeros(part.dim), tolc)
                    membership = max(membership, dv)
                    dual = max(dual, d / tol2[off:off + part.dim].min())
                else:
                    for k in range(part.dim):
                        e, wv, tl = eta[off + k], Lz[off + k], tol2[off + k]
                        dist = 0.0
                        if part.kind == CONE_NONNEG:
                            membership = max(membership, e - tolc)
                            dist = abs(wv) if e < -tolc else max(0.0, -wv)
                        elif part.kind == CONE_FREE:
                            membership = max(membership, abs(e) - tolc)
                        elif part.kind == CONE_ZERO:
                            dist = abs(wv)
                        dual = max(dual, dist / tl)
                off += part.dim
            ix = int(el["seg1_off"][i]) + int(el["seg1_ydim"][i])  # risk scalar row
            e, wv = eta[ix], Lz[ix]
            membership = max(membership, e - tolc)
            dual = max(dual, (abs(wv) if e < -tolc else max(0.0, -wv)) / tol2[ix])
            for k in range(int(el["seg1_nc"][i])):
                ix2 = ix + 1 + k
                dual = max(dual, box_dist(eta[ix2], Lz[ix2], sp.C[i].lo[k], sp.C[i].hi[k]) / tol2[ix2])
        if i > 0:
            off, d = int(el["seg2_off"][i - 1]), int(el["seg2_dim"][i - 1])
            dist, dv = _soc_face_distance(Lz[off:off + d], eta[off:off + d], soc(0, i - 1)["a"], tolc)
            membership = max(membership, dv)
            dual = max(dual, dist / tol2[off:off + d].min())
        if i >= nnl:
            j = i - nnl
            off, nc, d = int(el["seg3_off"][j]), int(el["seg3_nc"][j]), int(el["seg3_socdim"][j])
            for k in range(nc):
                dual = max(dual, box_dist(eta[off + k], Lz[off + k], sp.CN[j].lo[k], sp.CN[j].hi[k]) / tol2[off + k])
            dist, dv = _soc_face_distance(Lz[off + nc:off + nc + d], eta[off + nc:off + nc + d], soc(1, j)["a"], tolc)
            membership = max(membership, dv)
            dual = max(dual, dist / tol2[off + nc:off + nc + d].min())
    return dict(primal=primal, dual=dual, membership=membership)
