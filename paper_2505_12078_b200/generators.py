"""Synthetic benchmark problems (the reference's case-study-1 family).

``gen_case1`` restates proj/src/generators.cpp:40-116 draw for draw from the
Philox stream (iid Markov tree with stopped branching, per-event dynamics and
costs, box constraints, AV@R risk at a random level).  ``gen_case1_perturbed``
adds an independent per-node perturbation so that no two nodes share matrices
(the roofline-graded runs must not be deduplicable).  The
``CONFIGS`` table pins the BASELINE.json shapes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .problem import Box, Raocp, ScenarioTree, avar_spec
from .rng import Philox


@dataclass
class Case1Dims:  # proj/include/spock/generators.hpp:18-25
    N: int
    nb: int
    nw: int
    nu: int
    nx: int
    nv: int = 0


def tree_nodes_up_to(nw: int, nb: int, t_max: int) -> int:  # generators.cpp:13-21
    total, width = 0, 1
    for t in range(t_max + 1):
        if 0 < t <= nb:
            width *= nw
        total += width
    return total


def sample_case1_dims(rng: Philox, desk_scale: bool) -> Case1Dims:  # generators.cpp:25-38
    nv_max = 10_000 if desk_scale else 100_000
    for _ in range(1_000_000):
        N = rng.uniform_int(5, 15)
        nb = rng.uniform_int(1, 3)
        nw = rng.uniform_int(2, 10)
        nu = rng.uniform_int(10, 300)
        nx = 2 * nu
        nv = nx * tree_nodes_up_to(nw, nb, N) + nu * tree_nodes_up_to(nw, nb, N - 1)
        if 1_000 <= nv <= nv_max:
            return Case1Dims(N, nb, nw, nu, nx, nv)
    raise RuntimeError("sample_case1_dims: rejection sampling failed")


def gen_case1(rng: Philox, dims: Case1Dims, gamma: Optional[float] = None,
              perturb: float = 0.0, perturb_seed: int = 0) -> Raocp:
    """gen_case1 (generators.cpp:40-116).

    ``gamma`` overrides the sampled AV@R level (config 1 uses 0.95) after the
    draw, so the stream is consumed exactly as the reference does.  With
    ``perturb > 0`` every non-root node gets A + e*G, B + e*G and cost factors
    (Qb + e*G)(.)', (Rb + e*G)(.)' with independent standard normals G from a
    separate numpy stream (``perturb_seed``).
    """
    nx, nu, nw = dims.nx, dims.nu, dims.nw
    for attempt in range(10_000):
        pi = rng.simplex(nw)
        if pi.min() >= 1e-4:
            break
        if attempt > 1000:
            raise RuntimeError("gen_case1: degenerate probability vector")
    g = rng.uniform()
    trans = np.tile(pi, (nw, 1))
    tree = ScenarioTree.from_markov(trans, pi, dims.N, dims.nb)
    B0 = rng.normal_matrix(nx, nu, 0.0, 1.0)
    q0 = rng.uniform_vector(nx, 0.0, 0.1)
    r0 = rng.uniform_vector(nu, 0.0, 100.0)
    Aw, Bw, Qb, Rb = [], [], [], []
    for _ in range(nw):
        Aw.append(np.eye(nx) + rng.normal_matrix(nx, nx, 0.0, 0.1))
        Bw.append(B0 + rng.normal_matrix(nx, nu, 0.0, 0.1))
        Qb.append(np.diag(q0) + rng.normal_matrix(nx, nx, 0.0, 0.1))
        Rb.append(np.diag(r0) + rng.normal_matrix(nu, nu, 0.0, 0.1))
    xbar = rng.uniform_vector(nx, 1.0, 2.0)
    ubar = rng.uniform_vector(nu, 0.0, 0.1)
    nn, nnl, nl = tree.num_nodes(), tree.num_nonleaf(), tree.num_leaves()
    ev = tree.event[1:]
    A = np.stack(Aw)[ev]
    B = np.stack(Bw)[ev]
    if perturb > 0.0:
        prs = np.random.default_rng(perturb_seed)
        A = A + perturb * prs.standard_normal(A.shape)
        B = B + perturb * prs.standard_normal(B.shape)
        Qf = np.stack(Qb)[ev] + perturb * prs.standard_normal((nn - 1, nx, nx))
        Rf = np.stack(Rb)[ev] + perturb * prs.standard_normal((nn - 1, nu, nu))
        Q = Qf @ Qf.transpose(0, 2, 1)
        R = Rf @ Rf.transpose(0, 2, 1)
    else:
        Qw = np.stack([m @ m.T for m in Qb])
        Rw = np.stack([m @ m.T for m in Rb])
        Q = Qw[ev]
        R = Rw[ev]
    Q = 0.5 * (Q + Q.transpose(0, 2, 1))
    R = 0.5 * (R + R.transpose(0, 2, 1))
    lo = np.concatenate([-xbar, -ubar])
    hi = np.concatenate([xbar, ubar])
    Gx = np.zeros((nx + nu, nx))
    Gx[:nx] = np.eye(nx)
    Gu = np.zeros((nx + nu, nu))
    Gu[nx:] = np.eye(nu)
    gamma_v = g if gamma is None else gamma
    risk = [avar_spec(gamma_v, tree.child_probs(i)) for i in range(nnl)]
    x_init = np.array([rng.uniform(-0.5 * xbar[k], 0.5 * xbar[k]) for k in range(nx)])
    return Raocp(
        tree=tree, nx=nx, nu=nu, A=A, B=B, c=np.zeros((nn - 1, nx)), Q=Q, R=R,
        q=np.zeros((nn - 1, nx)), r=np.zeros((nn - 1, nu)),
        QN=np.tile(np.diag(q0), (nl, 1, 1)), qN=np.zeros((nl, nx)),
        Gx=np.broadcast_to(Gx, (nnl, nx + nu, nx)), Gu=np.broadcast_to(Gu, (nnl, nx + nu, nu)),
        C=[Box(lo, hi)] * nnl, risk=risk,
        GN=np.broadcast_to(np.eye(nx), (nl, nx, nx)), CN=[Box(-xbar, xbar)] * nl,
        x_init=x_init, meta=dict(gamma=gamma_v, pi=pi, dims=dims, perturb=perturb))


def gen_case1_instance(seed: int, desk_scale: bool) -> Raocp:  # generators.cpp:118-122
    rng = Philox(seed)
    return gen_case1(rng, sample_case1_dims(rng, desk_scale))


# BASELINE.json configs resolved to concrete dims.
CONFIGS = {
    "c1": dict(N=5, nb=3, nw=2, nx=10, nu=5, gamma=0.95, perturb=0.0),
    "c2": dict(N=10, nb=5, nw=2, nx=50, nu=25, gamma=None, perturb=0.01),
    "c2p": dict(N=10, nb=8, nw=2, nx=50, nu=25, gamma=None, perturb=0.01),
    "c3": dict(N=12, nb=8, nw=3, nx=50, nu=25, gamma=None, perturb=0.01),
    "c4": dict(N=12, nb=4, nw=10, nx=50, nu=25, gamma=None, perturb=0.01),
    # configs[4] at one GPU's scale: the c5 state size (n_x 100 = 2 n_u)
    # on a (12, 4, 7) tree of 103 765 nodes (~56 GB of per-node blocks on the device)
    "c5s": dict(N=12, nb=7, nw=4, nx=100, nu=50, gamma=None, perturb=0.01),
    # n_x = 100 tree small enough for the CPU oracle's parity checks (9 557 nodes, wide path)
    "c5p": dict(N=7, nb=6, nw=4, nx=100, nu=50, gamma=None, perturb=0.01),
}


def make_config(name: str, seed: int = 1, **over) -> Raocp:
    cfg = dict(CONFIGS[name])
    cfg.update(over)
    dims = Case1Dims(N=cfg["N"], nb=cfg["nb"], nw=cfg["nw"], nu=cfg["nu"], nx=cfg["nx"])
    rng = Philox(seed)
    p = gen_case1(rng, dims, gamma=cfg["gamma"], perturb=cfg["perturb"], perturb_seed=seed)
    p.meta["config"] = name
    return p
