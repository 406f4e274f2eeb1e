"""Problem model mirrored from the reference's public C++ types.

``ScenarioTree`` (proj/include/spock/tree.hpp:14-88), ``RiskSpec``/``avar_spec``/
``expectation_spec`` (proj/include/spock/risk.hpp:26-65), ``Box`` and ``Raocp``
(proj/include/spock/problem.hpp:14-58).  Per-node data use the reference's
indexing: dynamics and stage costs at the child node (array index node-1),
constraints and risks per non-leaf node, terminal data per leaf (index
node-num_nonleaf).  Matrices are numpy arrays in (rows, cols) shape; packing to
the C-ABI (column-major, back to back) happens in ``capi.pack_problem``.

Validation of the tree arrays and of the problem data happens behind the C-ABI
(the reference's ``ScenarioTree::finalize_topology`` and ``Raocp::validate``);
the builders here only raise for malformed builder arguments, as the
reference's builders do.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

PROB_TOL = 1e-12

CONE_ZERO, CONE_NONNEG, CONE_SOC, CONE_FREE = 0, 1, 2, 3
RISK_AVAR, RISK_GENERAL = 0, 1


def _check_prob_vector(p: np.ndarray, what: str) -> None:
    if p.size == 0:
        raise ValueError(f"{what}: empty probability vector")
    if np.any(p <= 0.0):
        raise ValueError(f"{what}: probabilities must be positive")
    if abs(p.sum() - 1.0) > PROB_TOL:
        raise ValueError(f"{what}: probabilities must sum to 1")


class ScenarioTree:
    """Stage-contiguous BFS-numbered scenario tree (tree.hpp:10-88)."""

    def __init__(self, anc, event, prob, cond_prob, stop_stage: int, num_events: int):
        self.anc = np.asarray(anc, dtype=np.int32)
        self.event = np.asarray(event, dtype=np.int32)
        self.prob = np.asarray(prob, dtype=np.float64)
        self.cond_prob = np.asarray(cond_prob, dtype=np.float64)
        self.stop_stage = int(stop_stage)
        self.num_events = int(num_events)
        n = self.anc.size
        stage = np.zeros(n, dtype=np.int32)
        for i in range(1, n):
            stage[i] = stage[self.anc[i]] + 1
        self.stage = stage
        self.horizon = int(stage[-1])
        self.child_first = np.full(n, n, dtype=np.int32)
        self.child_count = np.zeros(n, dtype=np.int32)
        if n > 1:
            a = self.anc[1:]
            cnt = np.bincount(a, minlength=n)
            self.child_count = cnt.astype(np.int32)
            first = np.full(n, n, dtype=np.int64)
            np.minimum.at(first, a, np.arange(1, n))
            self.child_first = first.astype(np.int32)
        ss = np.zeros(self.horizon + 2, dtype=np.int32)
        np.add.at(ss, stage + 1, 1)
        self.stage_start = np.cumsum(ss).astype(np.int32)

    # tree.hpp:35-70
    def num_nodes(self) -> int:
        return int(self.anc.size)

    def num_nonleaf(self) -> int:
        return int(self.stage_start[self.horizon])

    def num_leaves(self) -> int:
        return self.num_nodes() - self.num_nonleaf()

    def stage_begin(self, t: int) -> int:
        return int(self.stage_start[t])

    def stage_end(self, t: int) -> int:
        return int(self.stage_start[t + 1])

    def is_leaf(self, i: int) -> bool:
        return self.child_count[i] == 0

    def children(self, i: int) -> range:
        return range(int(self.child_first[i]), int(self.child_first[i] + self.child_count[i]))

    def child_probs(self, i: int) -> np.ndarray:
        return self.cond_prob[self.children(i)].copy()

    # ScenarioTree::from_branching, proj/src/tree.cpp:91-139
    @staticmethod
    def from_branching(branching: Sequence[int], cond_probs: Optional[Sequence[np.ndarray]] = None) -> "ScenarioTree":
        N = len(branching)
        if N == 0:
            raise ValueError("from_branching: horizon must be positive")
        if any(b < 1 for b in branching):
            raise ValueError("from_branching: branching factors must be >= 1")
        anc, ev, prob, cp_ = [-1], [-1], [1.0], [1.0]
        first, count, seen = 0, 1, 0
        for t in range(N):
            b = branching[t]
            nxt = first + count
            for p in range(first, nxt):
                if not cond_probs:
                    cp = np.full(b, 1.0 / b)
                else:
                    if seen >= len(cond_probs):
                        raise ValueError("from_branching: missing conditional probability vector")
                    cp = np.asarray(cond_probs[seen], dtype=np.float64)
                    if cp.size != b:
                        raise ValueError("from_branching: conditional probability vector has wrong length")
                    _check_prob_vector(cp, "from_branching")
                seen += 1
                for k in range(b):
                    anc.append(p)
                    ev.append(k)
                    cp_.append(cp[k])
                    prob.append(prob[p] * cp[k])
            first = nxt
            count *= b
        nb = N
        while nb > 0 and branching[nb - 1] == 1:
            nb -= 1
        return ScenarioTree(anc, ev, prob, cp_, nb, max(branching))

    # ScenarioTree::from_markov, proj/src/tree.cpp:141-207
    @staticmethod
    def from_markov(transition: np.ndarray, initial: np.ndarray, horizon: int, stop_stage: int) -> "ScenarioTree":
        T = np.asarray(transition, dtype=np.float64)
        p0 = np.asarray(initial, dtype=np.float64)
        nw = T.shape[0]
        if T.shape[1] != nw:
            raise ValueError("from_markov: transition must be square")
        if p0.size != nw:
            raise ValueError("from_markov: initial distribution has wrong length")
        if horizon < 1:
            raise ValueError("from_markov: horizon must be positive")
        if stop_stage < 0 or stop_stage > horizon:
            raise ValueError("from_markov: stop stage outside [0, horizon]")
        for w in range(nw):
            if np.any(T[w] < 0) or abs(T[w].sum() - 1.0) > PROB_TOL:
                raise ValueError("from_markov: transition rows must be stochastic")
        if np.any(p0 < 0) or abs(p0.sum() - 1.0) > PROB_TOL:
            raise ValueError("from_markov: initial distribution must be stochastic")
        row0 = T.T @ p0
        anc, ev, prob, cp = [-1], [-1], [1.0], [1.0]
        first, nxt = 0, 1
        for t in range(horizon):
            end = nxt
            for p in range(first, end):
                row = row0 if t == 0 else T[ev[p]]
                if t < stop_stage:
                    any_ = False
                    for w in range(nw):
                        if row[w] <= 0.0:
                            continue
                        anc.append(p)
                        ev.append(w)
                        cp.append(float(row[w]))
                        prob.append(prob[p] * float(row[w]))
                        any_ = True
                    if not any_:
                        raise ValueError("from_markov: node with no positive successor")
                else:
                    best = 0
                    for w in range(1, nw):
                        if row[w] > row[best]:
                            best = w
                    anc.append(p)
                    ev.append(best)
                    cp.append(1.0)
                    prob.append(prob[p])
            first = end
            nxt = len(anc)
        return ScenarioTree(anc, ev, prob, cp, stop_stage, nw)


@dataclass
class ConePart:
    kind: int
    dim: int


@dataclass
class RiskSpec:
    """Conic risk rho(Z) = max{mu'Z : b - E mu - F nu in K} (risk.hpp:18-48)."""
    kind: int
    n: int
    E: np.ndarray
    F: np.ndarray
    b: np.ndarray
    cone: List[ConePart]
    gamma: float = 1.0
    pi: Optional[np.ndarray] = None

    def rows(self) -> int:
        return int(self.E.shape[0])


def dual_cone(parts: List[ConePart]) -> List[ConePart]:
    """Dual of a cone product (proj/src/risk.cpp:25-43): Zero <-> Free, the
    nonnegative orthant and the SOC are self-dual.  S3 projects the risk rows
    of eta onto this cone (projections.cpp:212-244)."""
    swap = {CONE_ZERO: CONE_FREE, CONE_FREE: CONE_ZERO}
    return [ConePart(swap.get(c.kind, c.kind), c.dim) for c in parts]


def avar_spec(gamma: float, pi: np.ndarray) -> RiskSpec:
    """AV@R_gamma with base probabilities pi (proj/src/risk.cpp:65-98)."""
    if gamma < 0.0 or gamma > 1.0:
        raise ValueError("avar_spec: gamma outside [0, 1]")
    pi = np.asarray(pi, dtype=np.float64)
    _check_prob_vector(pi, "risk")
    n = pi.size
    if gamma > 0.0:
        E = np.zeros((2 * n + 1, n))
        E[:n] = gamma * np.eye(n)
        E[n:2 * n] = -np.eye(n)
        E[2 * n] = 1.0
        b = np.zeros(2 * n + 1)
        b[:n] = pi
        b[2 * n] = 1.0
        cone = [ConePart(CONE_NONNEG, 2 * n), ConePart(CONE_ZERO, 1)]
    else:
        E = np.zeros((n + 1, n))
        E[:n] = -np.eye(n)
        E[n] = 1.0
        b = np.zeros(n + 1)
        b[n] = 1.0
        cone = [ConePart(CONE_NONNEG, n), ConePart(CONE_ZERO, 1)]
    return RiskSpec(RISK_AVAR, n, E, np.zeros((E.shape[0], 0)), b, cone, float(gamma), pi.copy())


def expectation_spec(pi: np.ndarray) -> RiskSpec:
    """Equality-form expectation E = I, b = pi, K = {0} (risk.cpp:100-114)."""
    pi = np.asarray(pi, dtype=np.float64)
    _check_prob_vector(pi, "risk")
    n = pi.size
    return RiskSpec(RISK_AVAR, n, np.eye(n), np.zeros((n, 0)), pi.copy(), [ConePart(CONE_ZERO, n)], 1.0, pi.copy())


@dataclass
class Box:
    lo: np.ndarray
    hi: np.ndarray

    def dim(self) -> int:
        return int(self.lo.size)


@dataclass
class Raocp:
    """Risk-averse OCP on a scenario tree (problem.hpp:29-58).

    Per-node arrays are stacked along axis 0 where the shape is uniform
    (A: (nn-1, nx, nx) ...); constraint data may be per-node lists.
    """
    tree: ScenarioTree
    nx: int
    nu: int
    A: np.ndarray
    B: np.ndarray
    c: np.ndarray
    Q: np.ndarray
    R: np.ndarray
    q: np.ndarray
    r: np.ndarray
    QN: np.ndarray
    qN: np.ndarray
    Gx: list
    Gu: list
    C: List[Box]
    risk: List[RiskSpec]
    GN: list
    CN: List[Box]
    x_init: np.ndarray
    meta: dict = field(default_factory=dict)

    def stage_cost(self, node: int, x: np.ndarray, u: np.ndarray) -> float:
        k = node - 1
        return float(x @ self.Q[k] @ x + u @ self.R[k] @ u + self.q[k] @ x + self.r[k] @ u)

    def terminal_cost(self, leaf: int, x: np.ndarray) -> float:
        k = leaf - self.tree.num_nonleaf()
        return float(x @ self.QN[k] @ x + self.qN[k] @ x)
