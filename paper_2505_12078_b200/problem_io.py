"""Problem and solution files of the reference ("spock-problem v1",
"spock-solution v1"; proj/src/problem_io.cpp, proj/include/spock/problem_io.hpp).

A self-describing container: a text header line with the magic, ``meta``
lines for integer (``i``) and string (``s``) fields, ``arr`` records with a
text header (``arr <name> f64|i64 <rows> <cols>``) followed by the little-endian
row-major payload and a newline, and ``end``.  Insertion order is kept, so
load-then-save round-trips byte for byte (problem_io.hpp:13-16), and a file
written here is read by the reference's loader and vice versa.  This lets the
CPU oracle, the B200 solver and the reference consume byte-identical problems
(SURVEY.md §8f-1).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

from .problem import (CONE_FREE, CONE_NONNEG, CONE_SOC, CONE_ZERO, RISK_AVAR, RISK_GENERAL, Box, ConePart, Raocp,
                      RiskSpec, ScenarioTree, avar_spec)

PROBLEM_MAGIC = "spock-problem v1"    # problem_io.cpp:10
SOLUTION_MAGIC = "spock-solution v1"  # problem_io.cpp:11


class ProblemIOError(RuntimeError):
    """std::runtime_error("problem_io: ...") of the reference (problem_io.cpp:13)."""


def _fail(msg: str):
    raise ProblemIOError("problem_io: " + msg)


@dataclass
class _Arr:
    name: str
    dtype: str  # 'f' or 'l'
    rows: int
    cols: int
    data: np.ndarray  # float64 or int64, row-major (rows, cols)


@dataclass
class Document:
    """Document (problem_io.hpp:16-50)."""
    meta: List[Tuple[str, str, str]] = field(default_factory=list)  # (tag, name, value)
    arrays: List[_Arr] = field(default_factory=list)

    # -- writers (problem_io.cpp:17-61)
    def put_int(self, name: str, v: int) -> None:
        self.meta.append(("i", name, str(int(v))))

    def put_str(self, name: str, v: str) -> None:
        self.meta.append(("s", name, v))

    def put_mat(self, name: str, m) -> None:
        m = np.asarray(m, dtype=np.float64)
        if m.ndim == 1:
            m = m.reshape(-1, 1)
        self.arrays.append(_Arr(name, "f", m.shape[0], m.shape[1], np.ascontiguousarray(m)))

    def put_vec(self, name: str, v) -> None:
        v = np.asarray(v, dtype=np.float64).reshape(-1)
        self.arrays.append(_Arr(name, "f", v.size, 1, v.reshape(-1, 1).copy()))

    def put_ints(self, name: str, v) -> None:
        v = np.asarray(v, dtype=np.int64).reshape(-1)
        self.arrays.append(_Arr(name, "l", v.size, 1, v.reshape(-1, 1).copy()))

    # -- readers (problem_io.cpp:63-103)
    def get_int(self, name: str) -> int:
        for tag, n, v in self.meta:
            if tag == "i" and n == name:
                return int(v)
        _fail("missing integer field " + name)

    def get_str(self, name: str) -> str:
        for tag, n, v in self.meta:
            if tag == "s" and n == name:
                return v
        _fail("missing string field " + name)

    def _find(self, name: str) -> _Arr:
        for a in self.arrays:
            if a.name == name:
                return a
        _fail("missing array " + name)

    def has(self, name: str) -> bool:
        return any(n == name for _, n, _ in self.meta) or any(a.name == name for a in self.arrays)

    def get_mat(self, name: str) -> np.ndarray:
        a = self._find(name)
        if a.dtype != "f":
            _fail("array " + name + " is not f64")
        return a.data.reshape(a.rows, a.cols).copy()

    def get_vec(self, name: str) -> np.ndarray:
        a = self._find(name)
        if a.dtype != "f" or a.cols != 1:
            _fail("array " + name + " is not an f64 vector")
        return a.data.reshape(-1).copy()

    def get_ints(self, name: str) -> np.ndarray:
        a = self._find(name)
        if a.dtype != "l":
            _fail("array " + name + " is not i64")
        return a.data.reshape(-1).astype(np.int64)

    # -- files (problem_io.cpp:105-166)
    def save(self, path: str, magic: str) -> None:
        out = bytearray()
        out += (magic + "\n").encode()
        for tag, name, value in self.meta:
            out += f"meta {tag} {name} {value}\n".encode()
        for a in self.arrays:
            out += f"arr {a.name} {'f64' if a.dtype == 'f' else 'i64'} {a.rows} {a.cols}\n".encode()
            dt = "<f8" if a.dtype == "f" else "<i8"
            out += np.ascontiguousarray(a.data, dtype=dt).tobytes(order="C")
            out += b"\n"
        out += b"end\n"
        try:
            with open(path, "wb") as f:
                f.write(bytes(out))
        except OSError:
            _fail("cannot open " + path + " for writing")

    @staticmethod
    def load(path: str, expected_magic: str) -> "Document":
        try:
            with open(path, "rb") as f:
                buf = f.read()
        except OSError:
            _fail("cannot open " + path)
        pos = 0

        def line() -> str:
            nonlocal pos
            e = buf.find(b"\n", pos)
            if e < 0:
                return None
            s = buf[pos:e].decode()
            pos = e + 1
            return s

        first = line()
        if first != expected_magic:
            _fail(f"{path}: bad magic (expected '{expected_magic}')")
        doc = Document()
        while True:
            ln = line()
            if ln is None:
                _fail("missing end marker in " + path)
            if ln == "end":
                return doc
            kind, _, rest = ln.partition(" ")
            if kind == "meta":
                tag, _, rest2 = rest.partition(" ")
                name, _, value = rest2.partition(" ")
                doc.meta.append((tag, name, value))
            elif kind == "arr":
                parts = rest.split()
                name, dtype, rows, cols = parts[0], parts[1], int(parts[2]), int(parts[3])
                if rows < 0 or cols < 0:
                    _fail("negative array dims")
                dt = "f" if dtype == "f64" else "l"
                count = rows * cols
                nbytes = 8 * count
                if pos + nbytes > len(buf):
                    _fail("truncated payload for array " + name)
                data = np.frombuffer(buf, dtype="<f8" if dt == "f" else "<i8", count=count, offset=pos)
                pos += nbytes + 1  # trailing newline
                doc.arrays.append(_Arr(name, dt, rows, cols, data.reshape(rows, cols).copy()))
            else:
                _fail("unknown record '" + kind + "'")


_CONE_NAMES = {CONE_ZERO: "zero", CONE_NONNEG: "nn", CONE_SOC: "soc", CONE_FREE: "free"}
_CONE_KINDS = {v: k for k, v in _CONE_NAMES.items()}


def cone_to_string(parts: List[ConePart]) -> str:  # problem_io.cpp:170-185
    return ",".join(f"{_CONE_NAMES[p.kind]}:{p.dim}" for p in parts)


def cone_from_string(s: str) -> List[ConePart]:  # problem_io.cpp:187-208
    out = []
    for part in [x for x in s.split(",") if x != ""]:
        kind, sep, dim = part.partition(":")
        if not sep:
            _fail("bad cone descriptor " + s)
        if kind not in _CONE_KINDS:
            _fail("bad cone kind " + kind)
        out.append(ConePart(_CONE_KINDS[kind], int(dim)))
    return out


def _stack(mats) -> np.ndarray:  # stack_mats / stack_vecs, problem_io.cpp:210-224
    mats = [np.asarray(m, dtype=np.float64) for m in mats]
    if not mats:
        return np.zeros((0, 0))
    if mats[0].ndim == 1:
        return np.concatenate(mats)
    return np.concatenate(mats, axis=0)


def save_problem(path: str, p: Raocp, include_soc_translations: bool = False) -> None:
    """save_problem (problem_io.cpp:242-295)."""
    if include_soc_translations:
        raise ValueError("save_problem: SOC translations are derived data; the loaders rederive them "
                         "(problem_io.hpp:54-56) and this writer does not embed them")
    tr = p.tree
    nn, nnl, nl = tr.num_nodes(), tr.num_nonleaf(), tr.num_leaves()
    d = Document()
    d.put_int("num_nodes", nn)
    d.put_int("horizon", tr.horizon)
    d.put_int("stop_stage", tr.stop_stage)
    d.put_int("num_events", tr.num_events)
    d.put_int("nx", p.nx)
    d.put_int("nu", p.nu)
    d.put_ints("tree.anc", tr.anc)
    d.put_ints("tree.event", tr.event)
    d.put_vec("tree.prob", tr.prob)
    d.put_vec("tree.cond_prob", tr.cond_prob)
    d.put_vec("x_init", p.x_init)
    d.put_mat("dyn.A", _stack(p.A))
    d.put_mat("dyn.B", _stack(p.B))
    d.put_vec("dyn.c", _stack(p.c))
    d.put_mat("cost.Q", _stack(p.Q))
    d.put_mat("cost.R", _stack(p.R))
    d.put_vec("cost.q", _stack(p.q))
    d.put_vec("cost.r", _stack(p.r))
    d.put_mat("term.QN", _stack(p.QN))
    d.put_vec("term.qN", _stack(p.qN))
    for i in range(nnl):
        pre = f"cstr.{i}."
        d.put_mat(pre + "Gx", p.Gx[i])
        d.put_mat(pre + "Gu", p.Gu[i])
        d.put_vec(pre + "lo", p.C[i].lo)
        d.put_vec(pre + "hi", p.C[i].hi)
        rp = f"risk.{i}."
        rs = p.risk[i]
        if rs.kind == RISK_AVAR:
            d.put_str(rp + "kind", "avar")
            d.put_vec(rp + "gamma", [rs.gamma])
            d.put_vec(rp + "pi", rs.pi)
        else:
            d.put_str(rp + "kind", "general")
            d.put_str(rp + "cone", cone_to_string(rs.cone))
            d.put_mat(rp + "E", rs.E)
            d.put_mat(rp + "F", np.asarray(rs.F, dtype=np.float64).reshape(rs.E.shape[0], -1))
            d.put_vec(rp + "b", rs.b)
    for j in range(nl):
        pre = f"cstrN.{j}."
        d.put_mat(pre + "G", p.GN[j])
        d.put_vec(pre + "lo", p.CN[j].lo)
        d.put_vec(pre + "hi", p.CN[j].hi)
    d.save(path, PROBLEM_MAGIC)


def load_problem(path: str) -> Raocp:
    """load_problem (problem_io.cpp:297-358).  As in the reference, an
    expectation risk is stored as AV@R at gamma 1 and reloads as avar_spec(1, pi)."""
    d = Document.load(path, PROBLEM_MAGIC)
    nn, nx, nu = d.get_int("num_nodes"), d.get_int("nx"), d.get_int("nu")
    tree = ScenarioTree(d.get_ints("tree.anc"), d.get_ints("tree.event"), d.get_vec("tree.prob"),
                        d.get_vec("tree.cond_prob"), d.get_int("stop_stage"), d.get_int("num_events"))
    if tree.num_nodes() != nn or tree.horizon != d.get_int("horizon"):
        _fail("tree arrays disagree with num_nodes / horizon")
    nnl, nl = tree.num_nonleaf(), tree.num_leaves()

    def unstack(m, count, rows):
        return np.stack([m[k * rows:(k + 1) * rows] for k in range(count)]) if count else \
            np.zeros((0, rows) + m.shape[1:])

    A = unstack(d.get_mat("dyn.A"), nn - 1, nx)
    B = unstack(d.get_mat("dyn.B"), nn - 1, nx)
    c = unstack(d.get_vec("dyn.c"), nn - 1, nx)
    Q = unstack(d.get_mat("cost.Q"), nn - 1, nx)
    R = unstack(d.get_mat("cost.R"), nn - 1, nu)
    q = unstack(d.get_vec("cost.q"), nn - 1, nx)
    r = unstack(d.get_vec("cost.r"), nn - 1, nu)
    QN = unstack(d.get_mat("term.QN"), nl, nx)
    qN = unstack(d.get_vec("term.qN"), nl, nx)
    Gx, Gu, C, risk = [], [], [], []
    for i in range(nnl):
        pre = f"cstr.{i}."
        Gx.append(d.get_mat(pre + "Gx"))
        Gu.append(d.get_mat(pre + "Gu"))
        C.append(Box(d.get_vec(pre + "lo"), d.get_vec(pre + "hi")))
        rp = f"risk.{i}."
        if d.get_str(rp + "kind") == "avar":
            risk.append(avar_spec(float(d.get_vec(rp + "gamma")[0]), d.get_vec(rp + "pi")))
        else:
            E = d.get_mat(rp + "E")
            risk.append(RiskSpec(RISK_GENERAL, E.shape[1], E, d.get_mat(rp + "F"), d.get_vec(rp + "b"),
                                 cone_from_string(d.get_str(rp + "cone"))))
    GN, CN = [], []
    for j in range(nl):
        pre = f"cstrN.{j}."
        GN.append(d.get_mat(pre + "G"))
        CN.append(Box(d.get_vec(pre + "lo"), d.get_vec(pre + "hi")))
    return Raocp(tree=tree, nx=nx, nu=nu, A=A, B=B, c=c, Q=Q, R=R, q=q, r=r, QN=QN, qN=qN, Gx=Gx, Gu=Gu, C=C,
                 risk=risk, GN=GN, CN=CN, x_init=d.get_vec("x_init"))


_REASONS = {"converged": 0, "max_iters": 1, "stalled": 2, "cancelled": 3}


def save_solution(path: str, res) -> None:
    """save_solution (problem_io.cpp:360-375); res is a SolveResult of either
    solver (status dict with the reference's field names)."""
    st = res.status
    d = Document()
    d.put_int("iterations", st["iterations"])
    d.put_str("reason", st["reason"])
    d.put_int("k0", st["k0_steps"])
    d.put_int("k1", st["k1_steps"])
    d.put_int("k2", st["k2_steps"])
    d.put_int("stalled", st["stalled_steps"])
    d.put_vec("xi", [st["xi1_inf"], st["xi2_inf"]])
    d.put_vec("alpha", [st.get("alpha", 0.0)])
    d.put_vec("z", res.z)
    d.put_vec("z_scaled", res.z_scaled)
    d.put_vec("eta", res.eta)
    d.save(path, SOLUTION_MAGIC)


def load_solution(path: str) -> Dict:
    """load_solution (problem_io.cpp:377-408), as a plain dict."""
    d = Document.load(path, SOLUTION_MAGIC)
    reason = d.get_str("reason")
    xi = d.get_vec("xi")
    return {"iterations": d.get_int("iterations"),
            "reason": reason if reason in _REASONS else "cancelled",
            "k0_steps": d.get_int("k0"), "k1_steps": d.get_int("k1"), "k2_steps": d.get_int("k2"),
            "stalled_steps": d.get_int("stalled"), "xi1_inf": float(xi[0]), "xi2_inf": float(xi[1]),
            "alpha": float(d.get_vec("alpha")[0]), "z": d.get_vec("z"), "z_scaled": d.get_vec("z_scaled"),
            "eta": d.get_vec("eta")}
