"""Problem / solution files ("spock-problem v1", proj/src/problem_io.cpp):
format, byte-identical round trips, and that a reloaded problem is the same
problem for the solver (the CPU oracle here; the B200 library reads the same
Raocp)."""
import numpy as np
import pytest

from oracle.oracle import OracleSolver
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.problem import RISK_GENERAL, ConePart, RiskSpec, ScenarioTree
from paper_2505_12078_b200.problem_io import (Document, ProblemIOError, cone_from_string, cone_to_string,
                                              load_problem, load_solution, save_problem, save_solution)
from paper_2505_12078_b200.rng import Philox
from support import TinyOpts, make_tiny


def _problems():
    yield "c1", make_config("c1", seed=1)
    yield "tiny-avar", make_tiny(ScenarioTree.from_branching([2, 3]), 3, 2, 7, TinyOpts(gamma=0.4))
    p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 3, TinyOpts(gamma=0.5))
    # a general conic risk (max form written as a general spec) on the root
    n = 2
    E = np.vstack([-np.eye(n), np.ones((1, n))])
    p.risk[0] = RiskSpec(RISK_GENERAL, n, E, np.zeros((n + 1, 0)), np.r_[np.zeros(n), 1.0],
                         [ConePart(1, n), ConePart(0, 1)])
    yield "general-risk", p


PROBLEMS = list(_problems())


def test_document_format_header(tmp_path):
    d = Document()
    d.put_int("num_nodes", 7)
    d.put_str("note", "two words")
    d.put_vec("v", [1.0, 2.0])
    d.put_ints("ix", [3, -4])
    d.put_mat("M", [[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
    path = tmp_path / "doc.spk"
    d.save(str(path), "spock-problem v1")
    raw = path.read_bytes()
    lines = raw.split(b"\n")
    assert lines[0] == b"spock-problem v1"
    assert lines[1] == b"meta i num_nodes 7"
    assert lines[2] == b"meta s note two words"
    assert lines[3] == b"arr v f64 2 1"
    # payloads: little-endian, row-major
    off = raw.index(b"arr v f64 2 1\n") + len(b"arr v f64 2 1\n")
    assert np.frombuffer(raw[off:off + 16], dtype="<f8").tolist() == [1.0, 2.0]
    off = raw.index(b"arr M f64 2 3\n") + len(b"arr M f64 2 3\n")
    assert np.frombuffer(raw[off:off + 48], dtype="<f8").tolist() == [1, 2, 3, 4, 5, 6]
    assert raw.endswith(b"end\n")
    e = Document.load(str(path), "spock-problem v1")
    assert e.get_int("num_nodes") == 7 and e.get_str("note") == "two words"
    assert e.get_ints("ix").tolist() == [3, -4]
    np.testing.assert_array_equal(e.get_mat("M"), [[1, 2, 3], [4, 5, 6]])
    assert e.has("M") and not e.has("missing")


def test_document_errors(tmp_path):
    path = tmp_path / "bad.spk"
    path.write_bytes(b"not a spock file\n")
    with pytest.raises(ProblemIOError, match="bad magic"):
        Document.load(str(path), "spock-problem v1")
    path.write_bytes(b"spock-problem v1\narr x f64 4 1\n\x00\x00")
    with pytest.raises(ProblemIOError, match="truncated"):
        Document.load(str(path), "spock-problem v1")
    path.write_bytes(b"spock-problem v1\nmeta i n 1\n")
    with pytest.raises(ProblemIOError, match="missing end"):
        Document.load(str(path), "spock-problem v1")
    d = Document()
    with pytest.raises(ProblemIOError, match="missing integer"):
        d.get_int("n")


def test_cone_descriptor_round_trip():
    parts = [ConePart(0, 1), ConePart(1, 3), ConePart(2, 4), ConePart(3, 2)]
    s = cone_to_string(parts)
    assert s == "zero:1,nn:3,soc:4,free:2"
    assert cone_from_string(s) == parts
    with pytest.raises(ProblemIOError):
        cone_from_string("cube:3")


@pytest.mark.parametrize("name,p", PROBLEMS, ids=[n for n, _ in PROBLEMS])
def test_problem_round_trip_byte_identical(tmp_path, name, p):
    a, b = tmp_path / "a.spk", tmp_path / "b.spk"
    save_problem(str(a), p)
    q = load_problem(str(a))
    save_problem(str(b), q)
    assert a.read_bytes() == b.read_bytes()
    assert q.nx == p.nx and q.nu == p.nu and q.tree.num_nodes() == p.tree.num_nodes()
    np.testing.assert_array_equal(q.tree.anc, p.tree.anc)
    np.testing.assert_array_equal(q.A, p.A)
    np.testing.assert_array_equal(q.R, p.R)


@pytest.mark.parametrize("name,p", PROBLEMS, ids=[n for n, _ in PROBLEMS])
def test_reloaded_problem_is_the_same_problem(tmp_path, name, p):
    path = tmp_path / "p.spk"
    save_problem(str(path), p)
    q = load_problem(str(path))
    o1, o2 = OracleSolver(p), OracleSolver(q)
    assert o1.alpha == o2.alpha
    nz = o1.primal_layout()["n"]
    ne = o1.apply_L(np.zeros(nz)).size
    z = -1.0 + 2.0 * Philox(3).uniform_array(nz)
    e = -1.0 + 2.0 * Philox(4).uniform_array(ne)
    za, ea = o1.apply_T(z, e)
    zb, eb = o2.apply_T(z, e)
    np.testing.assert_array_equal(za, zb)
    np.testing.assert_array_equal(ea, eb)


def test_solution_round_trip(tmp_path):
    p = make_config("c1", seed=1)
    r = OracleSolver(p, max_iters=30).solve(p.x_init)
    path = tmp_path / "s.spk"
    save_solution(str(path), r)
    s = load_solution(str(path))
    assert s["iterations"] == r.status["iterations"] and s["reason"] == r.status["reason"]
    np.testing.assert_array_equal(s["z"], r.z)
    np.testing.assert_array_equal(s["eta"], r.eta)
    assert s["xi1_inf"] == r.status["xi1_inf"]


def test_expectation_reloads_as_avar_at_one(tmp_path):
    """problem_io.cpp:269-272,330-331: an expectation spec is stored as AV@R with
    gamma 1 and reloads as avar_spec(1, pi) (same risk value, AV@R structure)."""
    p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 3, TinyOpts(gamma=1.0))
    path = tmp_path / "e.spk"
    save_problem(str(path), p)
    q = load_problem(str(path))
    assert q.risk[0].gamma == 1.0
    assert q.risk[0].E.shape[0] == 2 * q.risk[0].n + 1
