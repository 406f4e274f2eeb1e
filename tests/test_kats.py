"""Known-answer tests that pin the input side shared by the product and the
oracle: published Philox4x32-10 vectors, the AV@R stacking and dual cones
(proj/tests/test_risk.cpp:29-87) and the scenario-tree builders
(proj/tests/test_tree.cpp:13-165)."""
import numpy as np
import pytest

from oracle import oracle
from paper_2505_12078_b200.problem import (CONE_FREE, CONE_NONNEG, CONE_SOC, CONE_ZERO, ConePart, ScenarioTree,
                                           avar_spec, dual_cone, expectation_spec)
from paper_2505_12078_b200.rng import Philox, _philox_blocks

# Random123 (Salmon et al., SC'11) kat_vectors, philox4x32 with 10 rounds:
# counter words c0..c3, key words k0 k1 -> output words.  Independent of this
# repo and of the reference: they pin the block function itself.
PHILOX_KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff),
     (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("ctr,key,out", PHILOX_KAT)
def test_philox4x32_10_published_vectors(ctr, key, out):
    c = sum(int(w) << (32 * i) for i, w in enumerate(ctr))
    got = _philox_blocks(key[0], key[1], c, 1)
    assert [int(x) for x in got] == list(out)


def test_philox_stream_starts_at_counter_zero():
    """rng.cpp:22-29: seed -> key, counter 0 (stream 0); the first u64 of seed 0
    is words 0|1 of the first published vector -- in Python and in the C++ oracle."""
    w = PHILOX_KAT[0][2]
    expect = w[0] | (w[1] << 32)
    assert int(Philox(0).next_u64_array(1)[0]) == expect
    assert int(oracle.philox_u64(0, 1)[0]) == expect
    # key (0xffffffff, 0xffffffff) = seed 2^64-1, counter 0 -> not the all-ones vector
    # (its counter differs), but the stream must still be the block function's
    k = (1 << 64) - 1
    blk = _philox_blocks(0xffffffff, 0xffffffff, 0, 1)
    assert int(Philox(k).next_u64_array(1)[0]) == int(blk[0]) | (int(blk[1]) << 32)
    assert int(oracle.philox_u64(k, 1)[0]) == int(blk[0]) | (int(blk[1]) << 32)


def test_avar_stacking_kat():  # test_risk.cpp:29-44
    s = avar_spec(0.5, np.array([0.5, 0.5]))
    assert s.rows() == 5
    E = np.array([[0.5, 0], [0, 0.5], [-1, 0], [0, -1], [1, 1]], dtype=float)
    assert np.abs(s.E - E).max() == 0.0
    assert np.abs(s.b - np.array([0.5, 0.5, 0, 0, 1])).max() == 0.0
    assert s.F.shape[1] == 0
    assert len(s.cone) == 2
    assert (s.cone[0].kind, s.cone[0].dim) == (CONE_NONNEG, 4)
    assert (s.cone[1].kind, s.cone[1].dim) == (CONE_ZERO, 1)


def test_avar_max_and_expectation_forms():  # risk.cpp:65-114
    pi = np.array([0.2, 0.3, 0.5])
    m = avar_spec(0.0, pi)
    assert m.rows() == 4 and np.array_equal(m.E[:3], -np.eye(3)) and np.array_equal(m.E[3], np.ones(3))
    assert [(c.kind, c.dim) for c in m.cone] == [(CONE_NONNEG, 3), (CONE_ZERO, 1)]
    e = expectation_spec(pi)
    assert np.array_equal(e.E, np.eye(3)) and np.array_equal(e.b, pi)
    assert [(c.kind, c.dim) for c in e.cone] == [(CONE_ZERO, 3)]


def test_avar_rejects_bad_input():  # test_risk.cpp:59-64
    for g, pi in ((1.5, [0.5, 0.5]), (-0.1, [0.5, 0.5]), (0.5, [0.6, 0.6]), (0.5, [1.0, 0.0])):
        with pytest.raises(ValueError):
            avar_spec(g, np.array(pi))


def test_dual_cone_kat():  # test_risk.cpp:65-75
    d = dual_cone([ConePart(CONE_NONNEG, 4), ConePart(CONE_ZERO, 1)])
    assert d[0].kind == CONE_NONNEG and d[1].kind == CONE_FREE
    assert dual_cone([ConePart(CONE_SOC, 5)])[0].kind == CONE_SOC


def test_dual_of_dual_is_identity():  # test_risk.cpp:77-87
    rng = Philox(11)
    for _ in range(50):
        parts = []
        for _ in range(int(rng.uniform_int(1, 4))):
            dim = int(rng.uniform_int(1, 4))
            k = int(rng.uniform_int(0, 3))
            parts.append({0: ConePart(CONE_ZERO, dim), 1: ConePart(CONE_NONNEG, dim),
                          2: ConePart(CONE_SOC, dim + 1)}.get(k, ConePart(CONE_FREE, dim)))
        dd = dual_cone(dual_cone(parts))
        assert [(c.kind, c.dim) for c in dd] == [(c.kind, c.dim) for c in parts]


# ---- scenario trees (test_tree.cpp) ----
def test_branching_2_1_uniform():  # :13-22
    t = ScenarioTree.from_branching([2, 1])
    assert t.num_nodes() == 5 and t.horizon == 2
    assert t.stage_begin(2) == 3 and t.stage_end(2) == 5
    assert t.prob[3] == pytest.approx(0.5, rel=1e-14) and t.prob[4] == pytest.approx(0.5, rel=1e-14)
    assert t.stop_stage == 1


def test_deterministic_chain():  # :24-29
    t = ScenarioTree.from_branching([1] * 7)
    assert t.num_nodes() == 8
    assert all(t.prob[i] == 1.0 for i in range(8))
    assert t.stop_stage == 0


def test_branching_explicit_probabilities():  # :31-45
    cp = [np.array([0.5, 0.3, 0.2])] + [np.array([0.5, 0.5])] * 3 + [np.ones(1)] * 6
    t = ScenarioTree.from_branching([3, 2, 1], cp)
    assert t.num_nodes() == 16
    c0 = t.child_first[1]
    for k in range(2):
        leaf = t.child_first[c0 + k]
        assert t.stage[leaf] == 3
        assert t.prob[leaf] == pytest.approx(0.25, rel=1e-14)


def test_branching_rejects_bad_inputs():  # :47-55
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([2, 0])
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([2], [np.array([0.7, 0.2])])
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([2], [np.array([1.0, 0.0])])


def test_markov_absorbing_chain():  # :57-65
    t = ScenarioTree.from_markov(np.eye(2), np.array([1.0, 0.0]), 3, 3)
    assert t.num_nodes() == 4
    for i in range(1, 4):
        assert t.event[i] == 0 and t.prob[i] == 1.0


def test_markov_uniform_full_binary():  # :67-73
    t = ScenarioTree.from_markov(np.full((2, 2), 0.5), np.array([0.5, 0.5]), 2, 2)
    assert t.num_nodes() == 7
    for j in range(t.stage_begin(2), t.stage_end(2)):
        assert t.prob[j] == pytest.approx(0.25, rel=1e-14)


def test_markov_pruning_kat():  # :75-93
    tm = np.array([[0.9, 0.1], [0.0, 1.0]])
    t = ScenarioTree.from_markov(tm, np.array([1.0, 0.0]), 2, 1)
    assert t.num_nodes() == 5
    assert t.stage_end(1) - t.stage_begin(1) == 2 and t.stage_end(2) - t.stage_begin(2) == 2
    assert t.event[1] == 0 and t.event[2] == 1
    assert t.cond_prob[1] == pytest.approx(0.9) and t.cond_prob[2] == pytest.approx(0.1)
    assert t.child_count[1] == 1 and t.child_count[2] == 1
    assert t.event[t.child_first[1]] == 0 and t.event[t.child_first[2]] == 1
    assert t.cond_prob[t.child_first[1]] == 1.0


def test_markov_rejects_non_stochastic():  # :95-99
    with pytest.raises(ValueError):
        ScenarioTree.from_markov(np.array([[0.9, 0.2], [0.5, 0.5]]), np.array([0.5, 0.5]), 2, 2)


def test_random_branching_invariants():  # :101-119
    rng = Philox(7)
    for _ in range(20):
        N = int(rng.uniform_int(1, 5))
        br = [int(rng.uniform_int(1, 3)) for _ in range(N)]
        t = ScenarioTree.from_branching(br)
        for s in range(t.horizon + 1):
            assert abs(t.prob[t.stage_begin(s):t.stage_end(s)].sum() - 1.0) < 1e-12
        for i in range(t.num_nodes()):
            for c in t.children(i):
                assert t.anc[c] == i
        assert np.all(np.diff(t.stage) >= 0)


def test_array_round_trip():  # :154-165
    t = ScenarioTree.from_branching([2, 3, 1])
    t2 = ScenarioTree(t.anc, t.event, t.prob, t.cond_prob, t.stop_stage, t.num_events)
    assert t2.num_nodes() == t.num_nodes()
    assert np.array_equal(t2.anc, t.anc) and np.array_equal(t2.stage, t.stage) and np.array_equal(t2.prob, t.prob)
