"""Philox stream and tree builders (proj/tests/test_tree.cpp, rng.cpp)."""
import numpy as np
import pytest

from oracle import oracle
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.rng import Philox


def test_philox_u64_stream_bit_exact_vs_cpp():
    for seed in (0, 1, 22, 0x9E3779B97F4A7C15):
        ref = oracle.philox_u64(seed, 1000)
        got = Philox(seed).next_u64_array(1000)
        assert np.array_equal(ref, got)


def test_philox_normals_match_cpp():
    for seed in (0, 5, 0x9E3779B97F4A7C15):
        ref = oracle.philox_normals(seed, 2001)
        r = Philox(seed)
        got = np.concatenate([r.normal_array(7), r.normal_array(1000), r.normal_array(994)])
        np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-15)
        r2 = Philox(seed)
        got2 = np.array([r2.normal() for _ in range(50)])
        np.testing.assert_allclose(got2, ref[:50], rtol=1e-14, atol=1e-15)


def test_branching_tree_structure():
    t = ScenarioTree.from_branching([3, 2, 1])
    assert t.num_nodes() == 1 + 3 + 6 + 6
    assert t.horizon == 3 and t.stop_stage == 2
    assert list(t.stage_start) == [0, 1, 4, 10, 16]
    assert t.child_first[0] == 1 and t.child_count[0] == 3
    for s in range(t.horizon + 1):
        assert abs(t.prob[t.stage_begin(s):t.stage_end(s)].sum() - 1.0) < 1e-12


def test_markov_tree_prunes_and_stops():
    tm = np.array([[0.9, 0.1], [0.4, 0.6]])
    t = ScenarioTree.from_markov(tm, np.array([0.7, 0.3]), 3, 2)
    assert t.num_nodes() == 1 + 2 + 4 + 4
    # past the stop stage each node keeps its most probable successor
    for i in range(t.stage_begin(2), t.stage_end(2)):
        assert t.child_count[i] == 1
        c = t.child_first[i]
        assert t.event[c] == int(np.argmax(tm[t.event[i]]))
        assert t.cond_prob[c] == 1.0


def test_builder_argument_errors():
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([])
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([2, 0])
    with pytest.raises(ValueError):
        ScenarioTree.from_branching([2], [np.array([0.5, 0.6])])
