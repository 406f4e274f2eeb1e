"""BatchSolver host-side checks (no GPU): argument validation happens before any
solver is built; the GPU behaviour is in test_batch_gpu.py."""
import pytest

from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.solver import BatchSolver
from support import TinyOpts, make_tiny


def test_streams_must_be_positive():
    p = make_tiny(ScenarioTree.from_branching([2]), 2, 1, 3, TinyOpts())
    with pytest.raises(ValueError):
        BatchSolver(p, streams=0)


def test_c_abi_exports_grid_cap():
    from paper_2505_12078_b200 import capi
    assert "spock_solver_set_grid_cap" in capi.EXPORTED_SYMBOLS
    assert "spock_solver_grid" in capi.EXPORTED_SYMBOLS
