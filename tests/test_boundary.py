"""The drop-in boundary: C-ABI library loads, exports every declared symbol,
and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2505_12078_b200 import capi
from paper_2505_12078_b200.problem import ScenarioTree
from support import make_tiny

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "spock_b200.h")).read()
    return sorted(set(re.findall(r"\b(spock_[A-Za-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = capi.load_library()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(capi.EXPORTED_SYMBOLS) == names


def test_params_default_matches_reference():
    lib = capi.load_library()
    p = capi.Params()
    lib.spock_params_default(ctypes.byref(p))
    assert p.eps_abs == 1e-6 and p.eps_rel == 1e-6 and p.aa_memory == 3
    assert p.c0 == p.c1 == p.c2 == 0.99 and p.beta == 0.5 and p.sigma == 0.1 and p.lambda_ == 1.0
    assert p.max_iters == 50000 and p.max_backtracks == 40 and p.use_preconditioner == 1


def test_invalid_problem_rejected_before_device_work():
    """std::invalid_argument kinds surface as ValueError through the C-ABI."""
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_tiny(ScenarioTree.from_branching([2]), 2, 1, 3)
    p.R[0] = -np.eye(1)  # R must be PD (problem.cpp:69-70)
    with pytest.raises(ValueError, match="positive definite"):
        SpockSolver(p)
    p = make_tiny(ScenarioTree.from_branching([2]), 2, 1, 3)
    with pytest.raises(ValueError, match="aa_memory"):
        SpockSolver(p, aa_memory=0)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_tiny(ScenarioTree.from_branching([2]), 2, 1, 3)
    with pytest.raises(RuntimeError, match="CUDA"):
        SpockSolver(p)
