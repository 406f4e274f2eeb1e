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


@pytest.mark.gpu
def test_wrong_sizes_and_dtypes_raise_value_error():
    """The reference throws std::invalid_argument on wrong dimensions
    (solver.cpp:191,200-201); the Python mirror checks lengths and dtypes before
    any pointer reaches the library (a short buffer would be read or written out
    of bounds)."""
    import numpy as np
    import torch
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config("c1", seed=1)
    s = SpockSolver(p, max_iters=3)
    with pytest.raises(ValueError, match="x_init"):
        s.solve(np.zeros(p.nx + 1))
    with pytest.raises(ValueError, match="warm"):
        s.solve(p.x_init, warm=(np.zeros(s.nz - 1), np.zeros(s.neta)))
    with pytest.raises(ValueError):
        s.apply_T(np.zeros(s.nz - 1), np.zeros(s.neta))
    with pytest.raises(ValueError):
        s.apply_T(np.zeros(s.nz), np.zeros(s.neta), np.zeros(s.nz), np.zeros(s.neta - 2))
    with pytest.raises(ValueError):
        s.apply_T(torch.zeros(s.nz, dtype=torch.float32, device="cuda"),
                  torch.zeros(s.neta, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        s.apply_L(np.zeros(s.nz + 3))
    with pytest.raises(ValueError):
        s.apply_Lt(np.zeros(s.neta), out=np.zeros(s.nz, dtype=np.float32))
    z1, e1 = s.apply_T(np.zeros(s.nz), np.zeros(s.neta))  # the right sizes still work
    assert z1.shape == (s.nz,) and e1.shape == (s.neta,)


@pytest.mark.gpu
def test_dual_cone_projection_on_device():
    """S3 on the risk rows projects onto the dual cone (risk.cpp:25-43,
    projections.cpp:212-244): AV@R rows R+^{2n} x Free clamp the first 2n entries
    and leave the last; the expectation form Zero^n -> Free leaves all n."""
    import numpy as np
    from oracle.oracle import OracleSolver
    from paper_2505_12078_b200.problem import ScenarioTree
    from paper_2505_12078_b200.solver import SpockSolver
    from support import TinyOpts, make_tiny
    for gamma, ny_of in ((0.5, lambda n: 2 * n + 1), (1.0, lambda n: n)):
        p = make_tiny(ScenarioTree.from_branching([3, 2]), 2, 1, 5, TinyOpts(gamma=gamma))
        s = SpockSolver(p)
        o = OracleSolver(p, alpha=s.alpha)
        el = o.dual_layout()
        e = np.linspace(-3.0, 3.0, s.neta)
        got = s.proj_s3(e)
        np.testing.assert_allclose(got, o.proj_s3(e), rtol=1e-14, atol=1e-14)
        for i in range(p.tree.num_nonleaf()):
            n = int(p.tree.child_count[i])
            off, ny = int(el["seg1_off"][i]), int(el["seg1_ydim"][i])
            assert ny == ny_of(n)
            if gamma < 1.0:
                assert np.array_equal(got[off:off + 2 * n], np.maximum(e[off:off + 2 * n], 0.0))
                assert got[off + 2 * n] == e[off + 2 * n]
            else:
                assert np.array_equal(got[off:off + n], e[off:off + n])


def test_layout_flags_pack():
    """The product's packer hands numpy stacks over as they are (row-major
    blocks, one shared constraint block when G is a broadcast); the oracle's
    packer keeps the reference's column-major layout."""
    from paper_2505_12078_b200 import capi
    from paper_2505_12078_b200.generators import make_config
    p = make_config("c1", seed=1)
    fast = capi.pack_problem(p)
    slow = capi.pack_problem(p, fast=False)
    assert fast.desc.layout == capi.SPOCK_LAYOUT_ROW_MAJOR | capi.SPOCK_LAYOUT_SHARED_G
    assert slow.desc.layout == 0


@pytest.mark.gpu
def test_layout_flags_same_solver():
    """Row-major / shared-G descriptor and the reference's column-major one give
    bitwise the same solver (same alpha, same T)."""
    import ctypes as C
    from paper_2505_12078_b200 import capi
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.rng import Philox
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config("c2", seed=2)
    a = SpockSolver(p)
    orig = capi.pack_problem
    try:
        capi.pack_problem = lambda q, fast=True: orig(q, fast=False)
        b = SpockSolver(p)
    finally:
        capi.pack_problem = orig
    assert a.alpha == b.alpha
    z = -1.0 + 2.0 * Philox(5).uniform_array(a.nz)
    e = -1.0 + 2.0 * Philox(6).uniform_array(a.neta)
    za, ea = a.apply_T(z, e)
    zb, eb = b.apply_T(z, e)
    assert np.array_equal(za, zb) and np.array_equal(ea, eb)
