"""test_cp_agrees_with_supermann instances (test_solver.cpp:297-318) on every
loop: |z0(SuperMann) - z0(CP)| and each solution's distance to a tight CP
solution (oracle, eps 1e-10).  Usage (GPU box): python tools/cp_vs_sm_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from support import TinyOpts, make_tiny, small_trees  # noqa: E402
from test_solver import _ill_conditioned  # noqa: E402
from oracle.oracle import OracleSolver  # noqa: E402
from paper_2505_12078_b200.rng import Philox  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402


def mk(env, p, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return SpockSolver(p, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


rng = Philox(30)
for n, tree in enumerate(small_trees()):
    p = make_tiny(tree, 2, 1, rng.next_u64(), TinyOpts(gamma=0.6))
    if _ill_conditioned(p, 1e-5):
        continue
    kw = dict(eps_abs=1e-6, eps_rel=1e-6, max_iters=200000)
    ref = OracleSolver(p, eps_abs=1e-11, eps_rel=1e-11, max_iters=2000000).solve_cp().z
    row = [f"inst {n}"]
    for name, env in (("oracle", None), ("graph", {"SPOCK_CLUSTER": "0"}), ("cluster", {"SPOCK_CLUSTER": "1"})):
        s = OracleSolver(p, **kw) if env is None else mk(env, p, **kw)
        a, b = s.solve(), s.solve_cp()
        sc = max(1.0, abs(ref[0]))
        row.append(f"{name}: sm {a.status['reason'][:4]} {a.status['iterations']} it |dz0| {abs(a.z[0]-b.z[0])/sc:.1e} "
                   f"err sm {np.abs(a.z-ref).max()/sc:.1e} cp {np.abs(b.z-ref).max()/sc:.1e}")
    print(" | ".join(row), flush=True)
