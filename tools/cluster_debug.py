import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
from support import TinyOpts, make_tiny
def mk(env, p, **kw):
    old = {k: os.environ.get(k) for k in env}; os.environ.update(env)
    try: return SpockSolver(p, **kw)
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
for name, p in [("tiny", make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 31, TinyOpts(gamma=0.5, box_halfwidth=1.0))), ("c1", make_config("c1", seed=1))]:
    s = mk({"SPOCK_CLUSTER": "1"}, p, max_iters=40, eps_abs=1e-14, eps_rel=1e-14)
    g = mk({"SPOCK_CLUSTER": "0"}, p, max_iters=40, eps_abs=1e-14, eps_rel=1e-14, alpha=s.alpha)
    print(name, s.loop_path, g.loop_path, flush=True)
    for m in ("solve", "solve_cp"):
        a = getattr(s, m)(p.x_init); b = getattr(g, m)(p.x_init)
        print(m, "branches eq", a.status["branches"] == b.status["branches"], "zs", np.abs(a.z_scaled).max(), np.abs(b.z_scaled).max(),
              "dzs", np.abs(a.z_scaled - b.z_scaled).max(), "deta", np.abs(a.eta - b.eta).max(), "dz", np.abs(a.z - b.z).max(), flush=True)
