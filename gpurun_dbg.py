import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from oracle.oracle import OracleSolver
from paper_2505_12078_b200.solver import SpockSolver
from paper_2505_12078_b200.problem import ScenarioTree
from support import TinyOpts, make_tiny
p = make_tiny(ScenarioTree.from_branching([2, 2]), 2, 1, 31, TinyOpts(gamma=0.5, box_halfwidth=1.0))
g = SpockSolver(p, max_iters=6, eps_abs=1e-14, eps_rel=1e-14)
o = OracleSolver(p, alpha=g.alpha, max_iters=6, eps_abs=1e-14, eps_rel=1e-14)
for k in (1, 2, 3, 4):
    g2 = SpockSolver(p, max_iters=k, eps_abs=1e-14, eps_rel=1e-14)
    o2 = OracleSolver(p, alpha=g2.alpha, max_iters=k, eps_abs=1e-14, eps_rel=1e-14)
    a, b = g2.solve(), o2.solve()
    print(k, a.status['branches'], b.status['branches'], a.status['rnorm_history'], b.status['rnorm_history'],
          np.abs(a.z_scaled - b.z_scaled).max(), a.status['n_T'], b.status['n_T'], a.status['xi1_inf'], b.status['xi1_inf'])
