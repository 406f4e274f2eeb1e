import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
p = make_config(sys.argv[1] if len(sys.argv) > 1 else "c2p", seed=2)
s = SpockSolver(p)
z = np.random.default_rng(1).standard_normal(s.nz); e = np.random.default_rng(2).standard_normal(s.neta)
for _ in range(2):
    s.apply_T(z, e)
print("ok", s.t_path)
