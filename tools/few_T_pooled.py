"""Two CP applications on an unperturbed (shared-matrix) instance through the
streaming kernel with pooled records (sanitizer target).
Usage: python tools/few_T_pooled.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SPOCK_T_UNFUSED", "1")
os.environ.setdefault("SPOCK_T_WIDE", "1")
import numpy as np  # noqa: E402
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

p = make_config(sys.argv[1] if len(sys.argv) > 1 else "c2p", seed=2, perturb=0.0)
s = SpockSolver(p)
z = np.random.default_rng(1).standard_normal(s.nz)
e = np.random.default_rng(2).standard_normal(s.neta)
for _ in range(2):
    s.apply_T(z, e)
print("ok", s.t_path)
