"""Cycle accounting of the streaming kernel's standalone L (SPOCK_WIDE_PROF=1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SPOCK_WIDE_PROF"] = "1"
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = SpockSolver(make_config(cfg, seed=1))
z = np.random.default_rng(0).standard_normal(s.nz)
for _ in range(20):
    s.apply_L(z)
s.__del__()
