"""Engines constructed concurrently from host threads must equal a sequentially
constructed one (alpha, T) bitwise.  python tools/setup_race_probe.py [config] [threads]"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2p"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = make_config(cfg, seed=2)
ref = SpockSolver(p)
z = np.random.default_rng(1).standard_normal(ref.nz)
e = np.random.default_rng(2).standard_normal(ref.neta)
tz, te = ref.apply_T(z, e)
for trial in range(3):
    sv = [None] * nt

    def make(k):
        sv[k] = SpockSolver(p)

    th = [threading.Thread(target=make, args=(k,)) for k in range(nt)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    for k, s in enumerate(sv):
        az, ae = s.apply_T(z, e)
        print(f"trial {trial} engine {k}: alpha diff {s.alpha - ref.alpha:.3e}  T diff "
              f"{np.max(np.abs(az - tz)) + np.max(np.abs(ae - te)):.3e}", flush=True)
