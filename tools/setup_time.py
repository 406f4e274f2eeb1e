"""Wall time of the problem generator and of solver construction (setup)
per config; with SPOCK_DEBUG_SETUP=1 the engine prints each setup phase.
Usage (GPU box): SPOCK_DEBUG_SETUP=1 python tools/setup_time.py c2,c3,c4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

for c in (sys.argv[1] if len(sys.argv) > 1 else "c3").split(","):
    t = time.time()
    p = make_config(c, seed=1)
    t1 = time.time()
    s = SpockSolver(p)
    print(c, "gen %.2f s, solver %.2f s," % (t1 - t, time.time() - t1), s.t_path, flush=True)
