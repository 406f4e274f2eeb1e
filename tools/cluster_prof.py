"""Phase profile of the cluster-resident loop on c1 (SPOCK_SMALL_PROF=1 clock64
totals of CTA 0's thread 0) for a fixed number of CP iterations; prints cycles
per iteration by class.  Usage (GPU box): SPOCK_SMALL_PROF=1 python tools/cluster_prof.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
p = make_config("c1", seed=1)
s = SpockSolver(p, max_iters=n, eps_abs=1e-14, eps_rel=1e-14)
print(s.loop_path, flush=True)
r = s.solve_cp(p.x_init)
print("iterations", r.status["iterations"], "n_T", r.status["n_T"], "n_L", r.status["n_L"], "n_Lt", r.status["n_Lt"], flush=True)
