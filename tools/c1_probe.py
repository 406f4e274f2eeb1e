"""Device time of T and of a CP iteration on the small configs per schedule knob
(environment set by the caller): python tools/c1_probe.py [config]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = make_config(cfg, seed=1)
s = SpockSolver(p, max_iters=3000, eps_abs=1e-30, eps_rel=1e-30)
s.bench_T(50)
t_us = 1000 * s.bench_T(1000) / 1000
s.solve_cp(p.x_init)
t = time.perf_counter()
r = s.solve_cp(p.x_init)
it_us = 1e6 * (time.perf_counter() - t) / r.status["iterations"]
env = {k: v for k, v in os.environ.items() if k.startswith("SPOCK_")}
print(json.dumps({"config": cfg, "env": env, "path": s.t_path, "T_us": t_us, "cp_iter_us": it_us}), flush=True)
