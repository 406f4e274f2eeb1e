"""Probe: (1) device time of one T on c2 against the fused grid cap
(SPOCK_FUSED_GRID), (2) B concurrent SuperMann solves (one solver and stream per
x_init, host threads) against B sequential ones.  Prints JSON lines."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(os.environ.get("PROBE_ITERS", "5000"))
p = make_config(cfg, seed=1)
for g in ([0, 16, 24, 32, 48, 64, 96, 148] if "--grid" in sys.argv else []):
    os.environ["SPOCK_FUSED_GRID"] = str(g)
    s = SpockSolver(p)
    s.bench_T(20)
    print(json.dumps({"probe": "grid", "config": cfg, "grid_cap": g, "T_ms": s.bench_T(200)}), flush=True)
    del s

rng = np.random.default_rng(3)
xs = [p.x_init * (1.0 + 0.2 * rng.standard_normal(p.x_init.shape)) for _ in range(64)]
plan = os.environ.get("PROBE_B", "1:0,2:74,4:74,8:37")
for B, g in [tuple(int(v) for v in item.split(":")) for item in plan.split(",")]:
    os.environ["SPOCK_FUSED_GRID"] = str(g)
    sv = [SpockSolver(p, max_iters=iters) for _ in range(B)]
    for s, x in zip(sv, xs):
        s.solve(x)  # warm (graph build)
    t = time.perf_counter()
    seq = [s.solve(x).status["iterations"] for s, x in zip(sv, xs)]
    t_seq = time.perf_counter() - t
    res = [None] * B

    def run(k):
        res[k] = sv[k].solve(xs[k]).status

    th = [threading.Thread(target=run, args=(k,)) for k in range(B)]
    t = time.perf_counter()
    for h in th:
        h.start()
    for h in th:
        h.join()
    t_par = time.perf_counter() - t
    print(json.dumps({"probe": "batch", "config": cfg, "B": B, "grid_cap": g, "seq_s": t_seq, "conc_s": t_par,
                      "iters": seq, "conc_iters": [r["iterations"] for r in res],
                      "reasons": [r["reason"] for r in res]}), flush=True)
    del sv
