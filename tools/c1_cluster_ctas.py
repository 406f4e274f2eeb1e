"""c1 CP iteration time on the cluster-resident loop per cluster size (SPOCK_CLUSTER_CTAS).
Usage (GPU box): python tools/c1_cluster_ctas.py 2 4 8"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
p = make_config("c1", seed=1)
for ctas in sys.argv[1:]:
    os.environ["SPOCK_CLUSTER_CTAS"] = ctas
    s = SpockSolver(p, max_iters=3000, eps_abs=1e-14, eps_rel=1e-14)
    row = {"ctas": ctas, "loop": s.loop_path}
    for method in ("solve_cp", "solve"):
        getattr(s, method)(p.x_init)
        t = time.perf_counter(); r = getattr(s, method)(p.x_init); dt = time.perf_counter() - t
        row[method + "_us_per_iter"] = round(dt * 1e6 / r.status["iterations"], 2)
    print(json.dumps(row), flush=True)
