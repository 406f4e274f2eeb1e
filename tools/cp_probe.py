import sys, time, json
sys.path.insert(0, '.')
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
for cfg, cap in (("c2", 300000),):
    p = make_config(cfg, seed=1)
    s = SpockSolver(p, max_iters=cap)
    t = time.perf_counter(); r = s.solve_cp(p.x_init); dt = time.perf_counter() - t
    st = r.status
    print(json.dumps(dict(config=cfg, s=dt, reason=st["reason"], iters=st["iterations"], xi=[st["xi1_inf"], st["xi2_inf"]])), flush=True)
