import sys, time, json
sys.path.insert(0, '.')
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
for cfg, cap in (("c2", 60000), ("c3", 3000)):
    p = make_config(cfg, seed=1)
    s = SpockSolver(p, max_iters=cap)
    t = time.perf_counter(); r = s.solve(p.x_init); dt = time.perf_counter() - t
    st = r.status
    print(json.dumps(dict(config=cfg, solve_s=dt, reason=st["reason"], iters=st["iterations"], n_T=st["n_T"], n_L=st["n_L"], n_Lt=st["n_Lt"], k=[st["k0_steps"], st["k1_steps"], st["k2_steps"], st["stalled_steps"]], xi=[st["xi1_inf"], st["xi2_inf"]], path=s.t_path)), flush=True)
