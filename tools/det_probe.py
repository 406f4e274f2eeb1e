import sys, os, numpy as np
sys.path.insert(0, '.')
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
p = make_config("c2p", seed=2)
kw = dict(max_iters=300, eps_abs=1e-9, eps_rel=1e-9)
a = SpockSolver(p, **kw); b = SpockSolver(p, **kw); b.set_grid_cap(74)
c = SpockSolver(p, **kw)
x = p.x_init
ra = [a.solve(x) for _ in range(3)]
rb = b.solve(x); rc = c.solve(x)
def d(u, v): return (u.status["branches"] == v.status["branches"], float(np.max(np.abs(u.z - v.z))))
print("A rep", d(ra[0], ra[1]), d(ra[0], ra[2]), "A vs C", d(ra[0], rc), "A vs B(cap)", d(ra[0], rb))
# T determinism
z = np.random.default_rng(1).standard_normal(a.nz); e = np.random.default_rng(2).standard_normal(a.neta)
ta = [a.apply_T(z, e) for _ in range(5)]; tb = b.apply_T(z, e)
print("T rep", [float(np.max(np.abs(t[0] - ta[0][0]))) + float(np.max(np.abs(t[1] - ta[0][1]))) for t in ta[1:]], "T cap", float(np.max(np.abs(tb[0] - ta[0][0]))) + float(np.max(np.abs(tb[1] - ta[0][1]))))
