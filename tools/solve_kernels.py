"""One short SuperMann solve on c2 (for an ncu launch list of the device loop):
python tools/solve_kernels.py [config] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
it = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = make_config(cfg, seed=1)
s = SpockSolver(p, max_iters=it)
algo = sys.argv[3] if len(sys.argv) > 3 else "solve"
r = getattr(s, algo)(p.x_init)
st = r.status
print({k: st[k] for k in ("iterations", "n_T", "n_L", "n_Lt", "k0_steps", "k1_steps", "k2_steps", "branches")})
