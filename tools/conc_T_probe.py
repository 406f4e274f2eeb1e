"""T applications from several host threads at once (engines with a capped fused
grid) against a sequential reference, bitwise.  python tools/conc_T_probe.py [config] [threads] [cap] [reps]"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2p"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 74
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
p = make_config(cfg, seed=2)
ref = SpockSolver(p)
rng = np.random.default_rng(1)
zs = [rng.standard_normal(ref.nz) for _ in range(4)]
es = [rng.standard_normal(ref.neta) for _ in range(4)]
outs = [ref.apply_T(z, e) for z, e in zip(zs, es)]
sv = [SpockSolver(p) for _ in range(nt)]
for s in sv:
    s.set_grid_cap(cap)
bad = [0] * nt


def run(k):
    for j in range(reps):
        q = (j + k) % 4
        az, ae = sv[k].apply_T(zs[q], es[q])
        if not (np.array_equal(az, outs[q][0]) and np.array_equal(ae, outs[q][1])):
            bad[k] += 1


th = [threading.Thread(target=run, args=(k,)) for k in range(nt)]
for h in th:
    h.start()
for h in th:
    h.join()
print(f"{cfg} threads={nt} cap={cap} reps={reps} env={ {k: v for k, v in os.environ.items() if k.startswith('SPOCK_')} }"
      f" path={sv[0].t_path}: differing T per thread {bad}", flush=True)
