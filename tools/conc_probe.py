"""Concurrency determinism probe: engines solving side by side from host threads
must give the sequential results bitwise.  python tools/conc_probe.py [config] [threads] [reps]"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2p"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
algo = os.environ.get("PROBE_ALGO", "solve")
p = make_config(cfg, seed=2)
kw = dict(max_iters=300, eps_abs=1e-9, eps_rel=1e-9)
x = p.x_init
ref = getattr(SpockSolver(p, **kw), algo)(x)
sv = [SpockSolver(p, **kw) for _ in range(nt)]
cap = int(os.environ.get("PROBE_CAP", "0"))
for s in sv:
    s.set_grid_cap(cap)
out = [[] for _ in range(nt)]


def run(k):
    for _ in range(reps):
        out[k].append(getattr(sv[k], algo)(x))


th = [threading.Thread(target=run, args=(k,)) for k in range(nt)]
for h in th:
    h.start()
for h in th:
    h.join()
bad = 0
for k in range(nt):
    for j, r in enumerate(out[k]):
        same = r.status["branches"] == ref.status["branches"] and np.array_equal(r.z, ref.z)
        if not same:
            bad += 1
            br, rb = r.status["branches"], ref.status["branches"]
            first = next((i for i in range(min(len(br), len(rb))) if br[i] != rb[i]), -1)
            dn = np.abs(r.status["rnorm_history"] - ref.status["rnorm_history"][:len(r.status["rnorm_history"])])
            firstn = int(np.argmax(dn > 0)) if np.any(dn > 0) else -1
            rn_a, rn_b = r.status["rnorm_history"], ref.status["rnorm_history"]
            ctx = slice(max(firstn - 2, 0), firstn + 3)
            print(f"thread {k} rep {j}: differs; first branch diff at {first}, first rnorm diff at {firstn}; "
                  f"branches {rb[max(firstn - 3, 0):firstn + 3]!r}; rel diff {dn[firstn] / abs(rn_b[firstn]):.3e}; "
                  f"rn {rn_a[ctx]} vs {rn_b[ctx]}")
print(f"{cfg} {algo} threads={nt} reps={reps} cap={cap} env={ {k: v for k, v in os.environ.items() if k.startswith('SPOCK_')} }: "
      f"{bad} of {nt * reps} differ")
