"""T on device buffers from several host threads (maximal kernel overlap), each
output compared bitwise with the sequential reference.
python tools/conc_T_dev_probe.py [config] [threads] [cap] [reps]"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2p"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 148
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2000
op = os.environ.get("PROBE_OP", "T")
p = make_config(cfg, seed=2)
ref = SpockSolver(p)
rng = np.random.default_rng(1)
Z = [torch.tensor(rng.standard_normal(ref.nz), device="cuda") for _ in range(4)]
E = [torch.tensor(rng.standard_normal(ref.neta), device="cuda") for _ in range(4)]
OZ = [torch.zeros_like(z) for z in Z]
OE = [torch.zeros_like(e) for e in E]


def apply(s, q, oz, oe):
    if op == "T":
        s.apply_T(Z[q], E[q], oz, oe)
    elif op == "L":
        s.apply_L(Z[q], oe)
    elif op == "Lt":
        s.apply_Lt(E[q], oz)
    else:  # M-norm (dots on device)
        oz[0] = s.m_norm(Z[q], E[q], 0.7)


for q in range(4):
    apply(ref, q, OZ[q], OE[q])
torch.cuda.synchronize()
sv = [SpockSolver(p) for _ in range(nt)]
for s in sv:
    s.set_grid_cap(cap)
bad = [0] * nt


def run(k):
    oz = [torch.zeros_like(z) for z in Z]
    oe = [torch.zeros_like(e) for e in E]
    for j in range(reps):
        q = (j + k) % 4
        apply(sv[k], q, oz[q], oe[q])
        if not (torch.equal(oz[q], OZ[q]) and torch.equal(oe[q], OE[q])):
            bad[k] += 1


th = [threading.Thread(target=run, args=(k,)) for k in range(nt)]
for h in th:
    h.start()
for h in th:
    h.join()
print(f"op={op} {cfg} threads={nt} cap={cap} reps={reps} env={ {k: v for k, v in os.environ.items() if k.startswith('SPOCK_')} }"
      f": differing T per thread {bad}", flush=True)
