"""Wall time of a capped SuperMann solve through the C-ABI (host x_init in, host
solution out) under schedule variants given as environment strings."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import sys, time, json; sys.path.insert(0, '.')
from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.solver import SpockSolver
p = make_config(sys.argv[1], seed=1)
s = SpockSolver(p, max_iters=int(sys.argv[2]))
s.solve(p.x_init)
t = time.perf_counter(); r = s.solve(p.x_init); dt = time.perf_counter() - t
st = r.status
print(json.dumps(dict(ms=1000 * dt, nT=st['n_T'], nL=st['n_L'], nLt=st['n_Lt'], T_per_s=st['n_T'] / dt)))
"""


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    iters = sys.argv[2] if len(sys.argv) > 2 else "500"
    for env in sys.argv[3:] or [""]:
        e = dict(os.environ)
        for kv in env.split():
            k, v = kv.split("=", 1)
            e[k] = v
        r = subprocess.run([sys.executable, "-c", CODE, cfg, iters], cwd=ROOT, env=e, capture_output=True, text=True)
        print(env or "default", r.stdout.strip()[-300:], r.stderr.strip()[-300:], flush=True)


if __name__ == "__main__":
    main()
