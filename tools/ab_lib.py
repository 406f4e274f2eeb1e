"""Same-box A/B of two builds of libspock_b200.so (SPOCK_LIB): bitwise
comparison of outputs and timing.  Runs itself once per library in a
subprocess.  Usage (GPU box):
    python tools/ab_lib.py paper_2505_12078_b200/_build_alt/lib_base.so paper_2505_12078_b200/_build/libspock_b200.so"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(out):
    sys.path.insert(0, ROOT)
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    res, tim = {}, {}
    p1 = make_config("c1", seed=1)
    s = SpockSolver(p1, max_iters=3000, eps_abs=1e-14, eps_rel=1e-14)
    for method in ("solve_cp", "solve"):
        getattr(s, method)(p1.x_init)
        t = time.perf_counter()
        r = getattr(s, method)(p1.x_init)
        tim["c1_" + method + "_us_per_iter"] = round((time.perf_counter() - t) * 1e6 / r.status["iterations"], 2)
        res["c1_" + method] = r.z
    for cfg in ("c1", "c2", "c2p"):  # default schedule (fused T on these)
        p = make_config(cfg, seed=1)
        g = SpockSolver(p)
        rng = np.random.default_rng(3)
        z, e = rng.standard_normal(g.nz), rng.standard_normal(g.neta)
        zo, eo = g.apply_T(z, e)
        res[cfg + "_T_" + g.t_path + "_z"], res[cfg + "_T_" + g.t_path + "_eta"] = zo, eo
        g.bench_T(20)
        tim[cfg + "_T_" + g.t_path + "_us"] = round(min(g.bench_T(400) for _ in range(3)) * 1e3 / 400, 2)
    for cfg in ("c1", "c2"):
        os.environ.update({"SPOCK_T_UNFUSED": "1", "SPOCK_T_WIDE": "0"})
        p = make_config(cfg, seed=1)
        g = SpockSolver(p)
        rng = np.random.default_rng(3)
        z, e = rng.standard_normal(g.nz), rng.standard_normal(g.neta)
        zo, eo = g.apply_T(z, e)
        res[cfg + "_T_stages_z"], res[cfg + "_T_stages_eta"] = zo, eo
        g.bench_T(20)
        tim[cfg + "_T_stages_us"] = round(min(g.bench_T(200) for _ in range(3)) * 1e3 / 200, 2)
    np.savez(out, **res)
    print(json.dumps(tim), flush=True)


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        return
    outs = []
    for lib in sys.argv[1:]:
        out = tempfile.mktemp(suffix=".npz")
        r = subprocess.run([sys.executable, __file__, "--child", out], env={**os.environ, "SPOCK_LIB": lib},
                           capture_output=True, text=True)
        print(lib, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:], flush=True)
        outs.append(np.load(out))
    a = outs[0]
    for b in outs[1:]:
        print({k: bool(np.array_equal(a[k], b[k])) for k in a.files})


if __name__ == "__main__":
    main()
