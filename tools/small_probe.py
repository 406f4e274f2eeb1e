"""c1 solve to tolerance on the cluster-resident loop (cluster.cuh), the
CTA-resident loop (small.cuh) and the device graph loop, beside the CPU
oracle: time, iterations, per-iteration cost.
Usage (GPU box): python tools/small_probe.py [config]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import oracle
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    tols = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1e-3, 1e-4, 1e-6]
    p = make_config(cfg, seed=1)
    for method in ("solve_cp", "solve"):
        for tol in tols:
            row = {"config": cfg, "method": method, "tol": tol}
            paths = os.environ.get("PROBE_PATHS", "cluster,small,graph").split(",")
            for path in paths:
                os.environ["SPOCK_SMALL"] = "1" if path == "small" else "0"
                os.environ["SPOCK_CLUSTER"] = "1" if path == "cluster" else "0"
                s = SpockSolver(p, max_iters=50000, eps_abs=tol, eps_rel=tol)
                os.environ.pop("SPOCK_SMALL", None)
                os.environ.pop("SPOCK_CLUSTER", None)
                getattr(s, method)(p.x_init)
                t = time.perf_counter()
                r = getattr(s, method)(p.x_init)
                ms = 1000 * (time.perf_counter() - t)
                row[path] = {"loop": s.loop_path, "ms": round(ms, 2), "iters": r.status["iterations"],
                             "reason": r.status["reason"], "us_per_iter": round(1000 * ms / max(1, r.status["iterations"]), 2)}
            o = oracle.OracleSolver(p, alpha=s.alpha, max_iters=50000, eps_abs=tol, eps_rel=tol)
            t = time.perf_counter()
            b = getattr(o, method)(p.x_init)
            ms = 1000 * (time.perf_counter() - t)
            row["cpu"] = {"ms": round(ms, 2), "iters": b.status["iterations"], "reason": b.status["reason"]}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
