"""Command-line front end (the reference specifies it, SPEC.md module `cli`; its
tools/spock_main.cpp is a stub).  Verbs on top of the B200 solver:

  generate-random --seed S --count C --out DIR [--desk-scale]
      case-study-1 problems (generators.cpp:118-122) as "spock-problem v1" files
  solve FILE [--algorithm spock|cp] [--eps-abs --eps-rel --max-iters] [--out SOL]
      solve, print the SpockStatus, write a "spock-solution v1" file;
      exit 0 on convergence, 1 otherwise
  bench DIR --out CSV [--time-limit-s T] [--max-iters K]
      every problem of DIR with both algorithms: BenchRecord rows (SPEC.md cli
      BenchRecord) and Dolan-More performance-profile data (profile-emit)
  profile-emit CSV --out CSV
      (tau, fraction solved) per solver from a bench CSV; failures have ratio inf
  shapes [N,nw,nb ...]
      device time of one CP application T per tree shape (configs[3])

`python -m paper_2505_12078_b200 <verb> ...`.  generate-ncs (the networked-
control case study) is out of scope.
"""
from __future__ import annotations

import argparse
import csv
import glob
import json
import math
import os
import sys
import time



def _solver(problem, args, cancelled=None):
    from .solver import SpockSolver
    kw = dict(eps_abs=args.eps_abs, eps_rel=args.eps_rel, max_iters=args.max_iters)
    return SpockSolver(problem, cancelled=cancelled, **kw)


def cmd_generate_random(args) -> int:
    from .generators import gen_case1_instance
    from .problem_io import save_problem
    os.makedirs(args.out, exist_ok=True)
    for k in range(args.count):
        seed = args.seed + k
        p = gen_case1_instance(seed, args.desk_scale)
        path = os.path.join(args.out, f"case1_seed{seed}.spk")
        save_problem(path, p)
        print(path)
    return 0


def cmd_solve(args) -> int:
    from .problem_io import load_problem, save_solution
    p = load_problem(args.file)
    s = _solver(p, args)
    t = time.perf_counter()
    r = (s.solve if args.algorithm == "spock" else s.solve_cp)(p.x_init)
    dt = time.perf_counter() - t
    st = r.status
    st["alpha"] = s.alpha
    print(json.dumps({"file": args.file, "algorithm": args.algorithm, "reason": st["reason"],
                      "iterations": st["iterations"], "xi1_inf": st["xi1_inf"], "xi2_inf": st["xi2_inf"],
                      "k0_k1_k2_stalled": [st["k0_steps"], st["k1_steps"], st["k2_steps"], st["stalled_steps"]],
                      "n_T": st["n_T"], "solve_s": dt, "schedule": s.t_path}))
    if args.out:
        save_solution(args.out, r)
    return 0 if st["reason"] == "converged" else 1


def _n_v(p) -> int:  # SPEC.md cli BenchRecord invariant
    tr = p.tree
    return p.nx * tr.num_nodes() + p.nu * tr.num_nonleaf()


def cmd_bench(args) -> int:
    from .problem_io import load_problem
    files = sorted(glob.glob(os.path.join(args.dir, "*.spk")))
    rows = []
    for f in files:
        p = load_problem(f)
        for algo in ("spock", "cp"):
            t0 = time.perf_counter()
            deadline = t0 + args.time_limit_s
            s = _solver(p, args, cancelled=lambda: time.perf_counter() > deadline)
            r = (s.solve if algo == "spock" else s.solve_cp)(p.x_init)
            wall = time.perf_counter() - t0
            st = r.status
            rows.append({
                "problem": os.path.basename(f), "n_v": _n_v(p), "n_x": p.nx, "n_u": p.nu,
                "n_w": p.tree.num_events, "N": p.tree.horizon, "n_b": p.tree.stop_stage, "solver": algo,
                "wall_s": f"{wall:.6f}", "iterations": st["iterations"], "reason": st["reason"],
                "k0": st["k0_steps"], "k1": st["k1_steps"], "k2": st["k2_steps"], "stalled": st["stalled_steps"],
                "xi1": f"{st['xi1_inf']:.6e}", "xi2": f"{st['xi2_inf']:.6e}",
                "peak_device_bytes": _peak_device_bytes()})
            print(json.dumps(rows[-1]), flush=True)
    with open(args.out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()) if rows else ["problem"])
        w.writeheader()
        w.writerows(rows)
    if args.profile_out:
        _write_profile(rows, args.profile_out)
    return 0


def _peak_device_bytes() -> int:
    try:
        import torch
        return int(torch.cuda.max_memory_allocated()) if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        return 0


def performance_profile(rows):
    """Dolan-More profiles (PAPER §8.1.2): per problem, r = t_solver / min_s t_s
    (failure: inf); rho_s(tau) = fraction of problems with r <= tau."""
    by_prob = {}
    for r in rows:
        ok = r["reason"] == "converged"
        by_prob.setdefault(r["problem"], {})[r["solver"]] = float(r["wall_s"]) if ok else math.inf
    solvers = sorted({r["solver"] for r in rows})
    ratios = {s: [] for s in solvers}
    for times in by_prob.values():
        best = min(times.values())
        for s in solvers:
            t = times.get(s, math.inf)
            ratios[s].append(t / best if math.isfinite(t) and best > 0 else (1.0 if t == best else math.inf))
    taus = sorted({x for v in ratios.values() for x in v if math.isfinite(x)} | {1.0})
    out = []
    for s in solvers:
        n = max(1, len(ratios[s]))
        for tau in taus:
            out.append({"solver": s, "tau": tau, "fraction_solved": sum(1 for x in ratios[s] if x <= tau) / n})
    return out


def _write_profile(rows, path):
    prof = performance_profile(rows)
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=["solver", "tau", "fraction_solved"])
        w.writeheader()
        w.writerows(prof)


def cmd_profile_emit(args) -> int:
    with open(args.csv) as fh:
        rows = list(csv.DictReader(fh))
    _write_profile(rows, args.out)
    return 0


def cmd_shapes(args) -> int:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.argv = ["shape_sweep"] + args.shapes
    sys.path.insert(0, os.path.join(here, "tools"))
    import shape_sweep
    shape_sweep.main()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2505_12078_b200")
    sub = ap.add_subparsers(dest="verb", required=True)

    def solver_flags(p):
        p.add_argument("--eps-abs", type=float, default=1e-6)
        p.add_argument("--eps-rel", type=float, default=1e-6)
        p.add_argument("--max-iters", type=int, default=50000)

    g = sub.add_parser("generate-random")
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--count", type=int, default=1)
    g.add_argument("--out", required=True)
    g.add_argument("--desk-scale", action="store_true")
    s = sub.add_parser("solve")
    s.add_argument("file")
    s.add_argument("--algorithm", choices=["spock", "cp"], default="spock")
    s.add_argument("--out")
    solver_flags(s)
    b = sub.add_parser("bench")
    b.add_argument("dir")
    b.add_argument("--out", required=True)
    b.add_argument("--profile-out")
    b.add_argument("--time-limit-s", type=float, default=300.0)
    solver_flags(b)
    pe = sub.add_parser("profile-emit")
    pe.add_argument("csv")
    pe.add_argument("--out", required=True)
    sh = sub.add_parser("shapes")
    sh.add_argument("shapes", nargs="*")
    args = ap.parse_args(argv)
    return {"generate-random": cmd_generate_random, "solve": cmd_solve, "bench": cmd_bench,
            "profile-emit": cmd_profile_emit, "shapes": cmd_shapes}[args.verb](args)


if __name__ == "__main__":
    sys.exit(main())
