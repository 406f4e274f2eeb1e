"""Device time of one CP application T per (config, schedule knobs) variant.

Each variant runs in its own process (the schedule is chosen from the
environment when the solver is built).  Usage on the GPU box:
  python tools/sweep_T.py c3,c4 "SPOCK_T_WIDE=0" "SPOCK_WIDE_WARPS=4 SPOCK_WIDE_SLOTS=3" ...
An empty variant list runs the default schedule.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfgs = sys.argv[1] if len(sys.argv) > 1 else "c3"
    envs = sys.argv[2:] or [""]
    code = ("import sys, json; sys.path.insert(0, '.'); import bench; "
            "from paper_2505_12078_b200.generators import make_config; "
            "from paper_2505_12078_b200.solver import SpockSolver; "
            "out = []\n"
            "for c in sys.argv[1].split(','):\n"
            "    p = make_config(c, seed=1); s = SpockSolver(p); s.bench_T(4, flush_l2=True)\n"
            "    ms = s.bench_T(30, flush_l2=True) / 30; b, n = s.traffic_model()\n"
            "    out.append(dict(config=c, nodes=p.tree.num_nodes(), path=s.t_path, ms_per_T=round(ms, 4), "
            "GBs=round(b[4] / ms / 1e6, 1), frac=round(b[4] / ms / 1e6 / 6551.0, 3)))\n"
            "print(json.dumps(out))")
    for env in envs:
        e = dict(os.environ)
        for kv in env.split():
            k, v = kv.split("=", 1)
            e[k] = v
        r = subprocess.run([sys.executable, "-c", code, cfgs], cwd=ROOT, env=e, capture_output=True, text=True)
        print(env or "default", r.stdout.strip()[-900:], r.stderr.strip()[-400:], flush=True)


if __name__ == "__main__":
    main()
