"""us per T of the default schedule on narrow configurations (CUDA-graph
replay, device-timed, best of 3 x 400; no L2 flush).  Usage:
python tools/fused_T_time.py [configs...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_12078_b200.generators import make_config  # noqa: E402
from paper_2505_12078_b200.solver import SpockSolver  # noqa: E402


def main():
    row = {}
    for cfg in sys.argv[1:] or ["c1", "c2", "c2p"]:
        s = SpockSolver(make_config(cfg, seed=1))
        s.bench_T(50)
        row[cfg] = {"path": s.t_path, "us_per_T": round(min(s.bench_T(400) for _ in range(3)) * 1e3 / 400, 2)}
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
