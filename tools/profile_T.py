"""Profiling driver (ncu --profile-from-start off): builds the config's solver,
warms up, then profiles `--steps` CP applications T (L2 flushed between them)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--flush", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    s = SpockSolver(make_config(a.config, seed=1))
    s.bench_T(4, use_graph=False, flush_l2=bool(a.flush))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    s.bench_T(a.steps, use_graph=False, flush_l2=bool(a.flush))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
