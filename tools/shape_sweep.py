"""BASELINE configs[3]: tree-structure sweep at ~1e5 nodes (varying branching
factor, stopping stage and horizon, PAPER Fig. 8).  For each
shape: one CP application T, device time with L2 flushed, algorithmic bytes and
fraction of the measured HBM copy peak.  Usage (GPU box):
    python tools/shape_sweep.py [N,nw,nb ...] > gpurun_out/shapes.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(12, 4, 7), (12, 10, 4), (12, 100, 2), (48, 3, 7), (100, 10, 3)]


def main():
    from paper_2505_12078_b200.generators import make_config, tree_nodes_up_to
    from paper_2505_12078_b200.solver import SpockSolver
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or SHAPES
    rows = []
    for N, nw, nb in shapes:
        t = time.time()
        p = make_config("c4", seed=1, N=N, nw=nw, nb=nb)
        gen = time.time() - t
        t = time.time()
        s = SpockSolver(p)
        setup = time.time() - t
        s.bench_T(3, flush_l2=True)
        k = 20
        ms = s.bench_T(k, flush_l2=True) / k
        b, launches = s.traffic_model()
        row = {"N": N, "nw": nw, "nb": nb, "nodes": p.tree.num_nodes(), "scenarios": p.tree.num_leaves(),
               "levels": 2 * N + 2, "schedule": s.t_path, "ms_per_T": ms, "T_bytes": b[4],
               "GBs": b[4] / ms / 1e6, "frac": b[4] / ms / 1e6 / peak, "gen_s": gen, "setup_s": setup}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del s


if __name__ == "__main__":
    main()
