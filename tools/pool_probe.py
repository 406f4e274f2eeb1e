"""Pooled blocks (Engine::compute_pool) on an unperturbed instance: T with
the records pointing every node at its class representative's blocks vs the
per-node blocks (SPOCK_POOL=0): bitwise equality, device ms per T (L2
flushed), the distinct block bytes, and the fp64 FLOP rate of T.
Usage (GPU box): python tools/pool_probe.py [config] [perturb]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def build(p, pool):
    os.environ["SPOCK_POOL"] = "1" if pool else "0"
    try:
        from paper_2505_12078_b200.solver import SpockSolver
        return SpockSolver(p)
    finally:
        os.environ.pop("SPOCK_POOL", None)


def main():
    import numpy as np
    import bench
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.rng import Philox
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5s"
    pert = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    p = make_config(cfg, seed=1, perturb=pert)
    sb = bench.survey_bytes(p)
    out = {"config": cfg, "perturb": pert, "nodes": p.tree.num_nodes(), "nx": p.nx, "flops_T": sb["F_T"]}
    res = {}
    for pool in (True, False):
        s = build(p, pool)
        z = -1.0 + 2.0 * Philox(3).uniform_array(s.nz)
        e = -1.0 + 2.0 * Philox(4).uniform_array(s.neta)
        zt, et = s.apply_T(z, e)
        s.bench_T(4, flush_l2=True)
        ms = s.bench_T(20, flush_l2=True) / 20
        res[pool] = (zt, et)
        key = "pooled" if pool else "per_node"
        out[key] = {"ms_per_T": ms, "tflops": sb["F_T"] / (ms / 1e3) / 1e12, "iter_per_s": 1e3 / ms}
        del s
    out["bitwise_equal"] = bool(np.array_equal(res[True][0], res[False][0]) and np.array_equal(res[True][1], res[False][1]))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
