"""BASELINE configs[4] at one GPU's scale (c5s: n_x 100, n_u 50, 103 765 nodes):
setup time, device T time (L2 flushed), algorithmic bytes and the fraction of
the HBM copy peak; also the DFMA work per T against the measured f64 peak.
Usage (GPU box): python tools/c5_probe.py [config] > gpurun_out/c5.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5s"
    import torch
    import bench
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    t0 = time.time()
    p = make_config(cfg, seed=1)
    t1 = time.time()
    s = SpockSolver(p)
    t2 = time.time()
    s.bench_T(4, flush_l2=True)
    torch.cuda.synchronize()
    k = 20
    ms = s.bench_T(k, flush_l2=True) / k
    b, launches = s.traffic_model()
    sb = bench.survey_bytes(p)
    peak, kind = bench._peaks()
    print(json.dumps({
        "config": cfg, "nodes": p.tree.num_nodes(), "nx": p.nx, "nu": p.nu, "path": s.t_path,
        "gen_s": t1 - t0, "setup_s": t2 - t1, "ms_per_T": ms, "iter_per_s": 1000.0 / ms,
        "lean_bytes": b[4], "frac_lean": b[4] / (ms / 1000.0) / 1e9 / peak,
        "survey_bytes": sb["B_T"], "frac_survey": sb["B_T"] / (ms / 1000.0) / 1e9 / peak,
        "flops": sb["F_T"], "tflops": sb["F_T"] / (ms / 1000.0) / 1e12, "peak_gbs": peak, "peak_kind": kind,
        "device_mem_gb": torch.cuda.max_memory_allocated() / 1e9 if torch.cuda.is_available() else None}))


if __name__ == "__main__":
    main()
