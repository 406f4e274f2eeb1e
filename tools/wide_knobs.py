"""Streaming-kernel knob sweep on one tree shape (same box, one generated
instance): ms per T (L2 flushed) and the lean-bytes roofline fraction per
variant.  Usage: python tools/wide_knobs.py N,nw,nb 'SPOCK_WIDE_SLOTS=4' 'SPOCK_WIDE_SLOTS=8 SPOCK_WIDE_CHUNK=1024' ..."""
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    N, nw, nb = (int(x) for x in sys.argv[1].split(","))
    p = make_config("c4", seed=1, N=N, nw=nw, nb=nb)
    variants = sys.argv[2:] or [""]
    for rep in range(2):
        for v in variants:
            env = dict(kv.split("=") for kv in v.split())
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            s = SpockSolver(p)
            for k, o in old.items():
                if o is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = o
            s.bench_T(3, flush_l2=True)
            ms = min(s.bench_T(10, flush_l2=True) / 10 for _ in range(2))
            b, _ = s.traffic_model()
            print(json.dumps({"shape": [N, nw, nb], "variant": v or "default", "rep": rep, "ms_per_T": round(ms, 4),
                              "frac": round(b[4] / ms / 1e6 / peak, 4)}), flush=True)
            del s
            gc.collect()


if __name__ == "__main__":
    main()
