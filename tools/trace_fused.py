"""Critical-path analysis of one traced fused T (SPOCK_FUSED_TRACE).

Runs on the GPU box: builds the config's solver, records 4 %globaltimer stamps
per item (start, dependencies acquired, flag released, end) and prints the
per-stage timeline of the backward and forward sweeps."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg="c2"):
    from paper_2505_12078_b200.generators import make_config
    from paper_2505_12078_b200.solver import SpockSolver
    p = make_config(cfg, seed=1)
    path = os.path.join(tempfile.gettempdir(), "fused_trace.bin")
    os.environ["SPOCK_FUSED_TRACE"] = path
    s = SpockSolver(p)
    s.bench_T(2, use_graph=False, flush_l2=True)
    tr = p.tree
    nn, nnl = tr.num_nodes(), tr.num_nonleaf()
    raw = np.fromfile(path, dtype=np.uint64).reshape(-1, 8).astype(np.float64)
    cyc = raw[:, 4:8]
    st = raw[:, :4]
    t0 = st[st > 0].min()
    st = np.where(st > 0, (st - t0) / 1000.0, np.nan)  # us
    print(f"{cfg}: nodes {nn}, items {len(st)}, T span {np.nanmax(st):.1f} us")
    s2 = st[nn:nn + nnl]
    print(f"S2 items: start {np.nanmin(s2[:,0]):.1f}..{np.nanmax(s2[:,0]):.1f} end max {np.nanmax(s2[:,3]):.1f}")
    c = cyc[:nn]
    ok = (c[:, 0] > 0) & (c[:, 1] > 0) & (c[:, 2] > 0) & (c[:, 3] > 0)
    c = c[ok]
    ph = np.array([c[:, 1] - c[:, 0], c[:, 2] - c[:, 1], c[:, 3] - c[:, 2]])
    print("backward non-leaf phases (cycles, median): children loads %.0f  GEMV round %.0f  stores %.0f"
          % tuple(np.median(ph, axis=1)))
    for name, base, order in (("backward", 0, lambda k: nn - 1 - k), ("forward", nn + nnl, lambda k: k)):
        print(f"-- {name}: stage  nodes  start(min/max)  deps-ok(min/max)  released(min/max)  end(max)")
        for t in (range(tr.horizon, -1, -1) if name == "backward" else range(tr.horizon + 1)):
            nodes = range(tr.stage_begin(t), tr.stage_end(t))
            rows = np.array([st[base + (nn - 1 - i if name == "backward" else i)] for i in nodes])
            print(f"   {t:3d} {len(nodes):6d}  {np.nanmin(rows[:,0]):7.1f}/{np.nanmax(rows[:,0]):7.1f}"
                  f"  {np.nanmin(rows[:,1]):7.1f}/{np.nanmax(rows[:,1]):7.1f}"
                  f"  {np.nanmin(rows[:,2]):7.1f}/{np.nanmax(rows[:,2]):7.1f}  {np.nanmax(rows[:,3]):7.1f}")


if __name__ == "__main__":
    main(*(sys.argv[1:] or ["c2"]))
