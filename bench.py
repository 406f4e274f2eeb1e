"""Benchmark of the B200 SPOCK hot path (driver contract: one JSON line on rank 0).

A *step* is one Chambolle-Pock application T (proj/src/solver.cpp:148-164) over
the whole scenario tree, the unit behind BASELINE.json's "CP iterations/s".
The headline workload is c4 -- BASELINE configs[3]'s ~1e5-node tree (N 12,
branching 10 to stage 4, 91 111 nodes, nx 50, nu 25), the largest
single-GPU config and the one the north star's >= 50 % roofline target is
quoted on -- from the reference's case-study-1 generator with an independent
per-node perturbation, so every node streams its own matrices.

  value : device-timed CP iterations/s, iterates resident in HBM, L2 flushed
          between steps (and the 14 GB of matrices exceed L2 anyway).
  e2e   : the same metric through the public C-ABI with host buffers: every
          step is one spock_solver_apply_T call on pinned host (z, eta), the
          host->device copy of the step's input, T, and the device->host copy of
          its result inside the timed region.
  roofline : the T kernel against MEASURED_PEAKS.json hbm_gbs; `achieved` uses
          SURVEY §8(d)'s algorithmic bytes; frac_lean uses the engine's leaner
          byte model (P never re-read, diagonal constraint maps) and frac_dram
          the ncu-measured DRAM bytes (profiles/ncu_traffic.json).
  cpu_baseline : the CPU oracle (restatement of the reference, same ThreadPool
          semantics) on the same instance, every host thread and one thread.
  sweep : c3, c2p, c2, each with its own cpu_baseline.
  solve_side_by_side : c1 time to tol (SuperMann and CP) and fixed-budget
          SuperMann on c2 / c3 / c4, GPU beside the CPU oracle.

--impl reference times the oracle's CPU T on the same config (the reference
itself cannot be built here: Eigen3 is absent).  N > 1 (torchrun): the headline
is strong scaling of one c4 tree split by subtrees below a split stage over all
ranks, one NCCL all-gather of the stage-ts records per T.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        time.sleep(0.1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx.append(float(f[1]))
                except ValueError:
                    continue
                for n, v in zip(names, f[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            os.unlink(self.path)
        except Exception:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _problem(config: str, seed: int):
    from paper_2505_12078_b200.generators import make_config
    return make_config(config, seed=seed)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def survey_bytes(p) -> dict:
    """Algorithmic bytes of one CP application T by SURVEY.md §8(d)'s model
    (each per-node operand once per phase that uses it, P re-read in the S1
    sweeps, dense constraint maps, the two z re-reads): c2 46 797 736 B,
    c2p 216 943 784 B, c4 (12, 10, 4) 19 145 623 720 B.  Plus its flop count F_T."""
    tr = p.tree
    nn, nnl, nl = tr.num_nodes(), tr.num_nonleaf(), tr.num_leaves()
    nr, nx, nu = nn - 1, p.nx, p.nu
    pp, pN = nx + nu, nx
    nch = tr.child_count[:nnl].astype(np.int64)
    gam = np.array([r.gamma for r in p.risk])
    ny = np.where(gam > 0, 2 * nch + 1, nch + 1)
    ny = np.where(np.array([len(r.cone) == 1 for r in p.risk]), nch, ny)
    nz = 1 + nn * nx + nnl * nu + int(ny.sum()) + 2 * nr
    ne = int((ny + 1 + (nx + nu)).sum()) + nr * (pp + 2) + nl * (nx + pN + 2)
    ML = nr * (pp * (nx + nu) + (nx + nu)) + int(ny.sum()) + nl * (pN * nx + nx)
    BL = 8 * (ML + nz + ne)
    BS1b = 8 * (nr * (nx * nu + 2 * nx * nx + nx) + nnl * (nu * nu + nu * nx) + 2 * (nn * nx + nnl * nu))
    BS1f = 8 * (nr * (nx * nx + nx * nu + nx) + nnl * (nu * nx + nu) + nn * nx + nnl * nu)
    BS2 = 16 * int((ny + 2 * nch).sum())
    BS3 = 8 * (nr * (pp + 2) + nnl * 2 * (nx + nu) + nl * (2 * nx + pN + 2) + 2 * ne)
    F = 2 * (2 * nr * pp * (nx + nu) + 2 * nl * nx * nx) + nr * (8 * nx * nx + 6 * nx * nu) + nnl * (2 * nu * nu + 4 * nu * nx)
    return {"B_T": int(2 * BL + BS1b + BS1f + BS2 + BS3 + 16 * nz), "F_T": int(F), "B_L": int(BL),
            "B_S1": int(BS1b + BS1f), "B_S2": int(BS2), "B_S3": int(BS3)}


def _workload(config: str, p) -> dict:
    tr = p.tree
    from paper_2505_12078_b200.generators import CONFIGS
    c = CONFIGS.get(config, {})
    nw = p.meta.get("dims").nw if p.meta.get("dims") is not None else c.get("nw")
    nb = p.meta.get("dims").nb if p.meta.get("dims") is not None else c.get("nb")
    return {"workload": f"{config}: random RAOCP nx={p.nx} nu={p.nu} N={tr.horizon} nw={nw} nb={nb} "
                        f"({tr.num_nodes()} nodes, {tr.num_leaves()} scenarios), AV@R, boxes, preconditioning on",
            "nodes": tr.num_nodes(), "nx": p.nx, "nu": p.nu, "horizon": tr.horizon,
            "per_node_perturbation": p.meta.get("perturb"), "step": "one CP application T over the whole tree",
            "l2": "flushed between timed steps (256 MiB rewrite outside the step events); the c3/c4 matrices "
                  "(5-14 GB) exceed the 126 MB L2 in any case"}


def _oracle(p, alpha=None):
    """The CPU oracle on p; with alpha given (the GPU solver's), its power
    iteration is skipped (ORACLE_SKIP_NORM: alpha is all T reads)."""
    from oracle import oracle
    if alpha is None:
        return oracle.OracleSolver(p)
    os.environ["ORACLE_SKIP_NORM"] = "1"
    try:
        return oracle.OracleSolver(p, alpha=alpha)
    finally:
        os.environ.pop("ORACLE_SKIP_NORM", None)


def cpu_baseline(o, budget_s: float = 12.0, one_thread_s: float = 6.0) -> dict:
    """The CPU oracle (restated reference, same ThreadPool semantics) on the same
    instance: a bounded sample with every host thread, then one with 1 thread."""
    from oracle import oracle
    L = oracle.lib()
    nt = L.oracle_num_threads()
    t1 = o.bench_T(1)  # ms per T (also warms the caches)
    k = int(max(2, min(500, budget_s * 1000.0 / max(t1, 1e-3))))
    ms = o.bench_T(k)
    oracle.set_num_threads(1)
    try:
        s1 = o.bench_T(1)
        k1 = int(max(1, min(200, one_thread_s * 1000.0 / max(s1, 1e-3))))
        ms1 = o.bench_T(k1) if k1 > 1 else s1
    finally:
        oracle.set_num_threads(nt)
    return {"value": k / (ms / 1000.0), "unit": "iter/s", "cores": nt, "kind": "port", "cpu_model": _cpu_model(),
            "sample": f"{k} CP applications T on the same instance ({ms / 1000.0:.1f} s, {nt} threads)",
            "one_thread": {"value": k1 / (ms1 / 1000.0), "unit": "iter/s", "sample": f"{k1} T, 1 thread"}}


def run_reference(args) -> None:
    """--impl reference: the reference's CPU implementation of the path (the
    oracle restatement; the reference itself needs Eigen3, absent here) on the
    same config, metric and unit, with every host thread.  Each step is one T
    over the whole tree; the timed steps are capped so the run stays within a
    few minutes (c4: ~0.5-1 s per T on 16 threads)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle
    p = _problem(args.config, args.seed)
    o = _oracle(p)
    per = o.bench_T(1)
    steps = args.steps
    timed = int(max(3, min(steps, 60000.0 / max(per, 1e-3))))
    o.bench_T(max(1, min(args.warmup, int(15000.0 / max(per, 1e-3)))))
    ms = o.bench_T(timed)
    val = timed / (ms / 1000.0)
    nt = oracle.lib().oracle_num_threads()
    line = {
        "impl": "reference", "metric": "CP iterations/s", "value": val, "unit": "iter/s", "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms / timed, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference case-study-1 generator, per-node perturbed)",
        "config": _workload(args.config, p),
        "cpu_baseline": {"value": val, "unit": "iter/s", "cores": nt, "kind": "port", "cpu_model": _cpu_model(),
                         "sample": f"{timed} of {steps} steps timed: CP applications T by the CPU restatement of the "
                                   f"reference (the reference needs Eigen3, absent here), {nt} threads"},
        "e2e": {"value": val, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def sweep_point(config: str, seed: int, steps: int, peak: float, cpu: bool) -> dict:
    from paper_2505_12078_b200.solver import SpockSolver
    p = _problem(config, seed)
    t0 = time.time()
    s = SpockSolver(p)
    setup = time.time() - t0
    s.bench_T(4, flush_l2=True)
    ms = s.bench_T(steps, flush_l2=True)
    bytes5, launches = s.traffic_model()
    sb = survey_bytes(p)
    tpt = ms / steps
    row = {"config": config, "nodes": p.tree.num_nodes(), "schedule": s.t_path,
           "kernel": {"fused": "k_T_fused", "wide": "k_T_wide", "stages": "per-stage kernels"}[s.t_path],
           "launches_per_T": launches, "iter_per_s": steps / (ms / 1000.0), "ms_per_T": tpt,
           "B_T_survey": sb["B_T"], "frac_survey": sb["B_T"] / (tpt / 1000.0) / 1e9 / peak,
           "B_T_lean": bytes5[4], "frac_lean": bytes5[4] / (tpt / 1000.0) / 1e9 / peak, "setup_s": setup}
    if cpu:
        row["cpu_baseline"] = cpu_baseline(_oracle(p, s.alpha), budget_s=4.0, one_thread_s=3.0)
        row["speedup_vs_cpu"] = row["iter_per_s"] / row["cpu_baseline"]["value"]
    return row


def seed_block(config: str, peak: float, cpu: bool, seeds=(1, 2, 3, 4, 5)) -> dict:
    """BASELINE.md §4 inputs are Philox seeds 1-5: the headline T on every
    seed (device ms, L2 flushed; lean-byte roofline), and c1's CP solve to
    1e-4 on every seed beside the CPU oracle (same iterations expected)."""
    from paper_2505_12078_b200.solver import SpockSolver
    out = {"config": config, "T": [], "c1_cp_1e-4": []}
    for sd in seeds:
        r = sweep_point(config, sd, 20, peak, False)
        out["T"].append({"seed": sd, "ms_per_T": r["ms_per_T"], "frac_lean": r["frac_lean"],
                         "frac_survey": r["frac_survey"]})
    if cpu:
        from oracle import oracle
        for sd in seeds:
            p = _problem("c1", sd)
            kw = dict(eps_abs=1e-4, eps_rel=1e-4, max_iters=50000)
            g = SpockSolver(p, **kw)
            g.solve_cp(p.x_init)
            a, gms = _timed(g.solve_cp, p.x_init)
            o = oracle.OracleSolver(p, alpha=g.alpha, **kw)
            b, cms = _timed(o.solve_cp, p.x_init)
            out["c1_cp_1e-4"].append({
                "seed": sd, "gpu_ms": gms, "cpu_ms": cms, "gpu_iterations": a.status["iterations"],
                "cpu_iterations": b.status["iterations"], "loop": g.loop_path,
                "solution_rel_diff": float(np.abs(a.z - b.z).max() / max(1.0, np.abs(b.z).max()))})
    ts = [x["ms_per_T"] for x in out["T"]]
    out["T_ms_min_median_max"] = [min(ts), sorted(ts)[len(ts) // 2], max(ts)]
    return out


def _prefix(a: str, b: str) -> int:
    n = min(len(a), len(b))
    for k in range(n):
        if a[k] != b[k]:
            return k
    return n


def _timed(fn, *a):
    t = time.perf_counter()
    r = fn(*a)
    return r, 1000.0 * (time.perf_counter() - t)


def solve_side_by_side(full: bool = False) -> dict:
    """Solve-level comparison with the CPU oracle (SuperMann
    solver.cpp:189-350, CP 182-187).  c1: time to tol 1e-3 / 1e-4 / 1e-6 for
    SuperMann and CP, the GPU (device-resident loop, public API) beside the
    oracle on every host thread and on one.  c2, c3, c4: fixed-budget SuperMann
    (tol 1e-3 is not reached by the reference algorithm on c2 within 20 000
    iterations), 500 iterations on the GPU and the same on the CPU for c2; the
    CPU runs a bounded prefix on c3 / c4 (--side-by-side full: 500 there too).
    Reported: ms per SuperMann iteration, T / L / L* counts, K0 / K1 / K2, the
    matching prefix of the branch strings and the ||r||_M agreement on it."""
    from oracle import oracle
    from paper_2505_12078_b200.solver import SpockSolver
    nt = oracle.lib().oracle_num_threads()
    out = {"cores": nt, "cpu_model": _cpu_model(), "c1_time_to_tol": [], "fixed_budget": []}
    p = _problem("c1", 1)
    for method in ("solve", "solve_cp"):
        for tol in (1e-3, 1e-4, 1e-6):
            kw = dict(eps_abs=tol, eps_rel=tol, max_iters=50000)
            g = SpockSolver(p, **kw)
            getattr(g, method)(p.x_init)  # graph build
            a, gms = _timed(getattr(g, method), p.x_init)
            o = oracle.OracleSolver(p, alpha=g.alpha, **kw)
            b, cms = _timed(getattr(o, method), p.x_init)
            oracle.set_num_threads(1)
            try:
                b1, c1ms = _timed(getattr(o, method), p.x_init)
            finally:
                oracle.set_num_threads(nt)
            out["c1_time_to_tol"].append({
                "method": "SuperMann" if method == "solve" else "CP", "tol": tol,
                "gpu": {"ms": gms, "reason": a.status["reason"], "iterations": a.status["iterations"],
                        "n_T": a.status["n_T"]},
                "cpu": {"ms": cms, "reason": b.status["reason"], "iterations": b.status["iterations"], "threads": nt},
                "cpu_1thread": {"ms": c1ms, "iterations": b1.status["iterations"]},
                "speedup_vs_cpu": cms / gms, "speedup_vs_cpu_1thread": c1ms / gms,
                "branch_prefix": _prefix(a.status["branches"], b.status["branches"]),
                "solution_rel_diff": float(np.abs(a.z - b.z).max() / max(1.0, np.abs(b.z).max()))})
    for cfg, gi, ci in (("c2", 500, 500), ("c3", 500, 500 if full else 12), ("c4", 500, 500 if full else 6)):
        try:
            p = _problem(cfg, 1)
            g = SpockSolver(p, max_iters=gi, eps_abs=1e-14, eps_rel=1e-14)
            g.solve(p.x_init)
            a, gms = _timed(g.solve, p.x_init)
            o = oracle.OracleSolver(p, alpha=g.alpha, max_iters=ci, eps_abs=1e-14, eps_rel=1e-14)
            b, cms = _timed(o.solve, p.x_init)
            d = _prefix(a.status["branches"], b.status["branches"])
            ra, rb = a.status["rnorm_history"][:d], b.status["rnorm_history"][:d]
            rel = float(np.max(np.abs(ra - rb) / np.maximum(np.abs(rb), 1e-300))) if d else None
            st = lambda r: {"iterations": r.status["iterations"], "n_T": r.status["n_T"], "n_L": r.status["n_L"],
                            "n_Lt": r.status["n_Lt"], "K0_K1_K2_KM": [r.status["k0_steps"], r.status["k1_steps"],
                                                                    r.status["k2_steps"], r.status["stalled_steps"]],
                            "rnorm_last": float(r.status["rnorm_history"][-1]) if len(r.status["rnorm_history"]) else None}
            out["fixed_budget"].append({
                "config": cfg, "nodes": p.tree.num_nodes(), "label": "fixed budget (tol 1e-14, not reached)",
                "gpu": dict(st(a), ms=gms, ms_per_iter=gms / max(1, a.status["iterations"])),
                "cpu": dict(st(b), ms=cms, ms_per_iter=cms / max(1, b.status["iterations"]), threads=nt),
                "speedup_per_iter": (cms / max(1, b.status["iterations"])) / (gms / max(1, a.status["iterations"])),
                "branch_prefix": d, "branch_compared": min(len(a.status["branches"]), len(b.status["branches"])),
                "rnorm_rel_diff_on_prefix": rel,
                "rnorm_trace_gpu_head": [float(x) for x in a.status["rnorm_history"][:8]],
                "rnorm_trace_cpu_head": [float(x) for x in b.status["rnorm_history"][:8]]})
            del g, o
        except Exception as ex:  # keep the rest of the block
            out["fixed_budget"].append({"config": cfg, "error": str(ex)[:200]})
    return out


def sharded_run(args, dist, peak: float, local: int) -> dict:
    """N > 1: strong scaling of one c4 T over the subtree-sharded tree (SURVEY
    §8e; north star decomposition): every rank holds the instance, owns its
    stage-ts subtrees, all-gathers the stage-ts exchange records once per T
    (NCCL on the solver's stream).  Device time on the solver's stream, max over
    ranks; e2e through ShardedSolver.apply_T with host buffers."""
    import torch
    from paper_2505_12078_b200.shard import ShardedSolver
    # the ranks share one host: generate the instance one rank at a time (the
    # generator's temporaries are several times the problem's ~5 GB on c4)
    p = None
    for r in range(dist.get_world_size()):
        if r == dist.get_rank():
            p = _problem(args.config, args.seed)
        dist.barrier()
    t0 = time.time()
    sh = ShardedSolver(p)
    setup_s = time.time() - t0
    for k in range(args.warmup):
        sh.bench_step(k & 1)
    st = sh.stream
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    dist.barrier()
    with ClockSampler(local) as clk:
        a.record(st)
        for k in range(args.steps):
            sh.bench_step(k & 1)
        b.record(st)
        b.synchronize()
        dist.barrier()
        # e2e: apply_T through the public API with host buffers (copies inside)
        z = np.ascontiguousarray(_rand_vec(sh.nz, 41))
        e = np.ascontiguousarray(_rand_vec(sh.neta, 42))
        n_e2e = max(3, min(args.steps, 20))
        sh.apply_T(z, e)
        dist.barrier()
        t1 = time.perf_counter()
        for _ in range(n_e2e):
            sh.apply_T(z, e)
        e2e_s = time.perf_counter() - t1
    ms = torch.tensor([a.elapsed_time(b) / args.steps, e2e_s], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_T, e2e_s = float(ms[0].item()), float(ms[1].item())
    sb = survey_bytes(p)
    bytes5, _ = sh.solver.traffic_model()
    pl = sh.plan
    return {"ms_per_T": ms_T, "e2e_s": e2e_s, "n_e2e": n_e2e, "setup_s": setup_s, "clocks": clk.summary(),
            "sb": sb, "lean": bytes5[4], "nz": sh.nz, "neta": sh.neta, "p": p,
            "plan": {"ranks": pl.world, "split_stage": pl.split_stage, "stage_nodes_per_rank": pl.q,
                     "exchange_bytes": pl.xbuf_len * 8,
                     "collective": f"all_gather ({dist.get_backend()}) of stage-ts records, once per T"
                                   + (", ncclAllGather enqueued by the library on the solver stream" if sh.native else "")}}


def _rand_vec(n, seed):
    from paper_2505_12078_b200.rng import Philox
    return -1.0 + 2.0 * Philox(seed).uniform_array(n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", help="headline workload (c4: BASELINE configs[3], ~1e5 nodes, "
                                                     "the largest single-GPU config)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sweep", default="c3,c2p,c2", help="extra single-GPU configs (N=1 only); '' disables")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--side-by-side", default="quick", choices=["quick", "full", "none"])
    ap.add_argument("--seeds", type=int, default=1, help="1: the seeds 1-5 block (headline T per seed, c1 CP "
                    "to 1e-4 per seed beside the oracle); 0: skip")
    ap.add_argument("--sharded", action="store_true", help="run the subtree-sharded path even on one rank "
                    "(exercises the N > 1 code path, NCCL included, on a single GPU)")
    ap.add_argument("--backend", default="nccl", help="process group backend for N>1 (gloo: code-path smoke test "
                                                          "with several ranks on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    ws, rank, local = _dist()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    peak, peak_kind = _peaks()
    if ws > 1 or args.sharded:
        import torch.distributed as dist
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + (os.getpid() % 1000)))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)
        R = sharded_run(args, dist, peak, local)
        if rank == 0:
            p, sb = R["p"], R["sb"]
            ms = R["ms_per_T"]
            ach = sb["B_T"] / (ms / 1000.0) / 1e9
            line = {
                "metric": "CP iterations/s", "value": 1000.0 / ms, "unit": "iter/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference case-study-1 generator, per-node perturbed)",
                "config": dict(_workload(args.config, p), parallelism=f"subtree-sharded over {ws} ranks"),
                "e2e": {"value": R["n_e2e"] / R["e2e_s"], "unit": "iter/s",
                        "h2d_bytes_per_step": int(8 * (R["nz"] + R["neta"]) * ws),
                        "d2h_bytes_per_step": int(8 * (R["nz"] + R["neta"]) * ws),
                        "call": "ShardedSolver.apply_T (spock_shard_apply_T, phase A, all-gather, phase B) on host "
                                "numpy buffers; bytes summed over ranks"},
                "roofline": {"bound": "hbm", "kernel": "k_T_wide (phases A + B per rank)", "achieved": ach,
                             "peak": peak * ws, "unit": "GB/s", "frac": ach / (peak * ws), "traffic": None,
                             "peak_kind": f"{peak_kind} x {ws} GPUs", "algorithmic_bytes": sb["B_T"],
                             "bytes_model": "SURVEY.md §8(d)", "frac_lean": R["lean"] / (ms / 1000.0) / 1e9 / (peak * ws)},
                "cpu_baseline": None, "gpu_launches": int(4 * args.steps * ws), "clocks": R["clocks"],
                "sharded": R["plan"], "setup_s": R["setup_s"],
            }
            print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return

    from paper_2505_12078_b200.solver import SpockSolver
    p = _problem(args.config, args.seed)
    t0 = time.time()
    s = SpockSolver(p)
    setup_s = time.time() - t0
    s.bench_T(args.warmup, flush_l2=True)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ms = s.bench_T(args.steps, flush_l2=True)
        torch.cuda.synchronize()
        # e2e: apply_T through the C-ABI with pinned host buffers, copies inside
        zh = torch.from_numpy(_rand_vec(s.nz, 41)).pin_memory()
        eh = torch.from_numpy(_rand_vec(s.neta, 42)).pin_memory()
        zo = torch.zeros(s.nz, dtype=torch.float64).pin_memory()
        eo = torch.zeros(s.neta, dtype=torch.float64).pin_memory()
        for _ in range(args.warmup):
            s.apply_T(zh, eh, zo, eo)
        n_e2e = max(10, min(args.steps, 100))
        t1 = time.perf_counter()
        for k in range(n_e2e):
            if k & 1:
                s.apply_T(zo, eo, zh, eh)
            else:
                s.apply_T(zh, eh, zo, eo)
        apply_s = time.perf_counter() - t1
    value = args.steps / (ms / 1000.0)
    kms = s.bench_kernels(10, flush_l2=True)
    bytes5, launches = s.traffic_model()
    sb = survey_bytes(p)
    fused = launches == 1
    names = ["L* (standalone adjoint)", "S1 sweeps (per-stage path)", "S2", "L (standalone)", "T"]
    kname = {"fused": "k_T_fused", "wide": "k_T_wide", "stages": "per-stage kernels"}[s.t_path]
    t_T = kms[4]  # average device ms of one T launch (one kernel on the fused / wide paths)
    ach = sb["B_T"] / (t_T / 1000.0) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.config, {}).get("T")
        except Exception:
            traffic = None
    o = None
    cpu = None
    if not args.no_cpu:
        o = _oracle(p, s.alpha)
        cpu = cpu_baseline(o)
        del o
    sweep = []
    if args.sweep:
        for c in [x for x in args.sweep.split(",") if x]:
            try:
                sweep.append(sweep_point(c, args.seed, max(20, min(args.steps, 100)), peak, not args.no_cpu))
            except Exception as ex:  # keep the headline line even if a sweep point fails
                sweep.append({"config": c, "error": str(ex)[:200]})
    seeds = None
    if args.seeds:
        try:
            seeds = seed_block(args.config, peak, not args.no_cpu)
        except Exception as ex:
            seeds = {"error": str(ex)[:300]}
    side = None
    if args.side_by_side != "none" and not args.no_cpu:
        try:
            side = solve_side_by_side(full=args.side_by_side == "full")
        except Exception as ex:
            side = {"error": str(ex)[:300]}
    line = {
        "metric": "CP iterations/s", "value": value, "unit": "iter/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference case-study-1 generator, per-node perturbed)",
        "config": _workload(args.config, p),
        "e2e": {"value": n_e2e / apply_s, "unit": "iter/s", "h2d_bytes_per_step": int(8 * (s.nz + s.neta)),
                "d2h_bytes_per_step": int(8 * (s.nz + s.neta)), "call": "spock_solver_apply_T, pinned host buffers",
                "steps": n_e2e},
        "roofline": {"bound": "hbm", "kernel": f"{kname} (one launch per CP application)" if launches == 1 else kname,
                     "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "peak_kind": peak_kind, "algorithmic_bytes": sb["B_T"], "bytes_model": "SURVEY.md §8(d)",
                     "avg_launch_ms": t_T, "flops": sb["F_T"],
                     "frac_lean": bytes5[4] / (t_T / 1000.0) / 1e9 / peak, "lean_bytes": bytes5[4],
                     "frac_dram": (traffic / (t_T / 1000.0) / 1e9 / peak) if traffic else None},
        "kernels_ms": dict(zip(names, [float(x) for x in kms])),
        "cpu_baseline": cpu,
        "gpu_launches": int(launches * args.steps),
        "clocks": clk.summary(),
        "setup_s": setup_s,
        "sweep": sweep,
        "solve_side_by_side": side,
        "seeds": seeds,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
