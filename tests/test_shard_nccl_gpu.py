"""The sharded path's NCCL branch (exchange and solve collectives on the
solver's stream, shard.py) on one rank: the N > 1 bench and solve code paths,
NCCL included, run on the single GPU the tests get (several ranks cannot share
one GPU under NCCL; the multi-rank logic is covered by the gloo tests).  GPU only."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, name, native, q):
    sys.path.insert(0, ROOT)
    os.environ["SPOCK_SHARD_NCCL"] = "1" if native else "0"
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2505_12078_b200.generators import make_config
        from paper_2505_12078_b200.rng import Philox
        from paper_2505_12078_b200.shard import ShardedSolver
        from paper_2505_12078_b200.solver import SpockSolver
        p = make_config(name, seed=1)
        sh = ShardedSolver(p, split_stage=2, max_iters=30)
        assert sh.native == native
        one = SpockSolver(p, alpha=sh.alpha, max_iters=30)
        z = -1.0 + 2.0 * Philox(3).uniform_array(sh.nz)
        e = -1.0 + 2.0 * Philox(53).uniform_array(sh.neta)
        za, ea = sh.apply_T(z, e)
        zb, eb = one.apply_T(z, e)
        err_T = max(float(np.abs(za - zb).max()), float(np.abs(ea - eb).max()))
        a, b = sh.solve(p.x_init), one.solve(p.x_init)
        same = a.status["branches"] == b.status["branches"]
        err_s = float(np.abs(a.z - b.z).max() / max(1.0, np.abs(b.z).max()))
        q.put((err_T, same, err_s, a.status["iterations"]))
    except Exception as ex:  # report instead of hanging the parent
        q.put((repr(ex), False, 0.0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("native", [True, False], ids=["library-nccl", "torch-nccl"])
@pytest.mark.parametrize("name", ["c1", "c2p"])
def test_sharded_nccl_one_rank_matches_one_gpu(name, native):
    """native: the library's own NCCL communicator (spock_shard_nccl_init, every
    collective enqueued from C++); else torch.distributed's NCCL collectives
    through the host callback."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_worker, args=(_free_port(), name, native, q))
    pr.start()
    err_T, same, err_s, iters = q.get(timeout=600)
    pr.join(timeout=60)
    assert not isinstance(err_T, str), err_T
    assert err_T <= 1e-12 and same and err_s <= 1e-9 and iters == 30, (err_T, same, err_s, iters)


def test_bench_sharded_path_one_rank():
    """bench.py's N > 1 branch (sharded c2p T, NCCL all-gathers, max over ranks,
    one JSON line) under torchrun with one process."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--sharded", "--config", "c2p", "--steps", "3", "--warmup", "3", "--no-cpu", "--sweep", "",
           "--side-by-side", "none"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["scaling"] == "strong"
    assert line["sharded"]["collective"].startswith("all_gather (nccl)")
    assert "enqueued by the library" in line["sharded"]["collective"]
