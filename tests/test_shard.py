"""Subtree sharding plan and exchange on CPU: ownership and
dependency order of every rank's item lists, and the all-gather of the
stage-ts exchange records over a world-size-2/3 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_12078_b200.generators import make_config
from paper_2505_12078_b200.problem import ScenarioTree
from paper_2505_12078_b200.shard import check_plan, default_split_stage, exchange, make_plan

TREES = [
    ("binary-4", ScenarioTree.from_branching([2, 2, 2, 2])),
    ("mixed", ScenarioTree.from_branching([3, 1, 2, 5])),
    ("fan-40", ScenarioTree.from_branching([40, 1, 1])),
    ("c2", make_config("c2", seed=1).tree),
]


@pytest.mark.parametrize("name,tree", TREES, ids=[n for n, _ in TREES])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_covers_tree_once(name, tree, world):
    plans = [make_plan(tree, 3, 2, world, r) for r in range(world)]
    check_plan(tree, plans)
    ts = plans[0].split_stage
    assert 1 <= ts <= tree.horizon
    # owned stage-ts ranges tile the stage in rank order
    assert plans[0].b0 == tree.stage_begin(ts)
    for a, b in zip(plans, plans[1:]):
        assert a.b1 == b.b0
    assert plans[-1].b1 == tree.stage_end(ts)


@pytest.mark.parametrize("ts", [1, 2, 3])
def test_plan_explicit_split_stage(ts):
    tree = ScenarioTree.from_branching([2, 3, 2])
    plans = [make_plan(tree, 2, 1, 2, r, split_stage=ts) for r in range(2)]
    check_plan(tree, plans)
    assert all(p.split_stage == ts for p in plans)


def test_default_split_stage_prefers_enough_subtrees():
    tree = ScenarioTree.from_branching([2, 2, 2, 2, 2])
    assert default_split_stage(tree, 1) == 2   # 4 nodes >= 4*1
    assert default_split_stage(tree, 2) == 3   # 8 nodes >= 4*2
    assert default_split_stage(tree, 64) == 5  # widest stage when none is wide enough


def test_plan_rejects_bad_arguments():
    tree = ScenarioTree.from_branching([2, 2])
    with pytest.raises(ValueError):
        make_plan(tree, 2, 1, 2, 2)
    with pytest.raises(ValueError):
        make_plan(tree, 2, 1, 2, 0, split_stage=0)
    with pytest.raises(ValueError):
        make_plan(tree, 2, 1, 2, 0, split_stage=3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, tree_branching, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree = ScenarioTree.from_branching(tree_branching)
        pl = make_plan(tree, 2, 1, world, rank)
        E = pl.record_len
        xbuf = torch.zeros(pl.xbuf_len, dtype=torch.float64)
        # rank writes the records of its stage-ts nodes: value = node + field/100
        for c in range(pl.b0, pl.b1):
            k = c - pl.bfirst
            xbuf[k * E:(k + 1) * E] = torch.tensor([c + f / 100.0 for f in range(E)], dtype=torch.float64)
        exchange(xbuf, pl)
        ok = True
        for c in range(pl.bfirst, pl.bfirst + pl.nbound):
            k = c - pl.bfirst
            want = torch.tensor([c + f / 100.0 for f in range(E)], dtype=torch.float64)
            ok &= bool(torch.equal(xbuf[k * E:(k + 1) * E], want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,branching", [(2, [2, 3, 2]), (3, [4, 2]), (2, [5, 1, 1])])
def test_exchange_allgather_gloo(world, branching):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, branching, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
