"""Subtree sharding of the CP operator T over G ranks.

The reference runs one process (proj/src/parallel.cpp is a thread pool over
the nodes of one stage); this is the B200 extension the north star names:
the tree is cut at a split stage ``ts``, rank ``r`` owns the stage-ts nodes
``[b0, b1) = [bfirst + r*q, bfirst + (r+1)*q)`` (``q = ceil(|stage ts| / G)``)
together with their subtrees, and every rank computes the stages ``< ts``
("the top") redundantly.  Because the tree is numbered breadth first with
contiguous children (proj/include/spock/tree.hpp:10-13,42-44), every owned
subtree is one contiguous node range per stage.

One T needs one exchange: after a rank's subtrees ran their backward items,
each stage-ts node contributes the terms its parent sums over its children
(the L* stage-cost adjoint adj_c and the S1 sweep term T12_c,
tree_operator.cpp:106-113 and projections.cpp:157-158,171) and the z / eta
entries S2 of its parent reads (projections.cpp:189-210); an all-gather of
those records lets every rank finish the top and then its subtrees' forward
items.  The stage-ts parent sums run in ascending child order, so the result
is deterministic for a fixed G (and equal to one GPU up to rounding).

``ShardPlan`` is pure host logic (no device needed, tested on CPU);
``ShardedSolver`` drives the device library over ``torch.distributed`` (NCCL
on a B200 box, gloo in the CPU tests and for several ranks sharing one GPU).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .problem import ScenarioTree


def default_split_stage(tree: ScenarioTree, world: int) -> int:
    """Smallest stage t >= 1 with at least 4 nodes per rank (else the widest
    stage), so each rank gets several subtrees and the replicated top stays
    small."""
    N = tree.horizon
    best, best_n = 1, -1
    for t in range(1, N + 1):
        n = tree.stage_end(t) - tree.stage_begin(t)
        if n >= 4 * world:
            return t
        if n > best_n:
            best, best_n = t, n
    return best


@dataclass
class ShardPlan:
    world: int
    rank: int
    split_stage: int
    bfirst: int
    nbound: int
    q: int
    b0: int
    b1: int
    owned: np.ndarray       # bool per node: top or in this rank's subtrees
    back_a: np.ndarray      # own subtrees' backward items, descending
    back_b: np.ndarray      # the top's backward items, descending
    s2: np.ndarray          # parents whose S2 this rank computes
    fwd: np.ndarray         # forward items, ascending
    record_len: int         # doubles per exchange record (2(nx+nu)+6)

    @property
    def xbuf_len(self) -> int:
        return self.world * self.q * self.record_len

    @property
    def slice(self) -> slice:
        """This rank's slice of the exchange buffer."""
        return slice(self.rank * self.q * self.record_len, (self.rank + 1) * self.q * self.record_len)


def make_plan(tree: ScenarioTree, nx: int, nu: int, world: int, rank: int,
              split_stage: Optional[int] = None) -> ShardPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard plan: bad rank / world size")
    ts = default_split_stage(tree, world) if split_stage is None else int(split_stage)
    if not 1 <= ts <= tree.horizon:
        raise ValueError("shard plan: split stage must be in [1, N]")
    nn, nnl = tree.num_nodes(), tree.num_nonleaf()
    bfirst = tree.stage_begin(ts)
    nbound = tree.stage_end(ts) - bfirst
    q = -(-nbound // world)
    b0 = bfirst + min(rank * q, nbound)
    b1 = bfirst + min((rank + 1) * q, nbound)
    root_ts = np.full(nn, -1, dtype=np.int64)
    owned = np.zeros(nn, dtype=bool)
    owned[:bfirst] = True
    for i in range(bfirst, nn):
        root_ts[i] = i if tree.stage[i] == ts else root_ts[tree.anc[i]]
    owned[bfirst:] = (root_ts[bfirst:] >= b0) & (root_ts[bfirst:] < b1)
    nodes = np.arange(nn, dtype=np.int32)
    bottom = nodes[(nodes >= bfirst) & owned]
    return ShardPlan(
        world=world, rank=rank, split_stage=ts, bfirst=bfirst, nbound=nbound, q=q, b0=b0, b1=b1, owned=owned,
        back_a=bottom[::-1].copy(), back_b=nodes[:bfirst][::-1].copy(),
        s2=nodes[:nnl][owned[:nnl]].copy(), fwd=nodes[owned].copy(), record_len=2 * (nx + nu) + 6)


def check_plan(tree: ScenarioTree, plans) -> None:
    """Invariants of a set of per-rank plans (used by the CPU tests): every
    node below the split stage is owned by exactly one rank, the top by all,
    and each rank's item lists respect the dependencies (children before
    parents backward, parents before children forward)."""
    nn = tree.num_nodes()
    cnt = np.zeros(nn, dtype=np.int64)
    for pl in plans:
        cnt += pl.owned
        pos = {}
        for k, i in enumerate(list(pl.back_a) + list(pl.back_b)):
            pos[int(i)] = k
        for i, k in pos.items():
            for c in range(tree.child_first[i], tree.child_first[i] + tree.child_count[i]):
                if pl.owned[c]:
                    assert pos[c] < k, (i, c)
        fpos = {int(i): k for k, i in enumerate(pl.fwd)}
        for c, k in fpos.items():
            if c > 0:
                assert fpos[int(tree.anc[c])] < k
    top = tree.stage_begin(plans[0].split_stage)
    assert np.all(cnt[:top] == len(plans))
    assert np.all(cnt[top:] == 1)


class _DevArray:
    """__cuda_array_interface__ view of n float64 at a device address."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def exchange(xbuf, plan: ShardPlan, group=None, stream=None) -> None:
    """All-gather every rank's slice of the exchange buffer (in place).  NCCL:
    device to device, ordered on ``stream`` (the solver's); gloo: through host
    memory (CPU tests, several ranks sharing one GPU)."""
    import torch
    import torch.distributed as dist
    own = xbuf[plan.slice]
    if dist.get_backend(group) == "nccl":
        with torch.cuda.stream(stream):
            dist.all_gather_into_tensor(xbuf, own.clone(), group=group)
        return
    if stream is not None:
        stream.synchronize()
    host = own.cpu()
    parts = [torch.empty_like(host) for _ in range(plan.world)]
    dist.all_gather(parts, host, group=group)
    xbuf.copy_(torch.cat(parts).to(xbuf.device))
    if xbuf.is_cuda:
        torch.cuda.synchronize(xbuf.device)


class ShardedSolver:
    """apply_T across the ranks of a torch.distributed group: each rank holds
    the whole problem (memory replicated), computes the top and its subtrees,
    and all-gathers the stage-ts exchange records once per T."""

    def __init__(self, problem, group=None, split_stage: Optional[int] = None, **params):
        import torch
        import torch.distributed as dist
        from . import capi
        from .solver import SpockSolver, _raise
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.solver = SpockSolver(problem, **params)
        self.lib = self.solver.lib
        self.plan = make_plan(problem.tree, problem.nx, problem.nu, self.world, self.rank, split_stage)
        pl = self.plan
        self.xbuf = torch.zeros(pl.xbuf_len, dtype=torch.float64, device="cuda")
        self._keep = [np.ascontiguousarray(a, dtype=np.int32) for a in (pl.back_a, pl.back_b, pl.s2, pl.fwd)]
        a, b, s2, f = self._keep
        P = C.POINTER(C.c_int32)
        _raise(self.lib, self.lib.spock_shard_setup(
            self.solver.h, self.world, self.rank, pl.split_stage, a.ctypes.data_as(P), a.size,
            b.ctypes.data_as(P), b.size, s2.ctypes.data_as(P), s2.size, f.ctypes.data_as(P), f.size,
            C.c_void_p(self.xbuf.data_ptr())))
        self.stream = torch.cuda.ExternalStream(self.lib.spock_solver_stream(self.solver.h))
        self._capi = capi
        self._raise = _raise
        # NCCL groups: the library runs the collectives itself (spock_shard_nccl_init:
        # ncclAllGather / ncclAllReduce on the solver stream, no Python per
        # exchange or reduction); SPOCK_SHARD_NCCL=0 keeps the torch.distributed path
        import os
        self.native = dist.get_backend(group) == "nccl" and os.environ.get("SPOCK_SHARD_NCCL", "1") != "0"
        if self.native:
            uid = (C.c_char * 128)()
            if self.rank == 0:
                _raise(self.lib, self.lib.spock_nccl_unique_id(C.cast(uid, C.c_void_p)))
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = (C.c_char * 128).from_buffer_copy(box[0])
            _raise(self.lib, self.lib.spock_shard_nccl_init(self.solver.h, C.cast(uid, C.c_void_p), self.world,
                                                             self.rank))

    @property
    def alpha(self) -> float:
        return self.solver.alpha

    @property
    def nz(self) -> int:
        return self.solver.nz

    @property
    def neta(self) -> int:
        return self.solver.neta

    def masks(self):
        zm = np.zeros(self.nz, dtype=np.uint8)
        em = np.zeros(self.neta, dtype=np.uint8)
        P = C.POINTER(C.c_uint8)
        self._raise(self.lib, self.lib.spock_shard_masks(self.solver.h, zm.ctypes.data_as(P), em.ctypes.data_as(P)))
        return zm.astype(bool), em.astype(bool)

    def _exchange(self):
        exchange(self.xbuf, self.plan, self.group, self.stream)

    def apply_T(self, z, eta, z_out=None, eta_out=None):
        """Sharded SpockSolver::apply_T (proj/src/solver.cpp:148-164): entries
        outside masks() are not computed on this rank."""
        from .solver import _ptr
        z = np.ascontiguousarray(z, dtype=np.float64)
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        z_out = np.zeros_like(z) if z_out is None else z_out
        eta_out = np.zeros_like(eta) if eta_out is None else eta_out
        nz, ne = self.nz, self.neta
        if self.native:  # phase 0, the NCCL all-gather and phase 1 in one call
            self._raise(self.lib, self.lib.spock_shard_apply_T(
                self.solver.h, 2, _ptr(z, nz, "apply_T: z"), _ptr(eta, ne, "apply_T: eta"),
                _ptr(z_out, nz, "apply_T: z_out"), _ptr(eta_out, ne, "apply_T: eta_out")))
            return z_out, eta_out
        self._raise(self.lib, self.lib.spock_shard_apply_T(self.solver.h, 0, _ptr(z, nz, "apply_T: z"),
                                                           _ptr(eta, ne, "apply_T: eta"), None, None))
        self._exchange()
        self._raise(self.lib, self.lib.spock_shard_apply_T(self.solver.h, 1, None, None, _ptr(z_out, nz, "apply_T: z_out"),
                                                           _ptr(eta_out, ne, "apply_T: eta_out")))
        return z_out, eta_out

    def weights(self):
        zw = np.zeros(self.nz, dtype=np.uint8)
        ew = np.zeros(self.neta, dtype=np.uint8)
        P = C.POINTER(C.c_uint8)
        self._raise(self.lib, self.lib.spock_shard_weights(self.solver.h, zw.ctypes.data_as(P), ew.ctypes.data_as(P)))
        return zw.astype(bool), ew.astype(bool)

    def _collective(self, user, op, ptr, n):
        """Called by the library during a sharded solve (spock_collective_fn)."""
        torch, dist = self.torch, self.dist
        try:
            if op == 0:
                exchange(self.xbuf, self.plan, self.group, self.stream)
                return 0
            if op == 3:  # all-gather of n doubles per rank, in place (rank r's at [r n, (r + 1) n))
                w, r = self.plan.world, self.plan.rank
                t = torch.as_tensor(_DevArray(ptr, n * w), device="cuda")
                if dist.get_backend(self.group) == "nccl":
                    with torch.cuda.stream(self.stream):  # ordered after the library's writes
                        own = t[r * n:(r + 1) * n].clone()
                        dist.all_gather_into_tensor(t, own, group=self.group)
                else:
                    self.stream.synchronize()
                    own = t[r * n:(r + 1) * n].clone()
                    parts = [torch.empty(n, dtype=torch.float64) for _ in range(w)]
                    dist.all_gather(parts, own.cpu(), group=self.group)
                    t.copy_(torch.cat(parts).to(t.device))
                    torch.cuda.synchronize()
                return 0
            t = torch.as_tensor(_DevArray(ptr, n), device="cuda")
            rop = dist.ReduceOp.SUM if op == 1 else dist.ReduceOp.MAX
            if dist.get_backend(self.group) == "nccl":
                with torch.cuda.stream(self.stream):
                    dist.all_reduce(t, op=rop, group=self.group)
            else:
                self.stream.synchronize()
                h = t.cpu()
                dist.all_reduce(h, op=rop, group=self.group)
                t.copy_(h)
                torch.cuda.synchronize()
            return 0
        except Exception:  # pragma: no cover - reported as a runtime error by the library
            return 1

    def _solve(self, fn, x_init, history_capacity):
        from .capi import COLLECTIVE_FN
        from .solver import SolveResult, _ptr, make_status, status_dict
        if not self.native and not hasattr(self, "_cb"):
            self._cb = COLLECTIVE_FN(self._collective)
            self._raise(self.lib, self.lib.spock_shard_set_collectives(self.solver.h, self._cb, None))
        st, rn, br = make_status(history_capacity)
        z = np.zeros(self.nz)
        zs = np.zeros(self.nz)
        e = np.zeros(self.neta)
        x = None if x_init is None else np.ascontiguousarray(x_init, dtype=np.float64).ravel()
        if x is not None and x.size != self.solver.problem.nx:
            raise ValueError("solve: x_init has wrong length")
        rc = fn(self.solver.h, _ptr(x), None, None, _ptr(z), _ptr(zs), _ptr(e), C.byref(st))
        self._raise(self.lib, rc)
        # every rank's own entries -> the whole solution on every rank
        zw, ew = self.weights()
        out = []
        nccl = self.dist.get_backend(self.group) == "nccl"
        for v, w in ((z, zw), (zs, zw), (e, ew)):
            t = self.torch.from_numpy(np.where(w, v, 0.0))
            if nccl:
                t = t.cuda()
            self.dist.all_reduce(t, group=self.group)
            out.append(t.cpu().numpy())
        return SolveResult(out[0], out[1], out[2], status_dict(st, rn, br))

    def solve(self, x_init=None, history_capacity: int = 100000):
        """SuperMann (proj/src/solver.cpp:176-180) over the subtree-sharded tree."""
        return self._solve(self.lib.spock_solver_solve, x_init, history_capacity)

    def solve_cp(self, x_init=None, history_capacity: int = 100000):
        """Plain CP (proj/src/solver.cpp:182-187) over the subtree-sharded tree."""
        return self._solve(self.lib.spock_solver_solve_cp, x_init, history_capacity)

    def bench_step(self, parity: int) -> None:
        """One sharded T on the device-resident scratch iterates (no host copies)."""
        if self.native:
            self._raise(self.lib, self.lib.spock_shard_bench(self.solver.h, 2, parity))
            return
        self._raise(self.lib, self.lib.spock_shard_bench(self.solver.h, 0, parity))
        self._exchange()
        self._raise(self.lib, self.lib.spock_shard_bench(self.solver.h, 1, parity))
