"""ctypes view of the C-ABI in include/spock_b200.h.

``pack_problem`` flattens a :class:`~.problem.Raocp` into the
``spock_problem_desc`` the C-ABI consumes: column-major matrices packed back to
back in the reference's per-node order (problem.hpp:25-28).  The returned
object keeps every numpy buffer alive for as long as the descriptor is used.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from .problem import Raocp

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)

SPOCK_OK, SPOCK_EINVAL, SPOCK_ERUNTIME, SPOCK_ECUDA = 0, 1, 2, 3
TERMINATION = {0: "converged", 1: "max_iters", 2: "stalled", 3: "cancelled"}


class ProblemDesc(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32), ("nx", C.c_int32), ("nu", C.c_int32),
        ("horizon", C.c_int32), ("stop_stage", C.c_int32), ("num_events", C.c_int32),
        ("anc", _I), ("event", _I), ("prob", _D), ("cond_prob", _D),
        ("A", _D), ("B", _D), ("c", _D), ("Q", _D), ("R", _D), ("q", _D), ("r", _D),
        ("QN", _D), ("qN", _D),
        ("nc", _I), ("Gx", _D), ("Gu", _D), ("C_lo", _D), ("C_hi", _D),
        ("ncN", _I), ("GN", _D), ("CN_lo", _D), ("CN_hi", _D),
        ("risk_kind", _I), ("risk_rows", _I), ("risk_nnu", _I),
        ("risk_E", _D), ("risk_F", _D), ("risk_b", _D), ("risk_gamma", _D), ("risk_pi", _D),
        ("cone_nparts", _I), ("cone_kind", _I), ("cone_dim", _I),
        ("x_init", _D),
        ("layout", C.c_int32),
    ]


SPOCK_LAYOUT_ROW_MAJOR, SPOCK_LAYOUT_SHARED_G = 1, 2


PROGRESS_FN = C.CFUNCTYPE(None, C.c_int32, C.c_double, C.c_char, C.c_void_p)
CANCEL_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p)


class Params(C.Structure):
    _fields_ = [
        ("eps_abs", C.c_double), ("eps_rel", C.c_double), ("alpha", C.c_double),
        ("aa_memory", C.c_int32),
        ("c0", C.c_double), ("c1", C.c_double), ("c2", C.c_double),
        ("beta", C.c_double), ("sigma", C.c_double), ("lambda_", C.c_double),
        ("max_iters", C.c_int32), ("max_backtracks", C.c_int32), ("use_preconditioner", C.c_int32),
        ("progress", PROGRESS_FN), ("cancelled", CANCEL_FN), ("user", C.c_void_p),
        ("poll_every", C.c_int32),
    ]


class Status(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("reason", C.c_int32),
        ("xi1_inf", C.c_double), ("xi2_inf", C.c_double),
        ("k0_steps", C.c_int32), ("k1_steps", C.c_int32), ("k2_steps", C.c_int32), ("stalled_steps", C.c_int32),
        ("alpha", C.c_double), ("op_norm_estimate", C.c_double), ("op_norm_iterations", C.c_int32),
        ("op_norm_analytic_bound", C.c_double), ("op_norm_converged", C.c_int32),
        ("rnorm_history", _D), ("branch_history", C.c_char_p),
        ("history_capacity", C.c_int32), ("history_len", C.c_int32),
        ("n_T", C.c_int64), ("n_L", C.c_int64), ("n_Lt", C.c_int64),
    ]


def default_params(**kw) -> Params:
    """SpockParams defaults (proj/include/spock/solver.hpp:15-35)."""
    p = Params()
    p.eps_abs = 1e-6
    p.eps_rel = 1e-6
    p.alpha = 0.0
    p.aa_memory = 3
    p.c0 = p.c1 = p.c2 = 0.99
    p.beta = 0.5
    p.sigma = 0.1
    p.lambda_ = 1.0
    p.max_iters = 50000
    p.max_backtracks = 40
    p.use_preconditioner = 1
    p.poll_every = 1
    for k, v in kw.items():
        if k == "lambda":
            k = "lambda_"
        if k == "use_preconditioner":
            v = int(bool(v))
        setattr(p, k, v)
    return p


def _d(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_I)


def _colmajor_stack(mats) -> np.ndarray:
    """Concatenate per-node matrices in column-major order."""
    if isinstance(mats, np.ndarray) and mats.ndim == 3:
        if mats.shape[0] == 0:
            return np.zeros(1)
        return np.ascontiguousarray(mats.transpose(0, 2, 1)).reshape(-1)
    parts = [np.asarray(m, dtype=np.float64).T.reshape(-1) for m in mats]
    return np.concatenate(parts) if parts and sum(p.size for p in parts) else np.zeros(1)


def _flat(vecs) -> np.ndarray:
    if isinstance(vecs, np.ndarray):
        return np.ascontiguousarray(vecs, dtype=np.float64).reshape(-1) if vecs.size else np.zeros(1)
    parts = [np.asarray(v, dtype=np.float64).reshape(-1) for v in vecs]
    out = np.concatenate(parts) if parts else np.zeros(0)
    return out if out.size else np.zeros(1)


def _rowmajor_stack(mats) -> np.ndarray:
    """Per-node matrices back to back in C order (no copy for a C-contiguous stack)."""
    if isinstance(mats, np.ndarray) and mats.ndim == 3:
        if mats.shape[0] == 0:
            return np.zeros(1)
        return np.ascontiguousarray(mats, dtype=np.float64).reshape(-1)
    parts = [np.asarray(m, dtype=np.float64).reshape(-1) for m in mats]
    return np.concatenate(parts) if parts and sum(p.size for p in parts) else np.zeros(1)


def _shared_block(mats):
    """The one block of a per-node stack that repeats a single matrix
    (np.broadcast_to: stride 0 on the node axis), else None."""
    if isinstance(mats, np.ndarray) and mats.ndim == 3 and mats.shape[0] > 0 and mats.strides[0] == 0:
        return np.ascontiguousarray(mats[0], dtype=np.float64).reshape(-1)
    return None


class PackedProblem:
    """spock_problem_desc plus the buffers it points into.

    ``fast`` (the product's default) passes numpy stacks as they are: row-major
    blocks (SPOCK_LAYOUT_ROW_MAJOR, transposed by the library on host threads)
    and one shared constraint block when G is a broadcast (SPOCK_LAYOUT_SHARED_G);
    ``fast=False`` packs the reference's column-major layout (the oracle reads
    only that)."""

    def __init__(self, p: Raocp, fast: bool = True):
        tr = p.tree
        self.keep = []
        d = ProblemDesc()
        d.num_nodes = tr.num_nodes()
        d.nx, d.nu = p.nx, p.nu
        d.horizon, d.stop_stage, d.num_events = tr.horizon, tr.stop_stage, tr.num_events

        def K(a):
            self.keep.append(a)
            return a

        d.anc = _i(K(np.ascontiguousarray(tr.anc, dtype=np.int32)))
        d.event = _i(K(np.ascontiguousarray(tr.event, dtype=np.int32)))
        d.prob = _d(K(np.ascontiguousarray(tr.prob, dtype=np.float64)))
        d.cond_prob = _d(K(np.ascontiguousarray(tr.cond_prob, dtype=np.float64)))
        stack = _rowmajor_stack if fast else _colmajor_stack
        d.layout = SPOCK_LAYOUT_ROW_MAJOR if fast else 0
        d.A = _d(K(stack(p.A)))
        d.B = _d(K(stack(p.B)))
        d.c = _d(K(_flat(p.c)))
        d.Q = _d(K(stack(p.Q)))
        d.R = _d(K(stack(p.R)))
        d.q = _d(K(_flat(p.q)))
        d.r = _d(K(_flat(p.r)))
        d.QN = _d(K(stack(p.QN)))
        d.qN = _d(K(_flat(p.qN)))
        nc = np.array([b.dim() for b in p.C], dtype=np.int32)
        d.nc = _i(K(nc if nc.size else np.zeros(1, np.int32)))
        ncN_ = np.array([b.dim() for b in p.CN], dtype=np.int32)
        shared = None
        if fast:
            sh = [_shared_block(p.Gx), _shared_block(p.Gu), _shared_block(p.GN)]
            if all(x is not None for x in sh) and nc.size and ncN_.size and (nc == nc[0]).all() \
                    and (ncN_ == ncN_[0]).all():
                shared = sh
                d.layout |= SPOCK_LAYOUT_SHARED_G
        d.Gx = _d(K(shared[0] if shared else stack(p.Gx)))
        d.Gu = _d(K(shared[1] if shared else stack(p.Gu)))
        d.C_lo = _d(K(_flat([b.lo for b in p.C])))
        d.C_hi = _d(K(_flat([b.hi for b in p.C])))
        ncN = np.array([b.dim() for b in p.CN], dtype=np.int32)
        d.ncN = _i(K(ncN if ncN.size else np.zeros(1, np.int32)))
        d.GN = _d(K(shared[2] if shared else stack(p.GN)))
        d.CN_lo = _d(K(_flat([b.lo for b in p.CN])))
        d.CN_hi = _d(K(_flat([b.hi for b in p.CN])))
        rk = np.array([r.kind for r in p.risk], dtype=np.int32)
        rr = np.array([r.rows() for r in p.risk], dtype=np.int32)
        rn = np.array([r.F.shape[1] if r.F.ndim == 2 else 0 for r in p.risk], dtype=np.int32)
        d.risk_kind = _i(K(rk if rk.size else np.zeros(1, np.int32)))
        d.risk_rows = _i(K(rr if rr.size else np.zeros(1, np.int32)))
        d.risk_nnu = _i(K(rn if rn.size else np.zeros(1, np.int32)))
        d.risk_E = _d(K(_colmajor_stack([r.E for r in p.risk])))
        Fs = [r.F for r in p.risk if r.F.size]
        d.risk_F = _d(K(_colmajor_stack(Fs) if Fs else np.zeros(1)))
        d.risk_b = _d(K(_flat([r.b for r in p.risk])))
        d.risk_gamma = _d(K(np.array([r.gamma for r in p.risk] or [0.0], dtype=np.float64)))
        pis = [r.pi for r in p.risk if r.kind == 0 and r.pi is not None]
        d.risk_pi = _d(K(_flat(pis) if pis else np.zeros(1)))
        d.cone_nparts = _i(K(np.array([len(r.cone) for r in p.risk] or [0], dtype=np.int32)))
        d.cone_kind = _i(K(np.array([c.kind for r in p.risk for c in r.cone] or [0], dtype=np.int32)))
        d.cone_dim = _i(K(np.array([c.dim for r in p.risk for c in r.cone] or [0], dtype=np.int32)))
        d.x_init = _d(K(np.ascontiguousarray(p.x_init, dtype=np.float64)))
        self.desc = d

    def ref(self):
        return C.byref(self.desc)


def pack_problem(p: Raocp, fast: bool = True) -> PackedProblem:
    return PackedProblem(p, fast)


def _lib_path() -> str:
    # SPOCK_LIB: an alternative in-tree build of the same library (tools/ A/B runs)
    alt = os.environ.get("SPOCK_LIB")
    if alt:
        return alt
    here = os.path.dirname(os.path.abspath(__file__))
    return os.path.join(here, "_build", "libspock_b200.so")


_LIB: Optional[C.CDLL] = None


COLLECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64)


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library; fail loudly if it is missing (no CPU fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _lib_path()
    if not os.path.exists(path):
        raise RuntimeError(
            f"spock-b200 CUDA library not built: {path} is missing; run __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.POINTER
    lib.spock_last_error.restype = C.c_char_p
    lib.spock_params_default.argtypes = [P(Params)]
    lib.spock_solver_create.argtypes = [P(ProblemDesc), P(Params), P(C.c_void_p)]
    lib.spock_solver_destroy.argtypes = [C.c_void_p]
    lib.spock_solver_dims.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64)]
    lib.spock_solver_alpha.argtypes = [C.c_void_p]
    lib.spock_solver_alpha.restype = C.c_double
    for fn in ("spock_solver_solve", "spock_solver_solve_cp"):
        getattr(lib, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, P(Status)]
    lib.spock_solver_apply_T.argtypes = [C.c_void_p] + [C.c_void_p] * 4
    lib.spock_op_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.spock_op_apply_adjoint.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.spock_op_m_norm.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, P(C.c_double)]
    for fn in ("spock_proj_s1", "spock_proj_s2", "spock_proj_s3"):
        getattr(lib, fn).argtypes = [C.c_void_p, C.c_void_p]
    lib.spock_solver_unscale_primal.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.spock_bench_T.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, P(C.c_double)]
    lib.spock_bench_kernels.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    lib.spock_traffic_model.argtypes = [C.c_void_p, C.c_void_p, P(C.c_int32)]
    lib.spock_solver_t_path.argtypes = [C.c_void_p]
    lib.spock_solver_t_path.restype = C.c_char_p
    PI = P(C.c_int32)
    lib.spock_shard_setup.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, PI, C.c_int32, PI, C.c_int32,
                                      PI, C.c_int32, PI, C.c_int32, C.c_void_p]
    lib.spock_shard_apply_T.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 4
    lib.spock_shard_bench.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
    lib.spock_shard_masks.argtypes = [C.c_void_p, P(C.c_uint8), P(C.c_uint8)]
    lib.spock_shard_weights.argtypes = [C.c_void_p, P(C.c_uint8), P(C.c_uint8)]
    lib.spock_shard_set_collectives.argtypes = [C.c_void_p, COLLECTIVE_FN, C.c_void_p]
    lib.spock_solver_stream.argtypes = [C.c_void_p]
    lib.spock_solver_stream.restype = C.c_void_p
    lib.spock_solver_set_grid_cap.argtypes = [C.c_void_p, C.c_int32]
    lib.spock_solver_grid.argtypes = [C.c_void_p]
    lib.spock_solver_grid.restype = C.c_int32
    lib.spock_solver_loop_path.argtypes = [C.c_void_p]
    lib.spock_solver_loop_path.restype = C.c_char_p
    lib.spock_anderson_lstsq.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
    lib.spock_nccl_unique_id.argtypes = [C.c_void_p]
    lib.spock_shard_nccl_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
    _LIB = lib
    return lib


EXPORTED_SYMBOLS = [
    "spock_last_error", "spock_params_default", "spock_solver_create", "spock_solver_destroy",
    "spock_solver_dims", "spock_solver_alpha", "spock_solver_solve", "spock_solver_solve_cp",
    "spock_solver_apply_T", "spock_op_apply", "spock_op_apply_adjoint", "spock_op_m_norm",
    "spock_proj_s1", "spock_proj_s2", "spock_proj_s3", "spock_solver_unscale_primal", "spock_bench_T",
    "spock_bench_kernels", "spock_traffic_model", "spock_solver_t_path", "spock_shard_setup", "spock_shard_apply_T",
    "spock_shard_bench", "spock_shard_masks", "spock_shard_weights", "spock_shard_set_collectives",
    "spock_solver_stream", "spock_solver_set_grid_cap", "spock_solver_grid", "spock_anderson_lstsq",
    "spock_solver_loop_path", "spock_nccl_unique_id", "spock_shard_nccl_init",
]


def anderson_lstsq(Md, r):
    """The solver's Anderson least squares (spock_anderson_lstsq): kappa =
    argmin ||M_d kappa - r|| with the reference's rank rules, double-double Gram."""
    import numpy as np
    lib = load_library()
    A = np.asfortranarray(Md, dtype=np.float64)
    b = np.ascontiguousarray(r, dtype=np.float64)
    k = np.zeros(A.shape[1])
    rc = lib.spock_anderson_lstsq(A.ctypes.data, A.shape[0], A.shape[1], b.ctypes.data, k.ctypes.data)
    if rc != SPOCK_OK:
        raise ValueError(lib.spock_last_error().decode())
    return k
