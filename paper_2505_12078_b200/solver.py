"""Python mirror of the reference's solver API over the C-ABI.

``SpockSolver`` mirrors ``spock::SpockSolver`` (proj/include/spock/solver.hpp:99-145):
construction performs the reference's setup (validation, preconditioning,
SOC epigraph data, offline factorisation, ||L|| estimate) behind
``spock_solver_create``; ``solve``/``solve_cp``/``apply_T`` and the operator
entry points map 1:1 onto the C-ABI functions.  Errors surface as the
reference's exception kinds: ``ValueError`` for std::invalid_argument and
``RuntimeError`` for std::runtime_error.

Vectors may be numpy arrays (host) or CUDA torch tensors (device); the library
detects the pointer kind.  There is no CPU fallback: if the CUDA library is
missing the constructor raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import capi
from .problem import Raocp


@dataclass
class SolveResult:
    z: np.ndarray
    z_scaled: np.ndarray
    eta: np.ndarray
    status: dict = field(default_factory=dict)


def _raise(lib, rc: int, prefix: str = "spock"):
    if rc == capi.SPOCK_OK:
        return
    msg = lib.spock_last_error().decode() if hasattr(lib, "spock_last_error") else prefix
    if rc == capi.SPOCK_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a, n: Optional[int] = None, what: str = "vector"):
    """Raw pointer of a numpy array or torch tensor: float64, contiguous and, when
    `n` is given, exactly n entries (the reference throws std::invalid_argument
    on wrong dimensions, proj/src/solver.cpp:191,200-201; here a short buffer
    would otherwise be read or written out of bounds by the library)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64:
            raise ValueError(f"{what}: dtype must be float64, got {a.dtype}")
        if not a.flags.c_contiguous:
            raise ValueError(f"{what}: must be contiguous")
        if n is not None and a.size != n:
            raise ValueError(f"{what} has wrong length ({a.size}, expected {n})")
        return a.ctypes.data
    # torch tensor
    import torch
    if not isinstance(a, torch.Tensor):
        raise ValueError(f"{what}: expected a numpy array or torch tensor, got {type(a).__name__}")
    if a.dtype != torch.float64:
        raise ValueError(f"{what}: dtype must be torch.float64, got {a.dtype}")
    if not a.is_contiguous():
        raise ValueError(f"{what}: must be contiguous")
    if n is not None and a.numel() != n:
        raise ValueError(f"{what} has wrong length ({a.numel()}, expected {n})")
    return a.data_ptr()


def _f64(a):
    """Host copy as contiguous float64 unless `a` is already a float64 array/tensor."""
    if a is None or (not isinstance(a, np.ndarray) and hasattr(a, "data_ptr")):
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


def _current_device():
    try:
        import torch
        return torch.cuda.current_device() if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover - torch without CUDA
        return None


def status_dict(st: capi.Status, rn: np.ndarray, br) -> dict:
    n = min(st.history_len, st.history_capacity)
    return dict(
        iterations=st.iterations, reason=capi.TERMINATION.get(st.reason, str(st.reason)),
        xi1_inf=st.xi1_inf, xi2_inf=st.xi2_inf, k0_steps=st.k0_steps, k1_steps=st.k1_steps,
        k2_steps=st.k2_steps, stalled_steps=st.stalled_steps, alpha=st.alpha,
        op_norm=dict(estimate=st.op_norm_estimate, iterations=st.op_norm_iterations,
                     analytic_bound=st.op_norm_analytic_bound, converged=bool(st.op_norm_converged)),
        rnorm_history=rn[:n].copy(), branches=br.raw[:n].decode(), history_len=st.history_len,
        n_T=st.n_T, n_L=st.n_L, n_Lt=st.n_Lt)


def make_status(capacity: int):
    st = capi.Status()
    rn = np.zeros(max(capacity, 1))
    br = C.create_string_buffer(max(capacity, 1))
    st.rnorm_history = rn.ctypes.data_as(C.POINTER(C.c_double))
    st.branch_history = C.cast(br, C.c_char_p)
    st.history_capacity = capacity
    return st, rn, br


class SpockSolver:
    """spock::SpockSolver over the B200 C-ABI."""

    def __init__(self, problem: Raocp, progress=None, cancelled=None, **params):
        self.lib = capi.load_library()
        self.problem = problem
        self.packed = capi.pack_problem(problem)
        self._cbs = []
        prm = capi.default_params(**params)
        if progress is not None:
            cb = capi.PROGRESS_FN(lambda k, w, b, u: progress(k, w, b.decode()))
            self._cbs.append(cb)
            prm.progress = cb
        if cancelled is not None:
            cb2 = capi.CANCEL_FN(lambda u: int(bool(cancelled())))
            self._cbs.append(cb2)
            prm.cancelled = cb2
        self.params = prm
        h = C.c_void_p()
        _raise(self.lib, self.lib.spock_solver_create(self.packed.ref(), C.byref(prm), C.byref(h)))
        self.h = h
        nz, ne = C.c_int64(), C.c_int64()
        self.lib.spock_solver_dims(self.h, C.byref(nz), C.byref(ne))
        self.nz, self.neta = nz.value, ne.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.spock_solver_destroy(h)
            self.h = None

    @property
    def alpha(self) -> float:
        return self.lib.spock_solver_alpha(self.h)

    def _run(self, fn, x_init, warm, capacity):
        st, rn, br = make_status(capacity)
        z = np.zeros(self.nz)
        zs = np.zeros(self.nz)
        e = np.zeros(self.neta)
        x = None if x_init is None else np.ascontiguousarray(x_init, dtype=np.float64).ravel()
        if x is not None and x.size != self.problem.nx:
            raise ValueError("solve: x_init has wrong length")
        wz = we = None
        if warm is not None:
            wz = np.ascontiguousarray(warm[0], dtype=np.float64).ravel()
            we = np.ascontiguousarray(warm[1], dtype=np.float64).ravel()
            if wz.size != self.nz or we.size != self.neta:
                raise ValueError("solve: warm start has wrong dimensions")
        rc = fn(self.h, _ptr(x), _ptr(wz), _ptr(we), _ptr(z), _ptr(zs), _ptr(e), C.byref(st))
        _raise(self.lib, rc)
        return SolveResult(z, zs, e, status_dict(st, rn, br))

    def solve(self, x_init=None, warm=None, history_capacity: int = 100000) -> SolveResult:
        """SpockSolver::solve (proj/src/solver.cpp:176-180)."""
        return self._run(self.lib.spock_solver_solve, x_init, warm, history_capacity)

    def solve_cp(self, x_init=None, warm=None, history_capacity: int = 100000) -> SolveResult:
        """SpockSolver::solve_cp (proj/src/solver.cpp:182-187)."""
        return self._run(self.lib.spock_solver_solve_cp, x_init, warm, history_capacity)

    def apply_T(self, z, eta, z_out=None, eta_out=None):
        """SpockSolver::apply_T (proj/src/solver.cpp:148-164)."""
        z, eta = _f64(z), _f64(eta)
        if z_out is None:
            z_out = np.empty(self.nz)
        if eta_out is None:
            eta_out = np.empty(self.neta)
        _raise(self.lib, self.lib.spock_solver_apply_T(self.h, _ptr(z, self.nz, "apply_T: z"), _ptr(eta, self.neta, "apply_T: eta"),
                                                       _ptr(z_out, self.nz, "apply_T: z_out"),
                                                       _ptr(eta_out, self.neta, "apply_T: eta_out")))
        return z_out, eta_out

    def apply_L(self, z, out=None):
        out = np.empty(self.neta) if out is None else out
        _raise(self.lib, self.lib.spock_op_apply(self.h, _ptr(_f64(z), self.nz, "apply: z"), _ptr(out, self.neta, "apply: out")))
        return out

    def apply_Lt(self, eta, out=None):
        out = np.empty(self.nz) if out is None else out
        _raise(self.lib, self.lib.spock_op_apply_adjoint(self.h, _ptr(_f64(eta), self.neta, "apply_adjoint: eta"),
                                                         _ptr(out, self.nz, "apply_adjoint: out")))
        return out

    def m_norm(self, z, eta, alpha: float) -> float:
        o = C.c_double()
        _raise(self.lib, self.lib.spock_op_m_norm(self.h, _ptr(_f64(z), self.nz, "m_norm: z"),
                                                  _ptr(_f64(eta), self.neta, "m_norm: eta"), alpha, C.byref(o)))
        return o.value

    def proj_s1(self, z):
        z = np.array(z, dtype=np.float64)
        _raise(self.lib, self.lib.spock_proj_s1(self.h, _ptr(z, self.nz, "proj_s1: z")))
        return z

    def proj_s2(self, z):
        z = np.array(z, dtype=np.float64)
        _raise(self.lib, self.lib.spock_proj_s2(self.h, _ptr(z, self.nz, "proj_s2: z")))
        return z

    def proj_s3(self, eta):
        eta = np.array(eta, dtype=np.float64)
        _raise(self.lib, self.lib.spock_proj_s3(self.h, _ptr(eta, self.neta, "proj_s3: eta")))
        return eta

    def unscale_primal(self, zs):
        out = np.empty(self.nz)
        _raise(self.lib, self.lib.spock_solver_unscale_primal(
            self.h, _ptr(np.ascontiguousarray(zs, dtype=np.float64), self.nz, "unscale_primal: z"), _ptr(out)))
        return out

    def bench_T(self, k: int, use_graph: bool = True, flush_l2: bool = False) -> float:
        """Device ms for k back-to-back CP applications (benchmark helper)."""
        ms = C.c_double()
        _raise(self.lib, self.lib.spock_bench_T(self.h, int(k), int(use_graph), int(flush_l2), C.byref(ms)))
        return ms.value

    def bench_kernels(self, k: int, flush_l2: bool = True) -> np.ndarray:
        """Average device ms of [L*, S1 sweeps, S2, L+S3, T]."""
        out = np.zeros(5)
        _raise(self.lib, self.lib.spock_bench_kernels(self.h, int(k), int(flush_l2), out.ctypes.data))
        return out

    @property
    def t_path(self) -> str:
        """Device schedule of T: 'fused', 'wide' or 'stages'."""
        return self.lib.spock_solver_t_path(self.h).decode()

    def traffic_model(self):
        """Algorithmic bytes of [L*, S1, S2, L+S3, T] and kernel launches per T."""
        out = np.zeros(5)
        n = C.c_int32()
        _raise(self.lib, self.lib.spock_traffic_model(self.h, out.ctypes.data, C.byref(n)))
        return out, n.value

    @property
    def loop_path(self) -> str:
        """Loop a solve runs: 'small' (one CTA), 'graph' (CUDA graph) or 'host'."""
        return self.lib.spock_solver_loop_path(self.h).decode()

    @property
    def grid(self) -> int:
        """CTAs of the fused T launch (0 when T runs on another schedule)."""
        return int(self.lib.spock_solver_grid(self.h))

    def set_grid_cap(self, ctas: int) -> None:
        """Cap the fused T launch at `ctas` CTAs (0: full device); before the first solve."""
        _raise(self.lib, self.lib.spock_solver_set_grid_cap(self.h, int(ctas)))


def residuals_xi(op, z, eta, z_next, eta_next, alpha: float):
    """Termination residuals of a CP step (proj/src/solver.cpp:31-43):
    xi1 = (z - z+)/alpha - L*(eta - eta+), xi2 = (eta - eta+)/alpha - L(z - z+),
    with `op`'s L and L* (the device operators for a SpockSolver)."""
    dz = np.asarray(z, dtype=np.float64) - np.asarray(z_next, dtype=np.float64)
    de = np.asarray(eta, dtype=np.float64) - np.asarray(eta_next, dtype=np.float64)
    return dz / alpha - op.apply_Lt(de), de / alpha - op.apply_L(dz)


class BatchSolver:
    """Several x_init of one problem solved side by side (batched
    multi-x_init / warm-started MPC solves; the reference solves one x_init per
    call, proj/include/spock/solver.hpp:104-105, warm start 58-61).

    On narrow trees one solve is bound by the latency of the 2N+2 dependent
    tree levels and leaves most SMs idle, so `streams` solvers -- each with its
    own device state, CUDA stream and cached solve graph, its fused T launch
    capped to 1/streams of the device's CTAs -- run concurrently from host
    threads (the C calls release the GIL).  Results are bitwise those of
    sequential SpockSolver solves: every T item and reduction has a fixed
    summation order whatever the grid.  On wide trees T is HBM-bound and the
    streams only overlap the small kernels."""

    def __init__(self, problem: Raocp, streams: int = 4, grid_cap: Optional[int] = None, **params):
        if streams < 1:
            raise ValueError("BatchSolver: streams must be >= 1")
        import threading
        self.solvers = [None] * streams
        errs = []
        dev = _current_device()

        def make(k):
            try:
                if dev is not None:  # the current device is per thread: build on the caller's
                    import torch
                    torch.cuda.set_device(dev)
                self.solvers[k] = SpockSolver(problem, **params)
            except Exception as e:  # surfaced in the caller's thread
                errs.append(e)

        th = [threading.Thread(target=make, args=(k,)) for k in range(streams)]
        for h in th:
            h.start()
        for h in th:
            h.join()
        if errs:
            raise errs[0]
        full = self.solvers[0].grid
        cap = grid_cap if grid_cap is not None else (max(16, full // streams) if streams > 1 else 0)
        for s in self.solvers:
            s.set_grid_cap(cap)

    def _run(self, algo: str, x_inits, warm):
        import threading
        n = len(x_inits)
        if warm is not None and len(warm) != n:
            raise ValueError("BatchSolver: one warm start per x_init")
        out = [None] * n
        errs = []
        nxt = [0]
        lock = threading.Lock()

        def worker(s):
            while True:
                with lock:
                    k = nxt[0]
                    nxt[0] += 1
                if k >= n or errs:
                    return
                try:
                    out[k] = getattr(s, algo)(x_inits[k], None if warm is None else warm[k])
                except Exception as e:  # surfaced in the caller's thread
                    errs.append(e)
                    return

        th = [threading.Thread(target=worker, args=(s,)) for s in self.solvers[:max(1, min(n, len(self.solvers)))]]
        for h in th:
            h.start()
        for h in th:
            h.join()
        if errs:
            raise errs[0]
        return out

    def solve(self, x_inits, warm=None):
        """SuperMann solves of every x_init (optional per-x_init warm (z, eta))."""
        return self._run("solve", x_inits, warm)

    def solve_cp(self, x_inits, warm=None):
        """Plain CP solves of every x_init."""
        return self._run("solve_cp", x_inits, warm)
