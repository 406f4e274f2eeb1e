"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the parity oracle.

The oracle (oracle/*.cpp) is a CPU restatement of the reference SPOCK solver
(arxiv/paper_2505_12078 proj/src/*.cpp).  This module exposes it with the same
method names as ``paper_2505_12078_b200.solver.SpockSolver`` so parity tests can
run both on byte-identical problems.  Only tests/, __graft_entry__.smoke() and
bench.py may import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2505_12078_b200 import capi
from paper_2505_12078_b200.solver import SolveResult, make_status, status_dict

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_LIB = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        P, V, D, I = C.POINTER, C.c_void_p, C.c_double, C.c_int
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_solver_create.argtypes = [P(capi.ProblemDesc), P(capi.Params), P(V)]
        L.oracle_solver_destroy.argtypes = [V]
        L.oracle_solver_dims.argtypes = [V, P(C.c_int64), P(C.c_int64)]
        L.oracle_solver_alpha.argtypes = [V]
        L.oracle_solver_alpha.restype = D
        L.oracle_opnorm.argtypes = [V, P(D), P(I), P(D), P(I)]
        for fn in ("oracle_solver_solve", "oracle_solver_solve_cp"):
            getattr(L, fn).argtypes = [V] * 7 + [P(capi.Status)]
        L.oracle_apply_T.argtypes = [V] * 5
        L.oracle_bench_T.argtypes = [V, I, P(D)]
        L.oracle_apply_L.argtypes = [V] * 3
        L.oracle_apply_Lt.argtypes = [V] * 3
        L.oracle_m_norm.argtypes = [V, V, V, D, P(D)]
        for fn in ("oracle_proj_s1", "oracle_proj_s2", "oracle_proj_s3"):
            getattr(L, fn).argtypes = [V, V]
        L.oracle_unscale_primal.argtypes = [V, V, V]
        L.oracle_primal_layout.argtypes = [V, V, V, V]
        L.oracle_dual_layout.argtypes = [V] * 9
        L.oracle_soc_dims.argtypes = [V, I, I, P(I), P(I), P(D)]
        L.oracle_soc_data.argtypes = [V, I, I, V, V, V, V]
        L.oracle_precond.argtypes = [V, V, V, V, V, P(D), P(I)]
        L.oracle_scaled_mat.argtypes = [V, I, I, V]
        L.oracle_cache_mat.argtypes = [V, I, I, V, P(I), P(I)]
        L.oracle_proj_soc.argtypes = [V, I]
        L.oracle_soc_quadlin.argtypes = [V, V, I, P(I), V, V, V, V]
        L.oracle_aa_create.argtypes = [I]
        L.oracle_aa_create.restype = V
        L.oracle_aa_destroy.argtypes = [V]
        L.oracle_aa_direction.argtypes = [V, V, I, V]
        L.oracle_colpiv_qr_solve.argtypes = [V, I, I, V, V]
        L.oracle_estimate_norm_identity.argtypes = [I]
        L.oracle_estimate_norm_identity.restype = D
        L.oracle_philox_normals.argtypes = [C.c_uint64, I, V]
        L.oracle_philox_u64.argtypes = [C.c_uint64, I, V]
        L.oracle_set_num_threads.argtypes = [I]
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data


def _chk(rc):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == capi.SPOCK_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


class OracleSolver:
    """CPU restatement of spock::SpockSolver (proj/src/solver.cpp)."""

    def __init__(self, problem, progress=None, cancelled=None, **params):
        self.L = lib()
        self.problem = problem
        self.packed = capi.pack_problem(problem, fast=False)  # the reference's column-major layout
        prm = capi.default_params(**params)
        self._cbs = []
        if progress is not None:
            cb = capi.PROGRESS_FN(lambda k, w, b, u: progress(k, w, b.decode()))
            self._cbs.append(cb)
            prm.progress = cb
        if cancelled is not None:
            cb2 = capi.CANCEL_FN(lambda u: int(bool(cancelled())))
            self._cbs.append(cb2)
            prm.cancelled = cb2
        h = C.c_void_p()
        _chk(self.L.oracle_solver_create(self.packed.ref(), C.byref(prm), C.byref(h)))
        self.h = h
        nz, ne = C.c_int64(), C.c_int64()
        self.L.oracle_solver_dims(self.h, C.byref(nz), C.byref(ne))
        self.nz, self.neta = nz.value, ne.value
        tr = problem.tree
        self.nn, self.nnl, self.nl = tr.num_nodes(), tr.num_nonleaf(), tr.num_leaves()

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.L.oracle_solver_destroy(self.h)
            self.h = None

    @property
    def alpha(self) -> float:
        return self.L.oracle_solver_alpha(self.h)

    def op_norm(self) -> dict:
        e, b = C.c_double(), C.c_double()
        it, cv = C.c_int(), C.c_int()
        self.L.oracle_opnorm(self.h, C.byref(e), C.byref(it), C.byref(b), C.byref(cv))
        return dict(estimate=e.value, iterations=it.value, analytic_bound=b.value, converged=bool(cv.value))

    def _run(self, fn, x_init, warm, cap):
        st, rn, br = make_status(cap)
        z, zs, e = np.zeros(self.nz), np.zeros(self.nz), np.zeros(self.neta)
        x = None if x_init is None else np.ascontiguousarray(x_init, dtype=np.float64)
        wz = we = None
        if warm is not None:
            wz = np.ascontiguousarray(warm[0], dtype=np.float64)
            we = np.ascontiguousarray(warm[1], dtype=np.float64)
        _chk(fn(self.h, _p(x), _p(wz), _p(we), _p(z), _p(zs), _p(e), C.byref(st)))
        return SolveResult(z, zs, e, status_dict(st, rn, br))

    def solve(self, x_init=None, warm=None, history_capacity: int = 100000):
        return self._run(self.L.oracle_solver_solve, x_init, warm, history_capacity)

    def solve_cp(self, x_init=None, warm=None, history_capacity: int = 100000):
        return self._run(self.L.oracle_solver_solve_cp, x_init, warm, history_capacity)

    def apply_T(self, z, eta):
        z = np.ascontiguousarray(z, dtype=np.float64)
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        zo, eo = np.empty_like(z), np.empty_like(eta)
        _chk(self.L.oracle_apply_T(self.h, _p(z), _p(eta), _p(zo), _p(eo)))
        return zo, eo

    def bench_T(self, k: int) -> float:
        ms = C.c_double()
        _chk(self.L.oracle_bench_T(self.h, int(k), C.byref(ms)))
        return ms.value

    def apply_L(self, z):
        z = np.ascontiguousarray(z, dtype=np.float64)
        o = np.empty(self.neta)
        _chk(self.L.oracle_apply_L(self.h, _p(z), _p(o)))
        return o

    def apply_Lt(self, eta):
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        o = np.empty(self.nz)
        _chk(self.L.oracle_apply_Lt(self.h, _p(eta), _p(o)))
        return o

    def m_norm(self, z, eta, alpha):
        o = C.c_double()
        _chk(self.L.oracle_m_norm(self.h, _p(np.ascontiguousarray(z, dtype=np.float64)),
                                  _p(np.ascontiguousarray(eta, dtype=np.float64)), alpha, C.byref(o)))
        return o.value

    def proj_s1(self, z):
        z = np.array(z, dtype=np.float64)
        _chk(self.L.oracle_proj_s1(self.h, _p(z)))
        return z

    def proj_s2(self, z):
        z = np.array(z, dtype=np.float64)
        _chk(self.L.oracle_proj_s2(self.h, _p(z)))
        return z

    def proj_s3(self, eta):
        eta = np.array(eta, dtype=np.float64)
        _chk(self.L.oracle_proj_s3(self.h, _p(eta)))
        return eta

    def unscale_primal(self, zs):
        o = np.empty(self.nz)
        _chk(self.L.oracle_unscale_primal(self.h, _p(np.ascontiguousarray(zs, dtype=np.float64)), _p(o)))
        return o

    # ---- setup exports ----
    def primal_layout(self) -> dict:
        b = np.zeros(3, np.int32)
        yo = np.zeros(max(self.nnl, 1), np.int32)
        yd = np.zeros(max(self.nnl, 1), np.int32)
        self.L.oracle_primal_layout(self.h, _p(b), _p(yo), _p(yd))
        return dict(n=self.nz, u_base=int(b[0]), tau_base=int(b[1]), s_base=int(b[2]),
                    y_off=yo[:self.nnl], y_dim=yd[:self.nnl])

    def dual_layout(self) -> dict:
        a = [np.zeros(max(n, 1), np.int32) for n in
             (self.nnl, self.nnl, self.nnl, self.nn - 1, self.nn - 1, self.nl, self.nl, self.nl)]
        self.L.oracle_dual_layout(self.h, *[_p(x) for x in a])
        keys = ["seg1_off", "seg1_nc", "seg1_ydim", "seg2_off", "seg2_dim", "seg3_off", "seg3_nc", "seg3_socdim"]
        lens = [self.nnl] * 3 + [self.nn - 1] * 2 + [self.nl] * 3
        out = {k: v[:n] for k, v, n in zip(keys, a, lens)}
        out["n"] = self.neta
        return out

    def soc(self, which: int, idx: int) -> dict:
        n, p, lm = C.c_int(), C.c_int(), C.c_double()
        self.L.oracle_soc_dims(self.h, which, idx, C.byref(n), C.byref(p), C.byref(lm))
        n, p = n.value, p.value
        hm = np.zeros(max(p * n, 1))
        qk = np.zeros(n)
        a = np.zeros(p + 2)
        sf = np.zeros(max(p * p, 1))
        self.L.oracle_soc_data(self.h, which, idx, _p(hm), _p(qk), _p(a), _p(sf))
        return dict(n=n, p=p, lambda_max=lm.value, head_map=hm[:p * n].reshape(n, p).T.copy(), q_kernel=qk, a=a,
                    sqrt_factor=sf[:p * p].reshape(p, p).T.copy())

    def precond(self) -> dict:
        nx, nu = self.problem.nx, self.problem.nu
        sx, su, sxN = np.zeros(nx), np.zeros(nu), np.zeros(nx)
        cs = np.zeros(max(self.nnl, 1))
        ch, ident = C.c_double(), C.c_int()
        self.L.oracle_precond(self.h, _p(sx), _p(su), _p(sxN), _p(cs), C.byref(ch), C.byref(ident))
        return dict(sx=sx, su=su, sxN=sxN, cstr_scale=cs[:self.nnl], c_hat=ch.value, is_identity=bool(ident.value))

    def scaled_mat(self, which: int, idx: int, shape) -> np.ndarray:
        o = np.zeros(shape[0] * shape[1])
        self.L.oracle_scaled_mat(self.h, which, idx, _p(o))
        return o.reshape(shape[1], shape[0]).T.copy()

    def cache_mat(self, which: int, idx: int) -> np.ndarray:
        r, c = C.c_int(), C.c_int()
        self.L.oracle_cache_mat(self.h, which, idx, None, C.byref(r), C.byref(c))
        o = np.zeros(max(r.value * c.value, 1))
        self.L.oracle_cache_mat(self.h, which, idx, _p(o), C.byref(r), C.byref(c))
        return o[:r.value * c.value].reshape(c.value, r.value).T.copy()


def proj_soc(v) -> np.ndarray:
    v = np.array(v, dtype=np.float64)
    _chk(lib().oracle_proj_soc(_p(v), v.size))
    return v


def soc_data_quadlin(Q, q) -> dict:
    Q = np.asarray(Q, dtype=np.float64)
    n = Q.shape[0]
    Qc = np.ascontiguousarray(Q.T)
    qv = np.ascontiguousarray(q, dtype=np.float64)
    p = C.c_int()
    hm, qk, a, sf = np.zeros(max(n * n, 1)), np.zeros(n), np.zeros(n + 2), np.zeros(max(n * n, 1))
    _chk(lib().oracle_soc_quadlin(_p(Qc), _p(qv), n, C.byref(p), _p(hm), _p(qk), _p(a), _p(sf)))
    p = p.value
    return dict(p=p, head_map=hm[:p * n].reshape(n, p).T.copy(), q_kernel=qk, a=a[:p + 2],
                sqrt_factor=sf[:p * p].reshape(p, p).T.copy())


class Anderson:
    def __init__(self, m: int):
        self.L = lib()
        self.h = self.L.oracle_aa_create(m)

    def direction(self, r) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        o = np.empty_like(r)
        self.L.oracle_aa_direction(self.h, _p(r), r.size, _p(o))
        return o

    def __del__(self):
        if getattr(self, "h", None):
            self.L.oracle_aa_destroy(self.h)
            self.h = None


def colpiv_qr_solve(A, b) -> np.ndarray:
    """Eigen ColPivHouseholderQR(A).setThreshold(1e-12).solve(b) as restated
    (orc_la.cpp; the reference's Anderson least squares, solver.cpp:73-75)."""
    A = np.asfortranarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.shape[1])
    lib().oracle_colpiv_qr_solve(A.ctypes.data, A.shape[0], A.shape[1], b.ctypes.data, x.ctypes.data)
    return x


def estimate_norm_identity(n: int) -> float:
    return lib().oracle_estimate_norm_identity(n)


def philox_normals(seed: int, n: int) -> np.ndarray:
    o = np.zeros(n)
    lib().oracle_philox_normals(seed, n, _p(o))
    return o


def philox_u64(seed: int, n: int) -> np.ndarray:
    o = np.zeros(n, dtype=np.uint64)
    lib().oracle_philox_u64(seed, n, _p(o))
    return o
