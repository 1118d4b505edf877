"""ctypes front end of oracle.c (plain C, fp64, -ffp-contract=off).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Argument marshalling only:
all arithmetic is in oracle.c, which cites PAPER.md for each step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from synth import CSR

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


MAXSTEP = 160


class _Trace(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("M_eff", C.c_int32),
        ("normal", C.c_int32),
        ("norm", C.c_double), ("a", C.c_double), ("r0", C.c_double), ("eps_g0", C.c_double),
        ("taylor_nnz_unf", C.c_int64 * MAXSTEP), ("taylor_nnz", C.c_int64 * MAXSTEP),
        ("taylor_passes", C.c_int32 * MAXSTEP),
        ("taylor_tau", C.c_double * MAXSTEP), ("taylor_dropped", C.c_double * MAXSTEP),
        ("taylor_l1", C.c_int64 * MAXSTEP), ("taylor_l2", C.c_int64 * MAXSTEP),
        ("sq_nnz_unf", C.c_int64 * MAXSTEP), ("sq_nnz", C.c_int64 * MAXSTEP),
        ("sq_passes", C.c_int32 * MAXSTEP),
        ("sq_eps_g", C.c_double * MAXSTEP), ("sq_tau", C.c_double * MAXSTEP),
        ("sq_dropped", C.c_double * MAXSTEP), ("sq_normIT", C.c_double * MAXSTEP),
        ("sq_l1", C.c_int64 * MAXSTEP), ("sq_l2", C.c_int64 * MAXSTEP),
        ("sq_fmas", C.c_double * MAXSTEP),
    ]


class _Options(C.Structure):
    _fields_ = [
        ("plan_norm", C.c_int32), ("normal", C.c_int32), ("threshold_mode", C.c_int32),
        ("filter", C.c_int32), ("m_cap", C.c_int32), ("n_window", C.c_int32),
        ("force_M", C.c_int32), ("force_N", C.c_int32), ("output_T", C.c_int32),
        ("nthreads", C.c_int32), ("ssat", C.c_int32), ("e_r", C.c_double),
    ]


@dataclass
class Options:
    plan_norm: str = "one"        # "one" (BASELINE.json) | "fro"
    normal: int = -1              # -1 auto (symmetric / skew-symmetric), 0, 1
    threshold_mode: str = "rel_prev"  # "rel_prev" (reading R4) | "abs" (P:422 as printed)
    filter: bool = True
    m_cap: int = 120
    n_window: int = 50
    force_M: int = -1
    force_N: int = -1
    output_T: bool = False
    nthreads: int = 1
    ssat: bool = False            # SSAT baseline (Table 1): E_0 = I + T^_0, E_i = E_{i-1}^2
    e_r: float = 0.1

    def to_c(self) -> _Options:
        return _Options(0 if self.plan_norm == "one" else 1, self.normal,
                        0 if self.threshold_mode == "rel_prev" else 1, int(self.filter),
                        self.m_cap, self.n_window, self.force_M, self.force_N,
                        int(self.output_T), self.nthreads, int(self.ssat), self.e_r)


def _L():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        lib.or_norm_one.restype = C.c_double
        lib.or_norm_one.argtypes = [C.c_int64, P, P, P]
        lib.or_norm_fro.restype = C.c_double
        lib.or_norm_fro.argtypes = [C.c_int64, P, P, P]
        lib.or_norm_fro_I_plus.restype = C.c_double
        lib.or_norm_fro_I_plus.argtypes = [C.c_int64, P, P, P]
        lib.or_bandwidth.argtypes = [C.c_int64, P, P, P, P]
        lib.or_r0_d.restype = C.c_double
        lib.or_r0_d.argtypes = [C.c_double, C.c_int]
        lib.or_plan.restype = C.c_int
        lib.or_plan.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, P, P]
        lib.or_alg41.restype = C.c_int
        lib.or_alg41.argtypes = [C.c_int64, P, C.c_double, C.c_double, P, P, P, P, C.c_int]
        lib.or_expm.restype = P
        lib.or_expm.argtypes = [C.c_int64, P, P, P, C.c_double, C.POINTER(_Options)]
        lib.or_spgemm.restype = P
        lib.or_spgemm.argtypes = [C.c_int64, P, P, P, P, P, P, C.c_double, C.c_double, C.c_int]
        lib.or_add.restype = P
        lib.or_add.argtypes = [C.c_int64, P, P, P, P, P, P]
        lib.or_spmm.restype = C.c_int
        lib.or_rcm.restype = C.c_int
        lib.or_rcm.argtypes = [C.c_int64, P, P, P]
        lib.or_spmm.argtypes = [C.c_int64, P, P, P, C.c_int64, P, P, C.c_int]
        lib.or_result_nnz.restype = C.c_int64
        lib.or_result_nnz.argtypes = [P]
        lib.or_result_n.restype = C.c_int64
        lib.or_result_n.argtypes = [P]
        lib.or_result_copy.argtypes = [P, P, P, P]
        lib.or_result_trace.restype = C.POINTER(_Trace)
        lib.or_result_trace.argtypes = [P]
        lib.or_result_free.argtypes = [P]
        lib.or_trace_size.restype = C.c_int
        lib.or_options_size.restype = C.c_int
        assert lib.or_trace_size() == C.sizeof(_Trace), "trace struct layout mismatch"
        assert lib.or_options_size() == C.sizeof(_Options), "options struct layout mismatch"
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _csr_args(H: CSR):
    rp = np.ascontiguousarray(H.rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(H.col, dtype=np.int32)
    v = np.ascontiguousarray(H.val, dtype=np.float64)
    return rp, ci, v


def _take_result(R) -> CSR:
    lib = _L()
    n = lib.or_result_n(R)
    nnz = lib.or_result_nnz(R)
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(max(nnz, 1), np.int32)
    v = np.zeros(max(nnz, 1), np.float64)
    lib.or_result_copy(R, _p(rp), _p(ci), _p(v))
    return CSR(int(n), rp, ci[:nnz].copy(), v[:nnz].copy())


def r0(x: float, M: int) -> float:
    """Eq. (4.5): (1/M!) sum_i x^{M+1+i}/(i!(i+M+1)) (long double, returned as double)."""
    return _L().or_r0_d(float(x), int(M))


def plan(norm: float, eps_tol: float, m_cap: int = 120, n_window: int = 50):
    """Eq. (4.20) enumeration -> (M, N); raises on infeasible."""
    M = C.c_int()
    N = C.c_int()
    if _L().or_plan(float(norm), float(eps_tol), m_cap, n_window, C.byref(M), C.byref(N)):
        raise ValueError("infeasible plan")
    return M.value, N.value


def alg41(x: np.ndarray, eps_g: float, e_r: float = 0.1):
    """Algorithm 4.1 -> (keep mask, tau_final, passes, dropped_norm, tau history)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    keep = np.zeros(max(len(x), 1), np.uint8)
    tau = C.c_double()
    dropped = C.c_double()
    hist = np.zeros(256, np.float64)
    passes = _L().or_alg41(len(x), _p(x), float(eps_g), float(e_r), _p(keep), C.byref(tau),
                           C.byref(dropped), _p(hist), 256)
    return keep[:len(x)].astype(bool), tau.value, passes, dropped.value, hist[:min(passes, 256)].copy()


def _trace_dict(t: _Trace) -> dict:
    d = {k: getattr(t, k) for k in ("status", "M", "N", "M_eff", "normal", "norm", "a", "r0", "eps_g0")}
    for k, _ in _Trace._fields_:
        if k not in d:
            d[k] = np.array(getattr(t, k)[:])
    return d


def expm(H: CSR, eps_tol: float = 1e-16, opts: Options | None = None, **kw):
    """Algorithm 4.2 -> (CSR of E = I + T^_N (or T^_N), trace dict)."""
    if opts is None:
        opts = Options(**kw)
    lib = _L()
    rp, ci, v = _csr_args(H)
    co = opts.to_c()
    R = lib.or_expm(H.n, _p(rp), _p(ci), _p(v), float(eps_tol), C.byref(co))
    try:
        tr = _trace_dict(lib.or_result_trace(R).contents)
        out = _take_result(R)
    finally:
        lib.or_result_free(R)
    if tr["status"] != 0:
        raise ValueError(f"oracle status {tr['status']}")
    return out, tr


def spgemm(A: CSR, B: CSR, self_coef: float = 0.0, divisor: float = 1.0, nthreads: int = 1) -> CSR:
    lib = _L()
    a = _csr_args(A)
    b = _csr_args(B)
    R = lib.or_spgemm(A.n, *map(_p, a), *map(_p, b), float(self_coef), float(divisor), nthreads)
    try:
        return _take_result(R)
    finally:
        lib.or_result_free(R)


def add(A: CSR, B: CSR) -> CSR:
    lib = _L()
    R = lib.or_add(A.n, *map(_p, _csr_args(A)), *map(_p, _csr_args(B)))
    try:
        return _take_result(R)
    finally:
        lib.or_result_free(R)


def spmm(A: CSR, X: np.ndarray, steps: int = 1) -> np.ndarray:
    """N1 apply: Y = A^steps X for a dense X (n x m or n), row order of or_spmm."""
    lib = _L()
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    X2 = np.ascontiguousarray(X.reshape(A.n, -1))
    Y = np.zeros_like(X2)
    rc = lib.or_spmm(A.n, *map(_p, _csr_args(A)), X2.shape[1], _p(X2), _p(Y), int(steps))
    if rc != 0:
        raise ValueError(f"or_spmm status {rc}")
    return Y.reshape(-1) if vec else Y


def rcm(H: CSR) -> np.ndarray:
    """N3: reverse Cuthill-McKee permutation of pattern(H + H^T) (perm[new] = old), the
    deterministic rules of or_rcm."""
    rp, ci, _ = _csr_args(H)
    perm = np.zeros(max(H.n, 1), np.int64)
    _L().or_rcm(H.n, _p(rp), _p(ci), _p(perm))
    return perm[:H.n]


def norm_one(H: CSR) -> float:
    return _L().or_norm_one(H.n, *map(_p, _csr_args(H)))


def norm_fro(H: CSR) -> float:
    return _L().or_norm_fro(H.n, *map(_p, _csr_args(H)))


def norm_fro_I_plus(T: CSR) -> float:
    return _L().or_norm_fro_I_plus(T.n, *map(_p, _csr_args(T)))


def bandwidth(H: CSR):
    l1 = C.c_int64()
    l2 = C.c_int64()
    rp, ci, _ = _csr_args(H)
    _L().or_bandwidth(H.n, _p(rp), _p(ci), C.byref(l1), C.byref(l2))
    return l1.value, l2.value
