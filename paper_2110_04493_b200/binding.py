"""ctypes binding of libsexpm (include/sexpm.h).  Argument marshalling only: every
step of the method runs in the library's sm_100a kernels.  PyTorch provides device
memory and streams.  There is no CPU fallback: if libsexpm.so is missing this module
raises on import of the library.

The functions keep the C names (sexpm_plan, sexpm_run, sexpm_stats_get, ...); the
`Plan` class and `expm` are thin conveniences over them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libsexpm.so")
MAXSTEP = 160

SEXPM_STATUS = {0: "OK", 1: "EINVAL", 2: "ENONFINITE", 3: "ETOL", 4: "EINFEASIBLE", 5: "ENOMEM",
                6: "ECUDA", 7: "ENCCL", 8: "ESTATE", 9: "EINTERNAL"}

EXPORTED = [
    "sexpm_options_init", "sexpm_nccl_unique_id", "sexpm_nccl_comm_init",
    "sexpm_nccl_comm_destroy", "sexpm_plan", "sexpm_plan_host", "sexpm_run",
    "sexpm_result_copy", "sexpm_stats_get", "sexpm_destroy", "sexpm_last_error",
    "sexpm_filtered_product", "sexpm_alg41", "sexpm_halo_ranges", "sexpm_partition_rows",
    "sexpm_abi_sizes", "sexpm_kernel_launches", "sexpm_release_cache", "sexpm_apply",
    "sexpm_spmm", "sexpm_rcm", "sexpm_plan_scalars", "sexpm_fp64_peak", "sexpm_virtual_comm_create",
    "sexpm_result_copy_async", "sexpm_result_wait",
]


class SexpmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"sexpm {SEXPM_STATUS.get(code, code)}: {msg}")
        self.code = code


class CsrIn(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("nnz", C.c_int64), ("rowptr", C.c_void_p), ("colidx", C.c_void_p),
                ("vals", C.c_void_p)]


class CsrOut(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("nnz", C.c_int64), ("rowptr", C.c_void_p), ("colidx", C.c_void_p),
                ("vals", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("plan_norm", C.c_int32), ("normal", C.c_int32),
                ("threshold_mode", C.c_int32), ("filter", C.c_int32), ("m_cap", C.c_int32),
                ("n_window", C.c_int32), ("force_M", C.c_int32), ("force_N", C.c_int32),
                ("output_T", C.c_int32), ("window_cols", C.c_int32), ("kernel", C.c_int32),
                ("ssat", C.c_int32), ("reorder", C.c_int32), ("sq_order", C.c_int32),
                ("exact_products", C.c_int32), ("sym_squaring", C.c_int32), ("e_r", C.c_double),
                ("stream", C.c_void_p), ("nccl_comm", C.c_void_p)]


_I64 = C.c_int64 * MAXSTEP
_I32 = C.c_int32 * MAXSTEP
_F64 = C.c_double * MAXSTEP


class Stats(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("M", C.c_int32), ("N", C.c_int32),
                ("M_eff", C.c_int32), ("normal", C.c_int32), ("world", C.c_int32),
                ("rank", C.c_int32),
                ("norm", C.c_double), ("a", C.c_double), ("r0", C.c_double), ("eps_g0", C.c_double),
                ("taylor_nnz_unf", _I64), ("taylor_nnz", _I64), ("taylor_passes", _I32),
                ("taylor_tau", _F64), ("taylor_ms", _F64), ("taylor_numeric_ms", _F64),
                ("taylor_numeric_bytes", _F64), ("taylor_fmas_i", _F64),
                ("sq_nnz_unf", _I64), ("sq_nnz", _I64), ("sq_staged", _I64), ("sq_passes", _I32),
                ("sq_eps_g", _F64), ("sq_tau", _F64), ("sq_normIT", _F64),
                ("sq_l1", _I64), ("sq_l2", _I64), ("sq_fmas", _F64), ("sq_ms", _F64),
                ("sq_numeric_ms", _F64), ("sq_bytes", _F64), ("sq_numeric_bytes", _F64),
                ("ms_plan", C.c_double), ("ms_taylor", C.c_double), ("ms_squaring", C.c_double),
                ("ms_finalize", C.c_double), ("ms_total", C.c_double),
                ("taylor_bytes", C.c_double), ("taylor_fmas", C.c_double),
                ("nnz_out", C.c_int64), ("gpu_launches", C.c_int32), ("retries", C.c_int32),
                ("taylor_fallback_rows", _I64), ("sq_fallback_rows", _I64), ("sq_first_ms", _F64), ("sq_kernel_ms", _F64), ("sq_bsr_blocks", _I64),
                ("sq_block_products", _F64),
                ("cache_hits", C.c_int64), ("cache_misses", C.c_int64),
                ("cache_releases", C.c_int64), ("cache_bytes_cached", C.c_double),
                ("cache_bytes_allocated", C.c_double), ("sq_order_used", C.c_int32),
                ("sq_exchange_ms", _F64), ("ms_order_host", C.c_double), ("ms_order_wait", C.c_double),
                ("taylor_window", C.c_int32), ("sq_sym_used", C.c_int32),
                ("sq_assemble_ms", _F64)]


_lib = None


def lib():
    """Load libsexpm.so (in-tree build).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2110_04493_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.sexpm_last_error.restype = C.c_char_p
        L.sexpm_options_init.argtypes = [C.POINTER(Options)]
        L.sexpm_nccl_unique_id.argtypes = [P]
        L.sexpm_nccl_comm_init.argtypes = [C.c_int, C.c_int, P, C.POINTER(C.c_void_p)]
        L.sexpm_nccl_comm_destroy.argtypes = [P]
        L.sexpm_plan.argtypes = [C.POINTER(CsrIn), C.c_double, C.POINTER(Options), C.POINTER(C.c_void_p)]
        L.sexpm_plan_host.argtypes = L.sexpm_plan.argtypes
        L.sexpm_run.argtypes = [P, C.POINTER(CsrOut)]
        L.sexpm_result_copy.argtypes = [P, P, P, P]
        L.sexpm_result_copy_async.argtypes = [P, P, P, P, C.POINTER(C.c_void_p)]
        L.sexpm_result_wait.argtypes = [P]
        L.sexpm_stats_get.argtypes = [P, C.POINTER(Stats)]
        L.sexpm_destroy.argtypes = [P]
        L.sexpm_filtered_product.argtypes = [P, C.POINTER(CsrIn), C.POINTER(CsrIn), C.c_double,
                                             C.c_double, C.c_double, C.POINTER(CsrOut),
                                             C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                             C.POINTER(C.c_int64)]
        L.sexpm_alg41.argtypes = [P, P, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.sexpm_halo_ranges.argtypes = [C.c_int, C.c_int, P, C.c_int64, C.c_int64, C.c_int64, P, P]
        L.sexpm_partition_rows.argtypes = [C.c_int64, P, C.c_int, P]
        L.sexpm_plan_scalars.argtypes = [C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, P, P, P,
                                         P, P]
        L.sexpm_abi_sizes.argtypes = [P]
        L.sexpm_kernel_launches.argtypes = [P]
        L.sexpm_fp64_peak.argtypes = [P, P]
        L.sexpm_virtual_comm_create.argtypes = [C.c_int, P]
        for f in EXPORTED:
            if f != "sexpm_last_error":
                getattr(L, f).restype = C.c_int
        sizes = (C.c_uint32 * 4)()
        L.sexpm_abi_sizes(sizes)
        want = (C.sizeof(Options), C.sizeof(Stats), C.sizeof(CsrIn), C.sizeof(CsrOut))
        if tuple(sizes) != want:
            raise RuntimeError(f"libsexpm ABI mismatch: C sizes {tuple(sizes)} vs ctypes {want}")
        _lib = L
    return _lib


def _check(code: int):
    if code != 0:
        raise SexpmError(code, lib().sexpm_last_error().decode())


# ---------------------------------------------------------------------------------------
# C-named wrappers
# ---------------------------------------------------------------------------------------
def sexpm_options_init(**kw) -> Options:
    o = Options()
    _check(lib().sexpm_options_init(C.byref(o)))
    for k, v in kw.items():
        if k == "plan_norm" and isinstance(v, str):
            v = {"one": 0, "fro": 1}[v]
        if k == "threshold_mode" and isinstance(v, str):
            v = {"rel_prev": 0, "abs": 1}[v]
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, int(v) if isinstance(v, bool) else v)
    return o


def _csr_in(n, rowptr, col, val, row_begin=0, row_end=None, host=False) -> CsrIn:
    rows = (len(rowptr) if host else rowptr.numel()) - 1
    if row_end is None:
        row_end = row_begin + rows
    ptr = (lambda a: a.ctypes.data) if host else (lambda t: t.data_ptr())
    nnz = int(rowptr[-1]) if rows >= 0 else 0
    return CsrIn(int(n), int(row_begin), int(row_end), nnz, ptr(rowptr), ptr(col), ptr(val))


def sexpm_plan(H: CsrIn, eps_tol: float, opts: Options):
    h = C.c_void_p()
    _check(lib().sexpm_plan(C.byref(H), float(eps_tol), C.byref(opts), C.byref(h)))
    return h


def sexpm_plan_host(H: CsrIn, eps_tol: float, opts: Options):
    h = C.c_void_p()
    _check(lib().sexpm_plan_host(C.byref(H), float(eps_tol), C.byref(opts), C.byref(h)))
    return h


def sexpm_run(h) -> CsrOut:
    out = CsrOut()
    _check(lib().sexpm_run(h, C.byref(out)))
    return out


def sexpm_result_copy(h, rowptr_ptr: int, col_ptr: int, val_ptr: int):
    _check(lib().sexpm_result_copy(h, C.c_void_p(rowptr_ptr), C.c_void_p(col_ptr), C.c_void_p(val_ptr)))


def sexpm_result_copy_async(h, rowptr_ptr: int, col_ptr: int, val_ptr: int):
    """Detaches the result and starts its copy; returns the ticket for sexpm_result_wait."""
    t = C.c_void_p()
    _check(lib().sexpm_result_copy_async(h, C.c_void_p(rowptr_ptr), C.c_void_p(col_ptr),
                                         C.c_void_p(val_ptr), C.byref(t)))
    return t


def sexpm_result_wait(ticket):
    _check(lib().sexpm_result_wait(ticket))


def sexpm_stats_get(h) -> dict:
    s = Stats()
    s.struct_size = C.sizeof(Stats)
    _check(lib().sexpm_stats_get(h, C.byref(s)))
    d = {}
    for k, _ in Stats._fields_:
        v = getattr(s, k)
        d[k] = np.ctypeslib.as_array(v).copy() if hasattr(v, "_length_") else v
    return d


def sexpm_virtual_comm_create(world: int) -> list:
    """`world` communicator handles of virtual ranks (one process, one GPU, one host thread
    per rank): pass handle r as nccl_comm of rank r's Plan."""
    arr = (C.c_void_p * world)()
    _check(lib().sexpm_virtual_comm_create(int(world), arr))
    return [arr[i] for i in range(world)]


def sexpm_fp64_peak() -> dict:
    """Measured fp64 throughput of the current device: DFMA and DMMA TF/s."""
    a, b = C.c_double(), C.c_double()
    _check(lib().sexpm_fp64_peak(C.byref(a), C.byref(b)))
    return {"dfma_tflops": a.value, "dmma_tflops": b.value}


def sexpm_kernel_launches() -> int:
    c = C.c_int64()
    _check(lib().sexpm_kernel_launches(C.byref(c)))
    return c.value


def sexpm_destroy(h):
    if h:
        _check(lib().sexpm_destroy(h))


def sexpm_release_cache():
    _check(lib().sexpm_release_cache())


def sexpm_nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().sexpm_nccl_unique_id(buf))
    return bytes(buf)


def sexpm_nccl_comm_init(rank: int, world: int, uid: bytes):
    buf = (C.c_char * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    _check(lib().sexpm_nccl_comm_init(rank, world, buf, C.byref(comm)))
    return comm


def sexpm_nccl_comm_destroy(comm):
    _check(lib().sexpm_nccl_comm_destroy(comm))


def sexpm_halo_ranges(world: int, rank: int, bounds, n: int, l1: int, l2: int):
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    lo = np.zeros(world, np.int64)
    hi = np.zeros(world, np.int64)
    _check(lib().sexpm_halo_ranges(world, rank, b.ctypes.data, n, l1, l2, lo.ctypes.data,
                                   hi.ctypes.data))
    return lo, hi


def sexpm_plan_scalars(norm: float, normal: int, eps_tol: float, m_cap: int = 120,
                       n_window: int = 50) -> dict:
    """Algorithm 4.2 steps 1-3 for a given plan norm (host only): M, N, a, r0, eps_g0."""
    M, N = C.c_int32(), C.c_int32()
    a, r0, e0 = C.c_double(), C.c_double(), C.c_double()
    _check(lib().sexpm_plan_scalars(float(norm), int(normal), float(eps_tol), int(m_cap),
                                    int(n_window), C.addressof(M), C.addressof(N), C.addressof(a),
                                    C.addressof(r0), C.addressof(e0)))
    return {"M": M.value, "N": N.value, "a": a.value, "r0": r0.value, "eps_g0": e0.value}


def sexpm_partition_rows(n: int, work, world: int):
    w = None if work is None else np.ascontiguousarray(work, dtype=np.float64)
    b = np.zeros(world + 1, np.int64)
    _check(lib().sexpm_partition_rows(n, None if w is None else w.ctypes.data, world, b.ctypes.data))
    return b


# ---------------------------------------------------------------------------------------
# torch conveniences
# ---------------------------------------------------------------------------------------
def _torch():
    import torch
    return torch


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the handle that names the legacy default stream


def stream_handle(stream) -> int:
    """cudaStream_t of a torch stream for sexpm_options.stream.  torch's default stream is the
    legacy default stream, whose handle 0 would read as "NULL = a stream created by the plan":
    pass cudaStreamLegacy instead, so the plan runs on the caller's stream."""
    h = int(stream.cuda_stream)
    return h if h != 0 else CUDA_STREAM_LEGACY


class Plan:
    """One e^H computation (Algorithm 4.2) bound to the current CUDA device and stream."""

    def __init__(self, n, rowptr, col, val, eps_tol=1e-16, row_begin=0, row_end=None,
                 nccl_comm=None, stream=None, **opts):
        torch = _torch()
        self._keep = (rowptr, col, val)
        if stream is None:
            stream = torch.cuda.current_stream()
        o = sexpm_options_init(**opts)
        o.stream = stream_handle(stream)
        if nccl_comm is not None:
            o.nccl_comm = nccl_comm
        self.n = int(n)
        H = _csr_in(n, rowptr, col, val, row_begin, row_end)
        self.h = sexpm_plan(H, eps_tol, o)
        self._keep = None

    def run(self):
        """Run and return (rowptr, col, val) device tensors of this rank's rows of E."""
        torch = _torch()
        out = sexpm_run(self.h)
        rows = out.row_end - out.row_begin
        dev = torch.device("cuda", torch.cuda.current_device())
        rp = torch.empty(rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(max(out.nnz, 1), dtype=torch.int32, device=dev)
        va = torch.empty(max(out.nnz, 1), dtype=torch.float64, device=dev)
        sexpm_result_copy(self.h, rp.data_ptr(), ci.data_ptr(), va.data_ptr())
        return rp, ci[:out.nnz], va[:out.nnz]

    def run_only(self) -> CsrOut:
        return sexpm_run(self.h)

    def apply(self, X, steps: int = 1, Y=None):
        """Y = R^steps X on the device (R = the last result, E by default): X a float64 CUDA
        tensor of shape (n, m) (or (n,)), row stride >= m.  Returns Y (new tensor unless
        given)."""
        return sexpm_apply(self.h, X, steps, Y)

    def stats(self) -> dict:
        return sexpm_stats_get(self.h)

    def close(self):
        if self.h:
            sexpm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def expm(n, rowptr, col, val, eps_tol=1e-16, **opts):
    """e^H for a device CSR (torch tensors int64 / int32 / float64 on CUDA)."""
    p = Plan(n, rowptr, col, val, eps_tol, **opts)
    try:
        E = p.run()
        return E, p.stats()
    finally:
        p.close()


def expm_host(n, rowptr: np.ndarray, col: np.ndarray, val: np.ndarray, eps_tol=1e-16,
              out=None, **opts):
    """End-to-end through the C ABI with HOST buffers: H2D inside sexpm_plan_host, D2H of
    the result inside sexpm_result_copy.  Returns numpy arrays (or fills `out`)."""
    torch = _torch()
    o = sexpm_options_init(**opts)
    o.stream = stream_handle(torch.cuda.current_stream())
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    H = _csr_in(n, rowptr, col, val, host=True)
    h = sexpm_plan_host(H, eps_tol, o)
    try:
        E = sexpm_run(h)
        rows = E.row_end - E.row_begin
        if out is None:
            out = (np.empty(rows + 1, np.int64), np.empty(max(E.nnz, 1), np.int32),
                   np.empty(max(E.nnz, 1), np.float64))
        if out[0].size < rows + 1 or out[1].size < E.nnz or out[2].size < E.nnz:
            raise ValueError(f"output buffers too small for nnz(E) = {E.nnz}")
        sexpm_result_copy(h, out[0].ctypes.data, out[1].ctypes.data, out[2].ctypes.data)
        st = sexpm_stats_get(h)
        return (out[0], out[1][:E.nnz], out[2][:E.nnz]), st
    finally:
        sexpm_destroy(h)


_ctx = None
_ctx_kernel = {}


def _context(kernel=0):
    """A plan on a 1x1 zero matrix: the device/stream context of the component entry points
    (one per accumulator choice `kernel`, see sexpm_options.kernel)."""
    global _ctx
    torch = _torch()
    if kernel == 0 and _ctx is not None:
        return _ctx
    if kernel in _ctx_kernel:
        return _ctx_kernel[kernel]
    dev = torch.device("cuda", torch.cuda.current_device())
    rp = torch.zeros(2, dtype=torch.int64, device=dev)
    ci = torch.zeros(1, dtype=torch.int32, device=dev)
    va = torch.zeros(1, dtype=torch.float64, device=dev)
    o = sexpm_options_init(kernel=kernel)
    o.stream = stream_handle(torch.cuda.current_stream())
    h = sexpm_plan(_csr_in(1, rp, ci, va), 1e-16, o)
    if kernel == 0:
        _ctx = h
    else:
        _ctx_kernel[kernel] = h
    return h


def sexpm_filtered_product(n, A, B, self_coef, divisor, eps_g, kernel=0, a_row0=0, b_row0=0):
    """One filtered product (K1-K4) on the GPU. A, B = (rowptr, col, val) device tensors of
    rows [a_row0, ...) and [b_row0, ...) of n x n matrices (B must hold every row A's columns
    reach).  Returns ((rowptr, col, val) tensors of A's rows, passes, tau, nnz_unf)."""
    torch = _torch()
    h = _context(kernel)
    Ai = _csr_in(n, *A, row_begin=a_row0)
    Bi = _csr_in(n, *B, row_begin=b_row0)
    out = CsrOut()
    passes = C.c_int32()
    tau = C.c_double()
    nu = C.c_int64()
    _check(lib().sexpm_filtered_product(h, C.byref(Ai), C.byref(Bi), float(self_coef),
                                        float(divisor), float(eps_g), C.byref(out),
                                        C.byref(passes), C.byref(tau), C.byref(nu)))
    dev = A[0].device
    rows = out.row_end - out.row_begin
    rp = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(out.nnz, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(out.nnz, 1), dtype=torch.float64, device=dev)
    sexpm_result_copy(h, rp.data_ptr(), ci.data_ptr(), va.data_ptr())
    return (rp, ci[:out.nnz], va[:out.nnz]), passes.value, tau.value, nu.value


def _dense2(X):
    if X.dim() == 1:
        return X.view(-1, 1)
    return X


def sexpm_apply(h, X, steps: int = 1, Y=None):
    """Y = R^steps X (sexpm_apply); X, Y float64 CUDA tensors (n, m), rows contiguous."""
    torch = _torch()
    X2 = _dense2(X)
    if X2.dtype != torch.float64 or X2.stride(1) != 1:
        raise ValueError("X must be float64 with contiguous rows")
    if Y is None:
        Y = torch.empty_like(X2, memory_format=torch.contiguous_format)
    Y2 = _dense2(Y)
    _check(lib().sexpm_apply(h, C.c_int64(X2.shape[1]), C.c_void_p(X2.data_ptr()),
                             C.c_int64(X2.stride(0)), C.c_void_p(Y2.data_ptr()),
                             C.c_int64(Y2.stride(0)), C.c_int32(int(steps))))
    return Y.view(X.shape) if X.dim() == 1 else Y


def sexpm_spmm(n, A, X, Y=None, kernel=0):
    """Y = A X for a device CSR A = (rowptr, col, val) of an n x n matrix and a float64 CUDA
    tensor X (n, m) (the kernel of sexpm_apply)."""
    torch = _torch()
    h = _context(kernel)
    Ai = _csr_in(n, *A)
    X2 = _dense2(X)
    if X2.dtype != torch.float64 or X2.stride(1) != 1:
        raise ValueError("X must be float64 with contiguous rows")
    rows = A[0].numel() - 1
    if Y is None:
        Y = torch.empty((rows, X2.shape[1]), dtype=torch.float64, device=X2.device)
    Y2 = _dense2(Y)
    _check(lib().sexpm_spmm(h, C.byref(Ai), C.c_int64(X2.shape[1]), C.c_void_p(X2.data_ptr()),
                            C.c_int64(X2.stride(0)), C.c_void_p(Y2.data_ptr()),
                            C.c_int64(Y2.stride(0))))
    return Y.view(-1) if X.dim() == 1 else Y


def sexpm_rcm(n, A):
    """Reverse Cuthill-McKee permutation (perm[new] = old) of a device CSR (all n rows)."""
    torch = _torch()
    h = _context()
    Ai = _csr_in(n, *A)
    perm = torch.empty(max(int(n), 1), dtype=torch.int64, device=A[0].device)
    _check(lib().sexpm_rcm(h, C.byref(Ai), C.c_void_p(perm.data_ptr())))
    return perm[:int(n)]


def sexpm_alg41(x, eps_g: float, e_r: float = 0.1):
    """Algorithm 4.1 over a device float64 tensor -> (passes, tau, dropped)."""
    h = _context()
    passes = C.c_int32()
    tau = C.c_double()
    dropped = C.c_double()
    _check(lib().sexpm_alg41(h, C.c_void_p(x.data_ptr()), x.numel(), float(eps_g), float(e_r),
                             C.byref(passes), C.byref(tau), C.byref(dropped)))
    return passes.value, tau.value, dropped.value
