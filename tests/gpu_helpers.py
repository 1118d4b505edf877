"""Shared helpers of the GPU parity tests: CSR <-> torch, the BASELINE.json north-star
parity criteria, and the oracle runner (all cores, bit-identical to 1 thread)."""
from __future__ import annotations

import os

import numpy as np
import scipy.sparse as sp

from synth import CSR

NTHREADS = max(1, os.cpu_count() or 1)


def to_dev(H: CSR, device="cuda:0"):
    import torch
    return (torch.from_numpy(H.rowptr).to(device), torch.from_numpy(H.col).to(device),
            torch.from_numpy(H.val).to(device))


def from_dev(n, rp, ci, va) -> CSR:
    return CSR(int(n), rp.cpu().numpy().astype(np.int64), ci.cpu().numpy().astype(np.int32),
               va.cpu().numpy().astype(np.float64))


def scipy_of(H: CSR):
    rows = H.rowptr.shape[0] - 1
    return sp.csr_matrix((H.val, H.col, H.rowptr), shape=(rows, H.n))


def parity(E_gpu: CSR, E_or: CSR, tau: float, rel_tol: float = 1e-11):
    """BASELINE.json north star: max |E_gpu - E_or| <= 1e-11 max|E_or| over the union of
    positions; >= 99.9 % of positions shared; every position held by only one side has
    |value| < 10 tau (tau = final Algorithm 4.1 threshold of the last step)."""
    A = scipy_of(E_gpu)
    B = scipy_of(E_or)
    D = (A - B).tocsr()
    maxabs = np.abs(B.data).max() if B.nnz else 0.0
    err = np.abs(D.data).max() if D.nnz else 0.0
    PA = A.copy()
    PA.data[:] = 1.0
    PB = B.copy()
    PB.data[:] = 1.0
    inter = PA.multiply(PB).nnz
    union = (PA + PB).nnz
    jacc = inter / union if union else 1.0
    only = (PA - PB).tocsr()
    only.eliminate_zeros()
    r, c = only.nonzero()
    vals = np.concatenate([np.asarray(A[r, c]).ravel(), np.asarray(B[r, c]).ravel()]) if len(r) else np.zeros(0)
    symdiff_max = np.abs(vals).max() if len(vals) else 0.0
    res = dict(err=err, maxabs=maxabs, rel=err / maxabs if maxabs else err, jaccard=jacc,
               n_only=len(r), symdiff_max=symdiff_max, tau=tau)
    ok = (err <= rel_tol * maxabs) and (jacc >= 0.999) and (symdiff_max < 10 * tau or len(r) == 0)
    return ok, res


def last_tau(tr_or: dict, st_gpu: dict | None = None) -> float:
    """Final Algorithm 4.1 threshold of the last filtered step (larger of the two sides)."""
    N, M = tr_or["N"], tr_or["M"]
    vals = []
    if N > 0:
        vals.append(tr_or["sq_tau"][N])
        if st_gpu is not None:
            vals.append(st_gpu["sq_tau"][N])
    else:
        Me = max(tr_or["M_eff"], 2)
        vals += [t for t in tr_or["taylor_tau"][2:Me + 2] if np.isfinite(t)]
    vals = [v for v in vals if np.isfinite(v)]
    return max(vals) if vals else 0.0
