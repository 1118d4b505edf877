"""World-size-2 (gloo, CPU) test of the row-partitioned squaring protocol the library runs
over NCCL: contiguous row blocks (`sexpm_partition_rows`), halo rows of
T^_{i-1} within its bandwidth (`sexpm_halo_ranges`, Lemma 3.1) exchanged with
point-to-point sends, every Algorithm 4.1 scalar (pass sums) gathered and summed in rank
order.  Each rank computes its rows with the oracle's product on (local + halo) rows; the
concatenated result must equal the single-process oracle squaring (kept sets identical up
to entries within rounding of tau)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2110_04493_b200 import binding as B
from synth import CSR, laplacian_2d, random_banded

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rows_as_full(T: CSR, r0: int, r1: int) -> CSR:
    """n x n CSR holding only rows [r0, r1) of T (others empty)."""
    rp = np.zeros(T.n + 1, np.int64)
    cnt = np.diff(T.rowptr)[r0:r1]
    rp[r0 + 1:r1 + 1] = np.cumsum(cnt)
    rp[r1 + 1:] = rp[r1]
    a, b = T.rowptr[r0], T.rowptr[r1]
    return CSR(T.n, rp, T.col[a:b].copy(), T.val[a:b].copy())


def _send_rows(T: CSR, lo: int, hi: int, dst: int):
    a, b = int(T.rowptr[lo]), int(T.rowptr[hi])
    meta = torch.tensor([lo, hi, b - a], dtype=torch.int64)
    dist.send(meta, dst)
    dist.send(torch.from_numpy(np.diff(T.rowptr[lo:hi + 1]).astype(np.int64)), dst)
    if b > a:
        dist.send(torch.from_numpy(T.col[a:b].astype(np.int64)), dst)
        dist.send(torch.from_numpy(T.val[a:b].copy()), dst)


def _recv_rows(src: int):
    meta = torch.zeros(3, dtype=torch.int64)
    dist.recv(meta, src)
    lo, hi, nnz = (int(x) for x in meta)
    cnt = torch.zeros(hi - lo, dtype=torch.int64)
    dist.recv(cnt, src)
    col = torch.zeros(nnz, dtype=torch.int64)
    val = torch.zeros(nnz, dtype=torch.float64)
    if nnz:
        dist.recv(col, src)
        dist.recv(val, src)
    return lo, hi, cnt.numpy(), col.numpy().astype(np.int32), val.numpy()


def _allsum(x: float) -> float:
    t = [None] * WORLD
    dist.all_gather_object(t, float(x))
    s = 0.0
    for v in t:  # rank order, identical on every rank
        s += v
    return s


def _worker(rank, port, T_full_parts, eps_g, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    rp, ci, va, n = T_full_parts
    T = CSR(n, rp, ci, va)
    bounds = B.sexpm_partition_rows(n, np.diff(rp).astype(np.float64) ** 2, WORLD)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    l1, l2 = O.bandwidth(T)
    lo_h, hi_h = B.sexpm_halo_ranges(WORLD, rank, bounds, n, l1, l2)
    # what each peer needs from me
    for h in range(WORLD):
        if h == rank:
            continue
        plo, phi = B.sexpm_halo_ranges(WORLD, h, bounds, n, l1, l2)
        # ordered exchange: lower rank sends first
        if rank < h:
            _send_rows(T, int(plo[rank]), int(phi[rank]), h)
            got = _recv_rows(h)
        else:
            got = _recv_rows(h)
            _send_rows(T, int(plo[rank]), int(phi[rank]), h)
        assert (got[0], got[1]) == (int(lo_h[h]), int(hi_h[h]))
    # B = local rows + halo rows only (everything else empty): Lemma 3.1 says enough
    need_lo, need_hi = max(0, r0 - l2), min(n, r1 + l1)
    Bm = _rows_as_full(T, need_lo, need_hi)
    A = _rows_as_full(T, r0, r1)
    Ct = O.spgemm(A, Bm, 2.0, 1.0)
    # Algorithm 4.1 with rank-order scalar sums (R1: m0 = 1, first pass unconditional)
    vals = Ct.val
    m, tau, passes = 1.0, float("inf"), 0
    while True:
        tau = eps_g / m
        s = _allsum(float(np.sum(vals[np.abs(vals) <= tau] ** 2)))
        b = np.sqrt(s)
        m = b / tau
        passes += 1
        if b <= eps_g * 1.1:
            break
    keep = np.abs(vals) > tau
    rows = np.repeat(np.arange(n), np.diff(Ct.rowptr))[keep]
    result_q.put((rank, rows, Ct.col[keep], vals[keep], tau, passes))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["heat2d", "banded"])
def test_two_rank_squaring_matches_single_process(case):
    B.lib()
    if case == "heat2d":
        H = laplacian_2d(18, 17, 0.8, "pm10", seed=4)
        T = O.spgemm(H, H, 1.0, 2.0)  # a banded iterate with the heat structure
    else:
        T = random_banded(240, 6, 0.5, 0.3, seed=8)
    eps_g = 1e-3 * O.norm_fro_I_plus(T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, (T.rowptr, T.col, T.val, T.n), eps_g, q))
             for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(WORLD)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: oracle product + oracle Algorithm 4.1
    Ct = O.spgemm(T, T, 2.0, 1.0)
    keep, tau, passes, _, _ = O.alg41(Ct.val, eps_g, 0.1)
    assert res[0][5] == res[1][5] == passes
    assert res[0][4] == pytest.approx(tau, rel=1e-12)
    rows_ref = np.repeat(np.arange(T.n), np.diff(Ct.rowptr))[keep]
    rows = np.concatenate([r[1] for r in res])
    cols = np.concatenate([r[2] for r in res])
    vals = np.concatenate([r[3] for r in res])
    assert np.array_equal(rows, rows_ref)
    assert np.array_equal(cols, Ct.col[keep])
    assert np.array_equal(vals, Ct.val[keep])
