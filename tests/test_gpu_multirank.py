"""The row-partitioned multi-rank path (Lemma 3.1's halo)
executed on ONE GPU with virtual ranks: W plans in one process, one host thread and one CUDA
stream per rank, connected by sexpm_virtual_comm_create (every collective = host barrier +
device-to-device copies; no kernel waits on another rank).  Runs the all-gather of H, the
scalar all-gathers of every Algorithm 4.1 pass (rank-order sums), the halo exchange of every
squaring and the block kernels on the halo slices -- the same driver code NCCL drives on
several GPUs -- and compares the assembled E with the oracle (north-star parity) and with the
single-rank run."""
import threading

import numpy as np
import pytest

import oracle as O
from synth import CSR, laplacian_2d, make_config, random_banded, structural_state_space

from gpu_helpers import NTHREADS, from_dev, last_tau, parity, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_04493_b200 import binding
    from paper_2110_04493_b200.build import build
    build()
    binding.lib()
    return binding


def run_ranks(B, H, bounds, eps_tol=1e-16, **opts):
    """E assembled from W virtual ranks' row blocks, plus every rank's stats."""
    import torch
    W = len(bounds) - 1
    comms = B.sexpm_virtual_comm_create(W)
    out = [None] * W
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            Hl = H.rows(r0, r1)
            with torch.cuda.stream(s):
                rp, ci, va = to_dev(Hl)
                s.synchronize()
                p = B.Plan(H.n, rp, ci, va, eps_tol, row_begin=r0, row_end=r1,
                           nccl_comm=comms[r], stream=s, **opts)
                E = p.run()
                s.synchronize()
                st = p.stats()
                p.close()
            out[r] = ([x.cpu().numpy() for x in E], st)
        except Exception as e:  # surface the failing rank's error
            errs.append((r, repr(e)))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in comms:
        B.sexpm_nccl_comm_destroy(c)
    assert not errs, errs
    rps, cols, vals = [], [], []
    off = 0
    for r in range(W):
        (rp, ci, va), _ = out[r]
        rps.append(rp[:-1] + off if r < W - 1 else rp + off)
        off += int(rp[-1])
        cols.append(ci)
        vals.append(va)
    E = CSR(H.n, np.concatenate(rps).astype(np.int64), np.concatenate(cols).astype(np.int32),
            np.concatenate(vals).astype(np.float64))
    return E, [o[1] for o in out]


CASES = {
    "heat2d_40": lambda: laplacian_2d(40, 40, 1.0, "pm10", seed=7),
    "config5_law_48": lambda: make_config(5, scale_down=48),
    "structural_20": lambda: structural_state_space(20, 20, 0.5, seed=8),
    "banded_nonsym": lambda: random_banded(900, 7, 0.5, 0.6, seed=9),
    "heat3d_10": lambda: make_config(4, scale_down=10),
}


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_virtual_ranks_match_oracle(B, W, name):
    H = CASES[name]()
    bounds = B.sexpm_partition_rows(H.n, np.diff(H.rowptr).astype(np.float64) ** 2, W)
    Eg, sts = run_ranks(B, H, bounds)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    st = sts[0]
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    assert all(s["world"] == W and s["rank"] == r for r, s in enumerate(sts))
    # every rank took the same Algorithm 4.1 decisions (rank-order scalar sums)
    for s in sts[1:]:
        N = int(st["N"])
        assert np.array_equal(s["sq_passes"][:N + 1], st["sq_passes"][:N + 1])
        assert np.array_equal(s["sq_tau"][:N + 1], st["sq_tau"][:N + 1])
        assert np.array_equal(s["sq_nnz"][:N + 1], st["sq_nnz"][:N + 1])
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    if name != "banded_nonsym":  # stencil rows: every rank squares on the block kernel
        if name.startswith(("heat2d", "config5")):  # 2D: aggregates of each rank's own rows
            assert st["sq_order_used"] in (1, 2)
        for s in sts:
            assert s["sq_fallback_rows"][1:int(s["N"]) + 1].sum() == 0
            assert all(s["sq_bsr_blocks"][1:int(s["N"]) + 1] > 0)


@pytest.mark.parametrize("bounds", [[0, 333, 1000, 1600], [0, 801, 1600], [0, 8, 1592, 1600]])
def test_virtual_ranks_unaligned_bounds(B, bounds):
    """Rank bounds that are not multiples of 8 (the block kernel needs aligned halo slices:
    such ranks fall back to the paged kernel) and a 1-block rank: still parity."""
    H = laplacian_2d(40, 40, 1.0, "pm10", seed=7)
    Eg, sts = run_ranks(B, H, np.array(bounds, np.int64))
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    ok, res = parity(Eg, Eo, last_tau(tr, sts[0]))
    assert ok, res


def test_virtual_ranks_equal_single_rank(B):
    """W = 3 against the one-rank run of the same plan (sq_order = 0 so both square in index
    order): the same plan, pattern sizes within flips, parity between the two."""
    H = make_config(5, scale_down=40)
    bounds = B.sexpm_partition_rows(H.n, None, 3)
    Eg, sts = run_ranks(B, H, bounds, sq_order=0)
    E1, st1 = run_ranks(B, H, np.array([0, H.n], np.int64), sq_order=0)
    st = sts[0]
    assert (st["M"], st["N"]) == (st1[0]["M"], st1[0]["N"])
    ok, res = parity(Eg, E1, max(st["sq_tau"][st["N"]], st1[0]["sq_tau"][st["N"]], 1e-300))
    assert ok, res


@pytest.mark.parametrize("W,steps,m", [(2, 1, 1), (2, 3, 5), (3, 2, 33), (4, 1, 64)])
def test_virtual_ranks_apply(B, W, steps, m):
    """N1 apply on the row partition (Y = E^steps X, each rank its rows of X and Y; every step
    exchanges the X rows within E's bandwidth): equals the oracle's SpMM of the assembled E
    (P:501-503)."""
    import torch
    H = laplacian_2d(36, 30, 1.0, "pm10", seed=11)
    n = H.n
    bounds = B.sexpm_partition_rows(n, np.diff(H.rowptr).astype(np.float64) ** 2, W)
    X = np.random.default_rng(5).standard_normal((n, m))
    comms = B.sexpm_virtual_comm_create(W)
    outE, outY, errs = [None] * W, [None] * W, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            Hl = H.rows(r0, r1)
            with torch.cuda.stream(s):
                rp, ci, va = to_dev(Hl)
                Xl = torch.from_numpy(np.ascontiguousarray(X[r0:r1])).cuda()
                s.synchronize()
                p = B.Plan(n, rp, ci, va, 1e-16, row_begin=r0, row_end=r1, nccl_comm=comms[r], stream=s)
                E = p.run()
                Y = p.apply(Xl, steps=steps)
                s.synchronize()
                p.close()
            outE[r] = [x.cpu().numpy() for x in E]
            outY[r] = Y.cpu().numpy()
        except Exception as e:
            errs.append((r, repr(e)))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in comms:
        B.sexpm_nccl_comm_destroy(c)
    assert not errs, errs
    rps, cols, vals, off = [], [], [], 0
    for r in range(W):
        rp, ci, va = outE[r]
        rps.append(rp[:-1] + off if r < W - 1 else rp + off)
        off += int(rp[-1])
        cols.append(ci)
        vals.append(va)
    E = CSR(n, np.concatenate(rps).astype(np.int64), np.concatenate(cols).astype(np.int32),
            np.concatenate(vals).astype(np.float64))
    Yg = np.concatenate(outY, axis=0).reshape(n, m)
    Yo = O.spmm(E, X, steps=steps)
    scale = np.abs(Yo).max()
    assert np.abs(Yg - Yo).max() <= 1e-13 * steps * scale
