"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same seeded
inputs (BASELINE.json north-star criteria, see gpu_helpers.parity)."""
import numpy as np
import pytest

import oracle as O
from synth import (CSR, csr_to_dense, dense_to_csr, diagonal, laplacian_2d, make_config,
                   neumann_laplacian_2d, random_banded, random_skew, tridiag)

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


def run_gpu(B, H, eps_tol=1e-16, **opts):
    rp, ci, va = to_dev(H)
    (erp, eci, eva), st = B.expm(H.n, rp, ci, va, eps_tol, **opts)
    return from_dev(H.n, erp, eci, eva), st


def run_both(B, H, eps_tol=1e-16, **opts):
    Eg, st = run_gpu(B, H, eps_tol, **opts)
    oo = {k: v for k, v in opts.items() if k not in ("window_cols", "kernel", "exact_products")}
    Eo, tr = O.expm(H, eps_tol, nthreads=NTHREADS, **oo)
    return Eg, st, Eo, tr


def assert_plan_equal(st, tr):
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    assert st["normal"] == tr["normal"]
    assert st["norm"] == pytest.approx(tr["norm"], rel=1e-14)
    assert st["a"] == pytest.approx(tr["a"], rel=1e-15)
    assert st["eps_g0"] == pytest.approx(tr["eps_g0"], rel=1e-13, abs=0)


def assert_parity(Eg, st, Eo, tr):
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    return res


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_baseline_configs_one_norm(B, cid):
    H = make_config(cid)
    Eg, st, Eo, tr = run_both(B, H)
    assert_plan_equal(st, tr)
    assert_parity(Eg, st, Eo, tr)
    assert st["M_eff"] == tr["M_eff"]
    for i in range(1, tr["N"] + 1):  # per-squaring pattern sizes agree within flips
        assert abs(st["sq_nnz"][i] - tr["sq_nnz"][i]) <= 1e-3 * tr["sq_nnz"][i] + 2


@pytest.mark.parametrize("cid", [1, 2])
def test_baseline_configs_fro_norm(B, cid):
    H = make_config(cid)
    Eg, st, Eo, tr = run_both(B, H, plan_norm="fro")
    assert_plan_equal(st, tr)
    assert_parity(Eg, st, Eo, tr)


def test_paper_tables_2_3_on_gpu(B):
    """Tables 2-3 reproduced by the CUDA path itself."""
    H = tridiag(10_000, 1.0, -2.0, 1.0)
    Eg, st = run_gpu(B, H, plan_norm="fro")
    assert (st["M"], st["N"]) == (20, 8)
    lam = [int(st["sq_l1"][i] + st["sq_l2"][i]) for i in range(1, 9)]
    assert lam == [14, 16, 18, 20, 22, 26, 32, 38]
    assert st["M_eff"] == 9 and st["taylor_nnz"][10] == 0


SMALL = {
    "heat2d_pm10_20": lambda: make_config(2, scale_down=20),
    "structural_24": lambda: make_config(3, scale_down=24),
    "heat3d_9": lambda: make_config(4, scale_down=9),
    "heat2d_uniform_33": lambda: make_config(5, scale_down=33),
    "neumann_15x13": lambda: neumann_laplacian_2d(15, 13, 0.7, seed=3),
    "banded_nonsym": lambda: random_banded(150, 5, 0.6, 1.5, seed=21),
    "banded_sym": lambda: random_banded(170, 4, 0.7, 2.0, seed=22, symmetric=True),
    "skew": lambda: random_skew(120, 3, 0.7, 1.5, seed=23),
    "diagonal": lambda: diagonal(np.linspace(-3, 2.5, 37)),
    "n1": lambda: diagonal([0.75]),
    "tridiag_ragged_997": lambda: tridiag(997, 0.3, -0.9, 0.6),
}


@pytest.mark.parametrize("name", sorted(SMALL))
@pytest.mark.parametrize("tol", [1e-16, 1e-10])
def test_small_cases(B, name, tol):
    H = SMALL[name]()
    Eg, st, Eo, tr = run_both(B, H, tol)
    assert_plan_equal(st, tr)
    assert_parity(Eg, st, Eo, tr)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_table1_matrices(B, k):
    import refs
    A = refs.table1_matrices()[k]
    H = dense_to_csr(A)
    Eg, st, Eo, tr = run_both(B, H, plan_norm="fro")
    assert_plan_equal(st, tr)
    assert_parity(Eg, st, Eo, tr)
    Ex = refs.table1_exact(k)
    assert np.linalg.norm(csr_to_dense(Eg) - Ex) / np.linalg.norm(Ex) < 1e-13


@pytest.mark.parametrize("window", [32, 96, 1000])
def test_window_chunking_and_ragged_tail(B, window):
    """Force many accumulator chunks (and a ragged last chunk) per row."""
    H = make_config(2, scale_down=24)
    Eg, st, Eo, tr = run_both(B, H, window_cols=window)
    assert_parity(Eg, st, Eo, tr)


def test_zero_matrix_gives_identity(B):
    import scipy.sparse as sps
    n = 50
    H = dense_to_csr(np.zeros((n, n)))
    Eg, st = run_gpu(B, H)
    assert (st["M"], st["N"]) == (0, 0)
    assert np.array_equal(csr_to_dense(Eg), np.eye(n))


def test_unfiltered_matches_oracle(B):
    H = random_banded(90, 3, 0.8, 1.0, seed=31)
    Eg, st, Eo, tr = run_both(B, H, filter=False)
    assert_parity(Eg, st, Eo, tr)
    assert all(st["sq_passes"][: st["N"] + 1] == 0)


def test_abs_threshold_mode(B):
    H = make_config(2, scale_down=16)
    Eg, st, Eo, tr = run_both(B, H, threshold_mode="abs")
    assert_parity(Eg, st, Eo, tr)


def test_output_T(B):
    H = make_config(1, scale_down=200)
    Eg, st, Eo, tr = run_both(B, H, output_T=True)
    assert_parity(Eg, st, Eo, tr)


def test_errors(B):
    import torch
    H = tridiag(10, 1.0, -2.0, 1.0)
    rp, ci, va = to_dev(H)
    bad = va.clone()
    bad[3] = float("nan")
    with pytest.raises(B.SexpmError) as e:
        B.expm(H.n, rp, ci, bad)
    assert e.value.code == 2
    with pytest.raises(B.SexpmError) as e:
        B.expm(H.n, rp, ci, va, 1e-17)
    assert e.value.code == 3
    ci2 = ci.clone()
    ci2[1], ci2[2] = ci[2], ci[1]
    with pytest.raises(B.SexpmError) as e:
        B.expm(H.n, rp, ci2, va)
    assert e.value.code == 1


def test_explicit_zeros_ignored(B):
    H = tridiag(300, 0.4, -0.8, 0.4)
    Hz = tridiag(300, 0.4, -0.8, 0.4)
    Hz.val[::7] = 0.0  # explicit zeros in the input are ignored by the library
    Hc = dense_to_csr(csr_to_dense(Hz))
    rp, ci, va = to_dev(Hz)
    (a, b, c), st = B.expm(Hz.n, rp, ci, va)
    Eo, tr = O.expm(Hc, 1e-16)
    ok, res = parity(from_dev(Hz.n, a, b, c), Eo, last_tau(tr, st))
    assert ok, res


def test_host_entry_point_matches_device(B):
    H = make_config(2, scale_down=30)
    (hrp, hci, hva), st_h = B.expm_host(H.n, H.rowptr, H.col, H.val)
    Eg, st = run_gpu(B, H)
    Eh = type(Eg)(H.n, hrp, hci, hva)
    ok, res = parity(Eh, Eg, last_tau({"N": st["N"], "M": st["M"], "M_eff": st["M_eff"],
                                         "sq_tau": st["sq_tau"], "taylor_tau": st["taylor_tau"]}))
    assert ok, res


# ---------------------------- component entry points ----------------------------------

def _rand_csr(n, bw, dens, seed, empty_rows=()):
    A = csr_to_dense(random_banded(n, bw, dens, 1.0, seed))
    for r in empty_rows:
        A[r, :] = 0
    return dense_to_csr(A)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("self_coef,divisor", [(2.0, 1.0), (0.0, 3.0), (0.0, 1.0)])
def test_filtered_product_vs_oracle(B, seed, self_coef, divisor):
    n = 257
    A = _rand_csr(n, 6, 0.5, 100 + seed, empty_rows=(0, 5, 128, 256))
    Bm = A if self_coef else _rand_csr(n, 3, 0.6, 200 + seed, empty_rows=(7,))
    eps_g = [0.0, 1e-4, 1e-2, 0.3, 2.0, 10.0][seed]
    (rp, ci, va), passes, tau, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(Bm),
                                                                  self_coef, divisor, eps_g)
    Ct = O.spgemm(A, Bm, self_coef, divisor)
    keep, tau_o, passes_o, _, _ = O.alg41(Ct.val, eps_g, 0.1)
    assert nnz_unf == Ct.nnz
    assert passes == passes_o
    if np.isfinite(tau_o):
        assert tau == pytest.approx(tau_o, rel=1e-12)
    G = csr_to_dense(from_dev(n, rp, ci, va))
    Cd = csr_to_dense(Ct)
    rows = np.repeat(np.arange(n), np.diff(Ct.rowptr))
    ref = np.zeros((n, n))
    ref[rows[keep], Ct.col[keep]] = Ct.val[keep]
    # kept sets equal except entries within rounding of tau
    diff = np.abs(G - ref)
    assert diff.max() <= 1e-13 * max(np.abs(Cd).max(), 1e-300) + 10 * (tau if np.isfinite(tau) else 0)


HAND = [
    ([1.0] * 4 + [1e-3] * 100, 5e-3, 0.01, 4, 6.25e-4),
    ([1.0, 1e-20], 1e-10, 0.1, 1, 1e-10),
    ([1.0] * 4, 1e-12, 0.1, 1, 1e-12),
    ([1.0] + [1e-4] * 16, 1e-3, 0.1, 1, 1e-3),
    ([1.0] * 2 + [4e-4] * 25 + [1e-4] * 100, 1e-3, 0.1, 3, 2e-4),
    ([5.0, 0.5], 1.0, 0.1, 1, 1.0),  # reading R1: the first pass always runs
]


@pytest.mark.parametrize("case", range(len(HAND)))
def test_alg41_hand_traces_gpu(B, case):
    import torch
    vals, eps_g, e_r, passes, tau = HAND[case]
    x = torch.tensor(vals, dtype=torch.float64, device="cuda")
    p, t, d = B.sexpm_alg41(x, eps_g, e_r)
    assert p == passes
    assert t == pytest.approx(tau, rel=1e-14)


def test_alg41_random_vs_oracle(B):
    import torch
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 5000))
        x = 10.0 ** rng.uniform(-22, 0, n) * rng.choice([-1.0, 1.0], n)
        eps_g = 10.0 ** rng.uniform(-20, -2)
        keep, tau_o, passes_o, dropped_o, _ = O.alg41(x, eps_g, 0.1)
        p, t, d = B.sexpm_alg41(torch.from_numpy(x).cuda(), eps_g, 0.1)
        assert p == passes_o
        assert t == pytest.approx(tau_o, rel=1e-12)
        assert d == pytest.approx(dropped_o, rel=1e-10, abs=1e-300)


@pytest.mark.parametrize("kernel", [0, 3, 5, 6, 7, 11, 13])
@pytest.mark.parametrize("name", ["heat2d_pm10_20", "structural_24", "heat3d_9", "banded_nonsym"])
def test_accumulator_variants(B, kernel, name):
    """Every K3 kernel (block-window 3, paged 5, Taylor pull 6 / diagonal 7, block-sparse
    exact 11 and tensor-core 13) meets parity."""
    H = SMALL[name]()
    Eg, st, Eo, tr = run_both(B, H, kernel=kernel)
    assert_parity(Eg, st, Eo, tr)


def assert_products_close(G, Ct, A, Bm, self_coef, row_slice=None):
    """C~ from the tensor-core kernel 13 (fused multiply-adds, K ascending in 8x8x4 steps)
    against the oracle's C~: same pattern, and every value within the running-sum rounding
    bound (m + 2) u sum_k |a_rk||b_kj| (+ |self a_rj|), m = the products of the row (Higham's
    gamma_m bound, u = 2^-53)."""
    Aa = CSR(A.n, A.rowptr, A.col, np.abs(A.val))
    Ba = CSR(Bm.n, Bm.rowptr, Bm.col, np.abs(Bm.val))
    Abs = O.spgemm(Aa, Ba, abs(self_coef), 1.0)
    rows_prod = np.array([np.diff(Bm.rowptr)[A.col[A.rowptr[r]:A.rowptr[r + 1]]].sum() + 1
                          for r in range(A.rowptr.size - 1)], dtype=np.float64)
    gs, cs = scipy_like(G), scipy_like(Ct)
    bound = scipy_like(Abs).multiply(2.0 ** -53 * (rows_prod[:, None] + 2)).toarray()
    if row_slice is not None:
        bound = bound[row_slice[0]:row_slice[1]]
    diff = np.abs((gs - cs).toarray())
    assert (diff <= bound + 1e-300).all(), float((diff - bound).max())
    # pattern: equal except where the exact value cancels to (near) zero
    pg, pc = (gs != 0).toarray(), (cs != 0).toarray()
    assert ((pg == pc) | (np.maximum(np.abs(gs.toarray()), np.abs(cs.toarray())) <= bound)).all()


def scipy_like(M):
    import scipy.sparse as sp
    return sp.csr_matrix((M.val, M.col, M.rowptr), shape=(M.rowptr.size - 1, M.n))


@pytest.mark.parametrize("kernel", [5, 11, 13])
@pytest.mark.parametrize("seed", range(4))
def test_bit_exact_products(B, seed, kernel):
    """The paged (5) and exact block (11) kernels accumulate the self term first, then
    ascending k with round-to-nearest products and sums (no FMA): C~ is bit-identical to the
    oracle.  The tensor-core block kernel (13) fuses the products: within the rounding
    bound."""
    import torch
    n = 300
    A = _rand_csr(n, 9, 0.6, 300 + seed, empty_rows=(3, 200))
    (rp, ci, va), passes, tau, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(A), 2.0, 1.0,
                                                                  0.0, kernel=kernel)
    Ct = O.spgemm(A, A, 2.0, 1.0)
    G = from_dev(n, rp, ci, va)
    if kernel == 13:
        assert_products_close(G, Ct, A, A, 2.0)
        return
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)  # bit-exact


@pytest.mark.parametrize("seed", range(3))
def test_taylor_pull_bit_exact(B, seed):
    """A Taylor term S~ = S^ H0 / i through the pull kernel equals the oracle bit for bit
    (ascending k along H0's columns, _rn products and sums, then / i)."""
    import torch
    from synth import laplacian_2d
    H = laplacian_2d(30, 30, 0.4, "pm10", seed=seed)
    S = O.spgemm(H, H, 0.0, 2.0)  # a realistic S^_2
    (g_rp, g_ci, g_va), passes, tau, nu = B.sexpm_filtered_product(H.n, to_dev(S), to_dev(H),
                                                                   0.0, 3.0, 0.0)
    G = from_dev(H.n, g_rp, g_ci, g_va)
    Ct = O.spgemm(S, H, 0.0, 3.0)
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)


@pytest.mark.parametrize("name", ["heat2d", "structural", "heat3d", "heat1d", "banded1d"])
def test_taylor_dia_bit_exact(B, name):
    """Unfiltered Taylor phase (filter off, N = 0) through the diagonal push kernel K5d:
    every term S~ = S^ H0 / i accumulates k ascending with _rn products and sums, the
    merges add exactly, so E = I + sum S^_i equals the oracle's bit for bit."""
    from synth import structural_state_space, laplacian_3d
    if name == "heat2d":
        H = laplacian_2d(40, 40, 0.6, "pm10", seed=3)
    elif name == "structural":
        H = structural_state_space(12, 10, 0.5, seed=4)
    elif name == "heat3d":
        H = laplacian_3d(8, 7, 6, 0.25, "u0812", seed=5)
    elif name == "heat1d":  # short rows: the thread-per-row kernel K5s
        H = tridiag(3001, 0.45, -0.9, 0.45)
    else:  # 5 diagonals, short rows, ragged ends (K5s)
        H = random_banded(2000, 2, 1.0, 0.3, seed=6)
    opts = dict(filter=0, force_N=0, force_M=9)
    Eg, st = run_gpu(B, H, kernel=7, **opts)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS, **opts)
    assert np.array_equal(Eg.rowptr, Eo.rowptr) and np.array_equal(Eg.col, Eo.col)
    assert np.array_equal(Eg.val, Eo.val)
    assert st["taylor_fmas"] > 0


@pytest.mark.parametrize("name", ["heat2d", "structural", "heat3d", "heat1d", "banded1d", "tiny"])
def test_taylor_window_bit_exact(B, name):
    """Unfiltered Taylor phase (filter off, N = 0) on the offset-window kernel K5w: every
    term is a dense row over the Minkowski sums of H0's offsets, products summed with the
    offsets descending (k ascending, the oracle's order) and divided by i, T^_0 accumulated
    term by term -- E = I + T^_0 equals the oracle's bit for bit."""
    from synth import structural_state_space, laplacian_3d
    if name == "heat2d":
        H = laplacian_2d(40, 40, 0.6, "pm10", seed=3)
    elif name == "structural":
        H = structural_state_space(12, 10, 0.5, seed=4)
    elif name == "heat3d":
        H = laplacian_3d(8, 7, 6, 0.25, "u0812", seed=5)
    elif name == "heat1d":
        H = tridiag(3001, 0.45, -0.9, 0.45)
    elif name == "banded1d":  # 5 diagonals, ragged ends
        H = random_banded(2000, 2, 1.0, 0.3, seed=6)
    else:  # fewer rows than the window's offsets
        H = tridiag(7, 0.45, -0.9, 0.45)
    opts = dict(filter=0, force_N=0, force_M=9)
    Eg, st = run_gpu(B, H, kernel=8, **opts)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS, **opts)
    assert st["taylor_window"] == 1
    assert np.array_equal(Eg.rowptr, Eo.rowptr) and np.array_equal(Eg.col, Eo.col)
    assert np.array_equal(Eg.val, Eo.val)
    assert st["taylor_fmas"] > 0


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_taylor_window_filtered_vs_oracle(B, cid):
    """Filtered Taylor phase on K5w (default for these stencils): per term the same Algorithm
    4.1 decisions as the oracle (nnz of S^_i, passes; tau within rounding of the pass sums),
    and T^_0 (output_T with N = 0) within the north-star criteria."""
    H = make_config(cid)
    Eg, st, Eo, tr = run_both(B, H, force_N=0, output_T=True)
    assert st["taylor_window"] == 1
    assert st["M_eff"] == tr["M_eff"]
    for i in range(2, tr["M_eff"] + 1):
        assert st["taylor_nnz_unf"][i] == tr["taylor_nnz_unf"][i]
        assert abs(int(st["taylor_nnz"][i]) - int(tr["taylor_nnz"][i])) <= max(2, tr["taylor_nnz"][i] // 10**6)
        assert st["taylor_passes"][i] == tr["taylor_passes"][i]
        assert st["taylor_tau"][i] == pytest.approx(tr["taylor_tau"][i], rel=1e-12)
    assert_parity(Eg, st, Eo, tr)


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_taylor_window_matches_dia(B, cid):
    """The window kernel (8) and the diagonal push kernel (7) take the same Taylor-phase
    decisions on the BASELINE configs (both reproduce the oracle's S~ bit for bit)."""
    H = make_config(cid)
    # the full window (the symmetric path's half window is not bit-exact: sym_squaring = 0)
    _, s8 = run_gpu(B, H, kernel=8, sym_squaring=0)
    _, s7 = run_gpu(B, H, kernel=7, sym_squaring=0)
    assert s8["taylor_window"] == 1 and s7["taylor_window"] == 0
    M = s8["M_eff"]
    assert M == s7["M_eff"]
    for i in range(2, M + 1):
        assert s8["taylor_nnz_unf"][i] == s7["taylor_nnz_unf"][i]
        assert s8["taylor_nnz"][i] == s7["taylor_nnz"][i]
        assert s8["taylor_tau"][i] == pytest.approx(s7["taylor_tau"][i], rel=1e-12)
    assert s8["sq_nnz"][0] == s7["sq_nnz"][0]


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_taylor_dia_default_matches_pull(B, cid):
    """Filtered runs through K5d (default) and the pull kernel (kernel=6) give the same
    Taylor-phase patterns (both reproduce the oracle's S~ bit for bit)."""
    H = make_config(cid)
    _, s7 = run_gpu(B, H, kernel=7)
    _, s6 = run_gpu(B, H, kernel=6)
    M = s7["M_eff"]
    assert M == s6["M_eff"]
    for i in range(2, M + 1):
        assert s7["taylor_nnz"][i] == s6["taylor_nnz"][i]
        # the two kernels stage rows in different pool orders, so the pass sums may differ
        # in the last bits
        assert s7["taylor_tau"][i] == pytest.approx(s6["taylor_tau"][i], rel=1e-12)


def _coo(n, rows, cols, vals):
    """CSR from COO triplets, duplicate (row, col) pairs dropped (first kept)."""
    from synth.configs import coo_to_csr
    rows, cols = np.asarray(rows, np.int64), np.asarray(cols, np.int64)
    _, first = np.unique(rows * n + cols, return_index=True)
    return coo_to_csr(n, rows[first], cols[first], np.asarray(vals, np.float64)[first])


@pytest.mark.parametrize("kernel", [5])
def test_long_b_rows(B, kernel):
    """B rows longer than a CTA (> 512 entries) in the paged kernel (A != B: not a
    squaring): A x B + 2A is bit-identical to the oracle."""
    n = 3000
    rng = np.random.default_rng(11)
    Bm = random_banded(n, 450, 0.85, 1.0, 12)
    rows = np.repeat(np.arange(n), 4)
    cols = np.clip(rows + rng.integers(-40, 41, rows.size), 0, n - 1)
    A = _coo(n, rows, cols, rng.uniform(-1, 1, rows.size))
    assert np.diff(Bm.rowptr).max() > 512
    (rp, ci, va), _, _, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(Bm), 2.0, 1.0, 0.0,
                                                           kernel=kernel)
    Ct = O.spgemm(A, Bm, 2.0, 1.0)
    G = from_dev(n, rp, ci, va)
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)


@pytest.mark.parametrize("kernel", [11, 13])
def test_block_kernel_fallback_wide_rows(B, kernel):
    """Block rows whose column span exceeds the block kernels' bitmaps fall through to the
    paged kernel; the result is unchanged (bit-identical to the oracle)."""
    n = 150_000
    rng = np.random.default_rng(13)
    rows = np.repeat(np.arange(n), 3)
    cols = rng.integers(0, n, rows.size)
    cols[::3] = rows[::3]
    A = _coo(n, rows, cols, rng.uniform(-1, 1, rows.size))
    (rp, ci, va), _, _, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(A), 2.0, 1.0, 0.0,
                                                           kernel=kernel)
    Ct = O.spgemm(A, A, 2.0, 1.0)
    G = from_dev(n, rp, ci, va)
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)


@pytest.mark.parametrize("kernel", [11, 13])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 17, 250, 1003])
def test_bsr_kernel_bit_exact_sizes(B, n, kernel):
    """The block kernels (BSR-8 view) on sizes that are not multiples of 8, with empty
    rows: C~ = 2A + A*A bit-identical to the oracle (11), within the rounding bound (13)."""
    A = _rand_csr(n, min(n, 12), 0.5, 400 + n, empty_rows=tuple(r for r in (0, 3, n // 2) if r < n))
    (rp, ci, va), _, _, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(A), 2.0, 1.0, 0.0,
                                                           kernel=kernel)
    Ct = O.spgemm(A, A, 2.0, 1.0)
    G = from_dev(n, rp, ci, va)
    if kernel == 13:
        assert_products_close(G, Ct, A, A, 2.0)
        return
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)


EMPTY_DIAG = {
    # a single entry in block (0, 1): block row 1 is empty, so no B_K of row 0 has block 1;
    # the self term 2 A alone must produce C~(0, 8)
    "single_offdiag": lambda: _coo(16, [0], [8], [1.5]),
    # strictly upper triangular (nilpotent, DAG-like): empty diagonal blocks everywhere
    "strict_upper": lambda: dense_to_csr(np.triu(csr_to_dense(random_banded(200, 20, 0.2, 1.0, 41)), 1)),
    # bipartite [[0, X], [0, 0]]
    "bipartite": lambda: dense_to_csr(np.block([[np.zeros((64, 64)), csr_to_dense(random_banded(64, 30, 0.3, 1.0, 42))],
                                               [np.zeros((64, 64)), np.zeros((64, 64))]])),
}


@pytest.mark.parametrize("kernel", [11, 13, 5])
@pytest.mark.parametrize("name", sorted(EMPTY_DIAG))
def test_block_kernels_empty_diagonal_blocks(B, kernel, name):
    """Squarings C~ = 2A + A*A where A has empty diagonal blocks: every self-term block is a
    candidate output block even when no product reaches it."""
    A = EMPTY_DIAG[name]()
    n = A.n
    (rp, ci, va), _, _, nnz_unf = B.sexpm_filtered_product(n, to_dev(A), to_dev(A), 2.0, 1.0, 0.0,
                                                           kernel=kernel)
    Ct = O.spgemm(A, A, 2.0, 1.0)
    G = from_dev(n, rp, ci, va)
    assert nnz_unf == Ct.nnz
    if kernel == 13:
        assert_products_close(G, Ct, A, A, 2.0)
        return
    assert np.array_equal(G.rowptr, Ct.rowptr) and np.array_equal(G.col, Ct.col)
    assert np.array_equal(G.val, Ct.val)


@pytest.mark.parametrize("kernel", [11, 13, 5])
@pytest.mark.parametrize("r0,r1,h0,h1", [(96, 200, 88, 208), (96, 203, 88, 216), (0, 57, 0, 64),
                                         (100, 180, 88, 192), (200, 257, 192, 257)])
def test_block_kernel_rank_slice_in_halo(B, kernel, r0, r1, h0, h1):
    """The multi-GPU shape of a squaring on one GPU: A = rows [r0, r1) of T, B = its halo rows
    [h0, h1) (Lemma 3.1 coverage).  Block-aligned slices (r0 - h0 and h0 multiples of 8) run
    the block kernel K3b on B's BSR view, the others fall through to K3p; C~ = 2A + A B is
    bit-identical to the oracle's rows either way."""
    n = 257
    T = _rand_csr(n, 6, 0.5, 900 + r0, empty_rows=(0, 100, 256))
    Ct = O.spgemm(T, T, 2.0, 1.0)
    def rows(M, a, b):
        rp = M.rowptr[a:b + 1] - M.rowptr[a]
        sl = slice(M.rowptr[a], M.rowptr[b])
        return CSR(n, rp.astype(np.int64), M.col[sl].copy(), M.val[sl].copy())
    A_, B_ = rows(T, r0, r1), rows(T, h0, h1)
    (rp, ci, va), _, _, nnz_unf = B.sexpm_filtered_product(n, to_dev(A_), to_dev(B_), 2.0, 1.0, 0.0,
                                                           kernel=kernel, a_row0=r0, b_row0=h0)
    G = from_dev(n, rp, ci, va)
    Cr = rows(Ct, r0, r1)
    if kernel == 13:
        assert_products_close(G, Cr, T, T, 2.0, row_slice=(r0, r1))
        return
    assert np.array_equal(G.rowptr, Cr.rowptr) and np.array_equal(G.col, Cr.col)
    assert np.array_equal(G.val, Cr.val)


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_aggregate_order_matches_index_order(B, cid):
    """Squarings in 8-row aggregate order (default) and in index order (sq_order = 0) give
    the same e^H up to rounding order (north-star parity between the two), the same plan,
    and the aggregate order does not execute more block products."""
    H = make_config(cid)
    Ea, sa = run_gpu(B, H)
    Ei, si = run_gpu(B, H, sq_order=0)
    assert (sa["M"], sa["N"]) == (si["M"], si["N"])
    ok, res = parity(Ea, Ei, max(si["sq_tau"][si["N"]], sa["sq_tau"][sa["N"]], 1e-300))
    assert ok, res
    N = sa["N"]
    assert sa["sq_block_products"][1:N + 1].sum() <= si["sq_block_products"][1:N + 1].sum()


@pytest.mark.parametrize("name", ["heat2d", "heat2d_ragged", "heat3d"])
def test_lattice_order_on_device(B, name, monkeypatch):
    """Grid stencils on one GPU: the squarings' aggregate relabelling is computed on the
    device (2D diamond tiles / 3D 2x2x2 cubes, sq_order_used 3 / 4) -- parity against the
    oracle, and against the host-thread aggregates (SEXPM_NO_LATTICE); no more block products
    than index order."""
    from synth import laplacian_3d
    if name == "heat2d":
        H = laplacian_2d(64, 48, 1.0, "pm10", seed=11)
    elif name == "heat2d_ragged":  # extents not multiples of the tiles (partial tiles)
        H = laplacian_2d(37, 29, 0.8, "pm10", seed=12)
    else:
        H = laplacian_3d(18, 16, 14, 0.25, "u0812", seed=13)
    Eg, st = run_gpu(B, H)
    assert st["sq_order_used"] == (4 if name == "heat3d" else 3)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    assert_parity(Eg, st, Eo, tr)
    monkeypatch.setenv("SEXPM_NO_LATTICE", "1")
    Eh, sh = run_gpu(B, H)
    assert sh["sq_order_used"] in (0, 1, 2)
    ok, res = parity(Eg, Eh, max(st["sq_tau"][st["N"]], sh["sq_tau"][sh["N"]], 1e-300))
    assert ok, res
    monkeypatch.delenv("SEXPM_NO_LATTICE")
    Ei, si = run_gpu(B, H, sq_order=0)
    N = st["N"]
    assert st["sq_block_products"][1:N + 1].sum() <= si["sq_block_products"][1:N + 1].sum()


def test_aggregate_order_with_reorder(B):
    """Both relabellings at once (RCM of a scrambled input, then the aggregates of the
    squarings): parity against the oracle."""
    import scipy.sparse as sp
    H0 = laplacian_2d(40, 30, 1.0)
    q = np.random.default_rng(3).permutation(H0.n)
    A = sp.csr_matrix((H0.val, H0.col, H0.rowptr), shape=(H0.n, H0.n))[q][:, q].tocsr()
    A.sort_indices()
    H = CSR(H0.n, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64))
    Eg, st = run_gpu(B, H, reorder=1)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    assert_parity(Eg, st, Eo, tr)


@pytest.mark.parametrize("g", [20])
def test_wide_3d_rows_on_tensor_core_kernel(B, g):
    """Config 4's law (3D 7-point heat, c ~ U(0.8, 1.2)) at 20^3: the squarings' block rows
    hold more blocks of A than the exact kernel's shared-memory row (K3b hands them to the
    paged kernel), while the tensor-core kernel takes every row (no fallback rows) and the
    result meets parity against the oracle (BASELINE config 4)."""
    H = make_config(4, scale_down=g)
    Eg, st, Eo, tr = run_both(B, H)
    assert_plan_equal(st, tr)
    assert_parity(Eg, st, Eo, tr)
    N = st["N"]
    assert N >= 1 and all(st["sq_fallback_rows"][1:N + 1] == 0)
    _, s11 = run_gpu(B, H, kernel=11)
    assert s11["sq_fallback_rows"][1:N + 1].sum() > 0  # K3b cannot hold these rows
