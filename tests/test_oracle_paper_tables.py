"""Pins of the oracle against the numbers PAPER.md prints.

* Table 3: lambda(T^_i) = 14,16,18,20,22,26,32,38 for
  H = tridiag(1,-2,1), n = 10^4, eps_tol = 1e-16, Frobenius plan (M, N) = (20, 8),
  squaring budget eps_g^(i) = a r_i ||I + T^_{i-1}||_F (reading R4).
* Table 2: lambda(S^_i) = 2i for i = 2..8, S^_i = 0 for i >= 10,
  "only eight matrix multiplications"; i = 9 printed 14 (reading R4b: +-2).
* Table 3's unfiltered row: lambda(T_i) = 40 * 2^i (doubling per squaring).
* Table 1: relative errors of the proposed method on five small
  matrices against 50-digit closed forms.
* Table 4: middle column of e^H for H = tridiag(-1,2,-1)/(n+1)
  against G_s = (-1)^s e^{2c} I_s(2c), c = 1/(n+1) (reading R14 of the garbled
  binomial series).
"""
import numpy as np
import pytest
from scipy.special import ive

import oracle as O
from synth import csr_to_dense, dense_to_csr, tridiag

import refs


@pytest.fixture(scope="module")
def toeplitz_run():
    H = tridiag(10_000, 1.0, -2.0, 1.0)
    return O.expm(H, 1e-16, plan_norm="fro")


def test_table3_filtered_bandwidths(toeplitz_run):
    _, tr = toeplitz_run
    assert (tr["M"], tr["N"]) == (20, 8)
    lam = [int(tr["sq_l1"][i] + tr["sq_l2"][i]) for i in range(1, 9)]
    assert lam == [14, 16, 18, 20, 22, 26, 32, 38]


def test_table2_taylor_bandwidths(toeplitz_run):
    _, tr = toeplitz_run
    lam = [int(tr["taylor_l1"][i] + tr["taylor_l2"][i]) for i in range(2, 9)]
    assert lam == [4, 6, 8, 10, 12, 14, 16]
    assert abs(int(tr["taylor_l1"][9] + tr["taylor_l2"][9]) - 14) <= 2
    assert tr["taylor_nnz"][10] == 0
    assert tr["M_eff"] == 9  # products for i = 2..9: eight multiplications


def test_table3_unfiltered_doubling():
    H = tridiag(1500, 1.0, -2.0, 1.0)
    _, tr = O.expm(H, 1e-16, plan_norm="fro", filter=False, force_M=20, force_N=3, output_T=True)
    lam = [int(tr["sq_l1"][i] + tr["sq_l2"][i]) for i in range(0, 4)]
    assert lam == [40, 80, 160, 320]


# printed relative errors of the proposed algorithm, Table 1
TABLE1 = {1: 3.19e-16, 2: 6.43e-17, 3: 3.15e-16, 4: 2.71e-14, 5: 1.39e-16}
# printed SSAT errors: a plain SSA without the incremental split is far worse
TABLE1_SSAT = {1: 2.06e-9, 2: 7.46e-9, 3: 1.82e-8, 4: 8.68e-14, 5: 5.44e-14}


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_table1_small_matrices(k):
    A = refs.table1_matrices()[k]
    Ex = refs.table1_exact(k)
    E, tr = O.expm(dense_to_csr(A), 1e-16, plan_norm="fro")
    err = np.linalg.norm(csr_to_dense(E) - Ex) / np.linalg.norm(Ex)
    # same order as the paper's printed error; far below the SSAT column
    assert err <= max(10 * TABLE1[k], 2e-15)
    assert err < TABLE1_SSAT[k]


def test_table4_middle_column():
    n = 2000
    c = 1.0 / (n + 1)
    H = tridiag(n, -c, 2 * c, -c)
    E, tr = O.expm(H, 1e-16, plan_norm="fro")
    assert tr["N"] == 0  # ||H||_F < 1: Taylor phase only (BASELINE.md caveat)
    col = csr_to_dense(E)[:, n // 2]
    s = np.abs(np.arange(n) - n // 2)
    G = (-1.0) ** s * np.exp(2 * c) * ive(s, 2 * c) * np.exp(2 * c)  # ive = I e^{-x}
    rel = np.linalg.norm(col - G) / np.linalg.norm(G)
    assert rel < 1e-15
    sparsity = E.nnz / n ** 2
    # loose pin: printed 0.0013 at n = 10^4 -> bandwidth ~ 13 per side; scale with n
    assert 0.3 < sparsity * n / (0.0013 * 10_000) < 3.0
