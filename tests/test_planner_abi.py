"""The product's planner (Algorithm 4.2 steps 1-3, Eq. 4.20) checked through the
C ABI (`sexpm_plan_scalars`, host only) against what the paper and mathematics fix -- not
against the oracle's code:
  * the paper's printed plan (M, N) = (20, 8) for ||H||_F = 244.9, eps_tol = 1e-16;
  * a brute-force enumeration of Eq. (4.20) with r0 from 30-digit quadrature of
    (1/M!) int_0^x t^M e^t dt (Eq. 4.5-4.6);
  * r0 against the same quadrature; the budgets a (Eq. 4.19 P:352 / reading R8) and
    eps_g^(0) against their printed definitions in 30 digits.
"""
import math

import mpmath as mp
import pytest

from paper_2110_04493_b200 import binding as B
from paper_2110_04493_b200.build import build


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def _mp_r0(x, M):
    return x ** (M + 1) * mp.quad(lambda u: u ** M * mp.e ** (x * u), [0, 1]) / mp.factorial(M)


def _brute(norm, tol, m_cap=120, n_window=50):
    with mp.workdps(30):
        N0 = max(math.ceil(math.log2(norm)), 0)
        best = None
        for N in range(N0, N0 + n_window + 1):
            x = mp.mpf(norm) / 2 ** N
            if x > 1:
                continue
            for M in range(0, m_cap + 1):
                if 2 ** N * _mp_r0(x, M) <= tol:
                    if best is None or M * 2 ** N < best[0]:
                        best = (M * 2 ** N, M, N)
                    break
    return best[1], best[2]


def test_paper_plan():
    s = B.sexpm_plan_scalars(244.9, 1, 1e-16)  # M = 20, N = 8
    assert (s["M"], s["N"]) == (20, 8)


@pytest.mark.parametrize("norm,tol", [(1.0, 1e-16), (2.0, 1e-16), (4.0, 1e-16), (5.93, 1e-12),
                                      (244.9, 1e-16), (0.3, 1e-8), (8.7, 1e-6), (3239.8, 1e-16),
                                      (0.5, 1e-16), (1024.0, 1e-16), (1025.0, 1e-10)])
def test_plan_bruteforce(norm, tol):
    s = B.sexpm_plan_scalars(norm, 1, tol)
    assert (s["M"], s["N"]) == _brute(norm, tol)


@pytest.mark.parametrize("norm", [0.7, 4.0, 244.9, 3239.8])
@pytest.mark.parametrize("normal", [0, 1])
def test_budgets(norm, normal):
    s = B.sexpm_plan_scalars(norm, normal, 1e-16)
    M, N = s["M"], s["N"]
    with mp.workdps(30):
        x = mp.mpf(norm) / 2 ** N
        r0 = _mp_r0(x, M)
        a = mp.mpf(1) / (N + 1) if normal else min(mp.mpf(1), 1 / mp.mpf(norm))
        eg0 = a * r0 / (M * mp.e ** (2 * x))
    assert s["r0"] == pytest.approx(float(r0), rel=1e-15)
    assert s["a"] == pytest.approx(float(a), rel=1e-15)
    assert s["eps_g0"] == pytest.approx(float(eg0), rel=1e-14)


def test_zero_and_errors():
    s = B.sexpm_plan_scalars(0.0, 1, 1e-16)
    assert (s["M"], s["N"]) == (0, 0) and s["eps_g0"] == 0.0
    with pytest.raises(B.SexpmError):
        B.sexpm_plan_scalars(4.0, 1, 1e-17)  # reading R13
    with pytest.raises(B.SexpmError):
        B.sexpm_plan_scalars(1e300, 1, 1e-16, 120, 2)  # infeasible in the window
    with pytest.raises(B.SexpmError):
        B.sexpm_plan_scalars(-1.0, 1, 1e-16)
