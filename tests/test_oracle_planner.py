"""Pins of the oracle's error model and planner (§4.1, §4.3).

r0 (Eq. 4.5) is pinned to two closed forms that are NOT its series:
  (a) r0(x, M) = (1/M!) int_0^x t^M e^t dt  (termwise integration of the series),
      evaluated by mpmath quadrature at 40 digits;
  (b) (-1)^{M+1} gamma(M+1, -x) / M! with the lower incomplete gamma written through
      Kummer's function, gamma(s, z) = z^s / s 1F1(s; s+1; -z) (mpmath hyp1f1), i.e.
      r0 = x^{M+1} / (M+1)! 1F1(M+1; M+2; x).
The plan (Eq. 4.20) is pinned to the paper's printed (M, N) = (20, 8)
for ||H||_F = 244.9 and to a brute-force mpmath enumeration.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle as O
from synth import tridiag


def test_r0_telescoping():
    # sum_i 1/(i!(i+1)) = e - 1
    assert O.r0(1.0, 0) == pytest.approx(math.e - 1, rel=1e-15)
    assert O.r0(0.0, 5) == 0.0


@pytest.mark.parametrize("x", [1e-3, 0.1, 0.5, 0.9566, 1.0])
@pytest.mark.parametrize("M", [0, 1, 5, 12, 20, 30])
def test_r0_vs_quadrature_and_gamma(x, M):
    with mp.workdps(40):
        xm = mp.mpf(x)
        # int_0^x t^M e^t dt = x^{M+1} int_0^1 u^M e^{x u} du  (scaled for relative accuracy)
        q = xm ** (M + 1) * mp.quad(lambda u: u ** M * mp.e ** (xm * u), [0, 1]) / mp.factorial(M)
        z = -xm
        gamma_lower = z ** (M + 1) / (M + 1) * mp.hyp1f1(M + 1, M + 2, -z)
        g = (-1) ** (M + 1) * gamma_lower / mp.factorial(M)
        assert abs(q - g) <= mp.mpf(10) ** -30 * abs(q)
        ref = float(q)
    assert O.r0(x, M) == pytest.approx(ref, rel=2e-16, abs=0)


def test_plan_paper_toeplitz():
    # PAPER.md §5.2: ||H|| = 244.9, eps_tol = 1e-16 -> M = 20, N = 8
    assert O.plan(244.9, 1e-16) == (20, 8)
    H = tridiag(10_000, 1.0, -2.0, 1.0)
    nf = O.norm_fro(H)
    assert nf == pytest.approx(244.9, abs=0.05)
    assert O.plan(nf, 1e-16) == (20, 8)


def test_plan_zero():
    assert O.plan(0.0, 1e-16) == (0, 0)


def _mp_r0(x, M):
    return x ** (M + 1) * mp.quad(lambda u: u ** M * mp.e ** (x * u), [0, 1]) / mp.factorial(M)


@pytest.mark.parametrize("norm,tol", [(1.0, 1e-16), (2.0, 1e-16), (4.0, 1e-16), (5.93, 1e-12),
                                      (244.9, 1e-16), (0.3, 1e-8), (8.7, 1e-6)])
def test_plan_bruteforce(norm, tol):
    """Independent enumeration with the integral form of r0 in 30 digits."""
    with mp.workdps(30):
        N0 = max(math.ceil(math.log2(norm)), 0)
        best = None
        for N in range(N0, N0 + 51):
            x = mp.mpf(norm) / 2 ** N
            if x > 1:
                continue
            for M in range(0, 121):
                if 2 ** N * _mp_r0(x, M) <= tol:
                    if best is None or M * 2 ** N < best[0]:
                        best = (M * 2 ** N, M, N)
                    break
    assert O.plan(norm, tol) == (best[1], best[2])


def test_plan_minimality():
    for norm in [0.5, 1.0, 3.0, 37.0, 244.9]:
        M, N = O.plan(norm, 1e-16)
        x = norm / 2 ** N
        assert x <= 1.0
        assert 2 ** N * O.r0(x, M) <= 1e-16
        if M > 0:
            assert 2 ** N * O.r0(x, M - 1) > 1e-16


def test_norms_closed_forms():
    H = tridiag(1000, 1.0, -2.0, 1.0)
    assert O.norm_one(H) == 4.0
    assert O.norm_fro(H) == pytest.approx(math.sqrt(4 * 1000 + 2 * 999), rel=1e-15)
    assert O.bandwidth(H) == (1, 1)
