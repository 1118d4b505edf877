"""Pins of the oracle's N1 apply: Y = A^steps X, the step
u_{k+1} = e^H u_k of the discretised system (Eq. 2.2).

Pinned against things other than itself: a dense matrix product (numpy), the
semigroup property E^k = e^{kH} through the 1D Dirichlet closed form
(refs.heat1d_exact), and the invariant E 1 = 1 of zero-row-sum generators.
"""
import numpy as np
import pytest

import oracle as O
from synth import csr_to_dense, neumann_laplacian_2d, random_banded
from synth.configs import CSR

import refs

U = 2.0 ** -53


def _tridiag(n, r):
    rp = [0]
    ci, va = [], []
    for i in range(n):
        for j, v in ((i - 1, r), (i, -2 * r), (i + 1, r)):
            if 0 <= j < n:
                ci.append(j)
                va.append(v)
        rp.append(len(ci))
    return CSR(n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(va, np.float64))


@pytest.mark.parametrize("m", [1, 3, 40])
def test_spmm_matches_dense_product(m):
    """Y = A X against numpy's dense product (different summation order): within the
    running-sum rounding bound nnz(row) u (|A| |X|)."""
    A = random_banded(300, 17, 0.4, 1.0, seed=5)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((300, m))
    Y = O.spmm(A, X)
    Ad = csr_to_dense(A)
    ref = Ad @ X
    bound = 40 * U * (np.abs(Ad) @ np.abs(X))
    assert np.all(np.abs(Y - ref) <= bound + 1e-300)


def test_spmm_vector_and_identity():
    """A = I gives X back exactly; a 1-D X gives a 1-D Y."""
    n = 50
    I = CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n))
    x = np.random.default_rng(3).standard_normal(n)
    assert np.array_equal(O.spmm(I, x), x)
    X = np.random.default_rng(4).standard_normal((n, 7))
    assert np.array_equal(O.spmm(I, X, steps=4), X)


def test_steps_are_powers_of_exp_closed_form():
    """E^k X = e^{kH} X: k steps with the oracle's E = e^H of the 1D Dirichlet heat
    matrix H = 0.5 tridiag(1,-2,1) against the closed form of e^{kH} (images / Bessel)."""
    n, r, k = 120, 0.5, 4
    H = _tridiag(n, r)
    E, tr = O.expm(H, 1e-16)
    X = np.random.default_rng(8).standard_normal((n, 5))
    Y = O.spmm(E, X, steps=k)
    Ek = refs.heat1d_exact(n, k * r)
    ref = Ek @ X
    # each step: E's forward error (<= 2 r_N relative, plus rounding) and the product's
    # rounding; the closed form itself is accurate to ~1e-16
    rN = tr["r0"] * 2.0 ** tr["N"]
    tol = k * (2 * rN + 200 * U) * np.abs(X).max() * 3
    assert np.abs(Y - ref).max() <= tol


def test_zero_row_sum_generator_conserves_ones():
    """A Neumann Laplacian has zero row sums, so e^H 1 = 1 and every step keeps 1."""
    H = neumann_laplacian_2d(12, 10, 0.7, seed=2)
    E, tr = O.expm(H, 1e-16)
    ones = np.ones(H.n)
    Y = O.spmm(E, ones, steps=6)
    rN = tr["r0"] * 2.0 ** tr["N"]
    assert np.abs(Y - 1.0).max() <= 6 * (4 * rN + 64 * U)
