"""Pins of the oracle against closed forms, invariants and dense references.

Bounds: the method's forward error is r_N (Eq. 4.2-4.6) relative, plus the
filter budget (Eq. 4.18-4.19: total <= (1+c) r_N, c = 1 for normal H), plus
rounding.  Tolerances below add a rounding allowance of a few hundred u on top.
"""
import numpy as np
import pytest

import oracle as O
from synth import (csr_to_dense, dense_to_csr, diagonal, laplacian_2d, make_config,
                   neumann_laplacian_2d, random_banded, random_skew)

import refs

U = 2.0 ** -53


@pytest.mark.parametrize("plan_norm", ["one", "fro"])
def test_config1_heat1d_closed_form(plan_norm):
    """BASELINE.json config 1: 0.5*tridiag(1,-2,1), n = 1000 vs the Bessel-image
    closed form of the Dirichlet heat kernel."""
    H = make_config(1)
    E, tr = O.expm(H, 1e-16, plan_norm=plan_norm)
    Ex = refs.heat1d_exact(1000, 0.5)
    err = np.abs(csr_to_dense(E) - Ex).max()
    assert err <= 4 * U * np.abs(Ex).max() + 1e-16
    assert (tr["M"], tr["N"]) == ((18, 1) if plan_norm == "one" else (16, 6))


def test_heat2d_uniform_kronecker():
    """Separable 2D Dirichlet heat (config 5's law, 24 x 24): e^H = E1 (x) E1."""
    H = laplacian_2d(24, 24, 0.5)
    for pn in ["one", "fro"]:
        E, tr = O.expm(H, 1e-16, plan_norm=pn)
        Ex = refs.heat2d_uniform_exact(24, 24, 0.5)
        rN = tr["r0"] * 2.0 ** tr["N"]
        bound = (2 * rN + 32 * (tr["N"] + 2) * U) * np.abs(Ex).max()
        assert np.abs(csr_to_dense(E) - Ex).max() <= bound


def test_diagonal_exact():
    d = np.array([-3.0, -0.5, 0.0, 1e-3, 0.7, 2.5])
    E, tr = O.expm(diagonal(d), 1e-16, output_T=True, plan_norm="fro")
    T = csr_to_dense(E)
    ref = np.expm1(d)
    steps = tr["M"] + tr["N"] + 2
    assert np.allclose(np.diag(T), ref, rtol=8 * steps * U, atol=1e-300)
    assert np.count_nonzero(T - np.diag(np.diag(T))) == 0


@pytest.mark.parametrize("tol", [1e-16, 1e-12, 1e-8])
def test_zero_row_sum_generator(tol):
    """Neumann Laplacian: H 1 = 0 => e^H 1 = 1."""
    H = neumann_laplacian_2d(14, 13, 0.7, seed=3)
    E, tr = O.expm(H, tol)
    rs = csr_to_dense(E).sum(axis=1)
    rN = tr["r0"] * 2.0 ** tr["N"]
    assert np.abs(rs - 1).max() <= 4 * rN + 64 * U


@pytest.mark.parametrize("tol", [1e-16, 1e-10])
def test_skew_symmetric_orthogonal(tol):
    H = random_skew(60, 4, 0.6, 1.5, seed=11)
    E, tr = O.expm(H, tol)
    assert tr["normal"] == 1
    Ed = csr_to_dense(E)
    rN = tr["r0"] * 2.0 ** tr["N"]
    dev = np.linalg.norm(Ed.T @ Ed - np.eye(60)) / np.linalg.norm(np.eye(60))
    assert dev <= 4 * (rN + 64 * U)


@pytest.mark.parametrize("seed,sym", [(1, True), (2, False), (3, False)])
@pytest.mark.parametrize("tol", [1e-16, 1e-12, 1e-8])
def test_dense_50digit_reference(seed, sym, tol):
    """n <= 200 class: the filtered result vs mpmath expm at 50 digits."""
    H = random_banded(36, 3, 0.7, 1.2, seed=seed, symmetric=sym)
    Ex = refs.mp_expm(csr_to_dense(H), dps=50)
    E, tr = O.expm(H, tol)
    rN = tr["r0"] * 2.0 ** tr["N"]
    err = np.linalg.norm(csr_to_dense(E) - Ex) / np.linalg.norm(Ex)
    c = 1.0 if tr["normal"] else max(1.0, tr["norm"])
    assert err <= (1 + c) * rN * 4 + 256 * U


@pytest.mark.parametrize("seed", [4, 5])
def test_filter_off_equals_dense_pim(seed):
    """Filter off (eps_g = 0) is the plain PIM; compare with a dense
    long-double PIM using the same (M, N)."""
    H = random_banded(80, 4, 0.8, 2.0, seed=seed)
    E, tr = O.expm(H, 1e-16, filter=False)
    Ed = refs.dense_pim_longdouble(csr_to_dense(H), tr["M"], tr["N"])
    err = np.linalg.norm(csr_to_dense(E) - Ed) / np.linalg.norm(Ed)
    assert err <= 64 * (tr["M"] + tr["N"]) * U


@pytest.mark.parametrize("tol", [1e-8, 1e-12])
def test_filtered_within_forward_bound_of_unfiltered(tol):
    """Eq. (4.18)-(4.19) with c = 1 for normal H: ||E_f - E_u|| <= r_N ||E_u||."""
    H = laplacian_2d(20, 20, 0.9, "pm10", seed=9)
    Ef, trf = O.expm(H, tol)
    Eu, tru = O.expm(H, tol, filter=False)
    rN = trf["r0"] * 2.0 ** trf["N"]
    A, B = csr_to_dense(Ef), csr_to_dense(Eu)
    assert np.linalg.norm(A - B) <= (rN + 64 * U) * np.linalg.norm(B)
    assert Ef.nnz < Eu.nnz


def test_symmetric_input_symmetric_output():
    H = make_config(2, scale_down=18)
    E, _ = O.expm(H, 1e-16)
    D = csr_to_dense(E)
    assert np.linalg.norm(D - D.T) <= 1e-12 * np.linalg.norm(D)


def test_spgemm_vs_dense_and_lemma31():
    """Products are pinned to numpy's dense matmul (library routine) and obey
    Lemma 3.1(b) l(AB) <= l(A) + l(B)."""
    rng = np.random.default_rng(0)
    for s in range(20):
        A = random_banded(40, int(rng.integers(0, 5)), 0.6, 1.0, seed=100 + s)
        B = random_banded(40, int(rng.integers(0, 5)), 0.6, 1.0, seed=200 + s)
        C = O.spgemm(A, B, self_coef=2.0, divisor=3.0)
        Ad, Bd = csr_to_dense(A), csr_to_dense(B)
        ref = (2.0 * Ad + Ad @ Bd) / 3.0
        assert np.allclose(csr_to_dense(C), ref, rtol=1e-14, atol=1e-15)
        la, lb, lc = (sum(O.bandwidth(X)) for X in (A, B, O.spgemm(A, B)))
        assert lc <= la + lb
        S = O.add(A, B)
        assert np.array_equal(csr_to_dense(S), Ad + Bd)
