"""Pins of the oracle's SSAT baseline: the same Taylor phase, then
E_0 = I + T^_0 and N plain squarings E_i = E_{i-1}^2 -- the "SSAT" column of Table 1
(P:442-451), whose loss of accuracy the paper's incremental split (Eq. 2.7) avoids.

Pinned against: the printed SSAT error of H_2 (7.46e-9, reproduced to 3 digits), the
closed forms of e^{H_k} (refs.table1_exact), the paper's claim that PIM's error stays at
the rounding level while SSAT's grows with N, and diagonal H (closed form exp(h)).
"""
import numpy as np
import pytest

import oracle as O
from synth import csr_to_dense, dense_to_csr, diagonal

import refs

U = 2.0 ** -53


def _rel(E, Ex):
    return np.linalg.norm(csr_to_dense(E) - Ex) / np.linalg.norm(Ex)


def test_table1_h2_ssat_printed_error():
    """Table 1, H_2: SSAT relative error 7.46e-9 as printed."""
    A = refs.table1_matrices()[2]
    E, tr = O.expm(dense_to_csr(A), 1e-16, plan_norm="fro", filter=False, ssat=True)
    assert _rel(E, refs.table1_exact(2)) == pytest.approx(7.46e-9, rel=0.01)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_ssat_loses_digits_pim_does_not(k):
    """H_1..H_3 need N = 20-39 squarings: SSAT's error grows far beyond the rounding level,
    the PIM (incremental split) stays at it, both against the closed forms."""
    A = refs.table1_matrices()[k]
    Ex = refs.table1_exact(k)
    Es, _ = O.expm(dense_to_csr(A), 1e-16, plan_norm="fro", filter=False, ssat=True)
    Ep, _ = O.expm(dense_to_csr(A), 1e-16, plan_norm="fro", filter=False)
    es, ep = _rel(Es, Ex), _rel(Ep, Ex)
    assert ep <= 2e-15
    assert es >= 1e-11 and es >= 1000 * ep


def test_ssat_diagonal_closed_form():
    """Diagonal H: E_N = (e^{h/2^N})^{2^N} entrywise; each squaring at most doubles the
    relative error, so |E - exp(h)| <= (2^N + M) 4u exp(h)."""
    h = np.linspace(-3.0, 2.5, 40)
    H = diagonal(h)
    E, tr = O.expm(H, 1e-16, ssat=True, filter=False)
    d = csr_to_dense(E).diagonal()
    assert np.all(np.abs(d - np.exp(h)) <= (2.0 ** tr["N"] + tr["M"]) * 4 * U * np.exp(h))
    assert E.nnz == H.n


def test_ssat_rejects_output_T():
    with pytest.raises(ValueError):
        O.expm(dense_to_csr(refs.table1_matrices()[4]), 1e-16, ssat=True, output_T=True)
