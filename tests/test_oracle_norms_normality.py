"""Pins of the oracle's plan norm and normality decision (Alg. 4.2 step 2; Eq. 4.19,
P:348-356; readings R8 and R16), chosen so that a row-sum / column-sum swap in the 1-norm or a
non-normal H classified as normal fails:
  * ||H||_1 = max column abs sum ("compatible norm"), checked against numpy / scipy on
    non-symmetric matrices whose row and column maxima differ;
  * Table 1's H_1 and config 3's structural state space (Eq. 2.1) are not
    normal: the trace must say normal = 0 and a = min(1, 1/||H||), not 1/(N+1);
  * symmetric and skew-symmetric H are normal (a = 1/(N+1));
  * a normal but neither symmetric nor skew-symmetric H (a circulant) is classified
    non-normal by reading R16 (the smaller, safer budget).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from synth import dense_to_csr, make_config, random_banded
from refs import table1_matrices


def _sp(H):
    return sp.csr_matrix((H.val, H.col, H.rowptr), shape=(H.n, H.n))


def test_norm_one_column_sums_not_row_sums():
    A = np.zeros((3, 3))
    A[0] = [1.0, -2.0, 3.0]  # row sum 6, largest column sum 3
    H = dense_to_csr(A)
    assert O.norm_one(H) == 3.0
    assert O.norm_one(H) == np.abs(A).sum(0).max() != np.abs(A).sum(1).max()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_norm_one_random_nonsymmetric(seed):
    H = random_banded(300, 7, 0.4, 2.0, seed=seed)
    S = _sp(H)
    assert abs(S - S.T).max() > 0
    ref = float(abs(S).sum(axis=0).max())
    assert O.norm_one(H) == pytest.approx(ref, rel=1e-15)
    assert O.norm_fro(H) == pytest.approx(sp.linalg.norm(S, "fro"), rel=1e-14)


def test_table1_H1_is_not_normal():
    A = table1_matrices()[1]
    H = dense_to_csr(A)
    E, tr = O.expm(H, 1e-16)
    assert tr["normal"] == 0
    nrm = np.abs(A).sum(0).max()  # 1-norm plan (default)
    assert tr["norm"] == nrm
    assert tr["a"] == pytest.approx(1.0 / nrm, rel=1e-15)
    assert tr["a"] != pytest.approx(1.0 / (tr["N"] + 1))


def test_structural_config3_is_not_normal():
    H = make_config(3, scale_down=20)  # the config-3 law on a small lattice
    S = _sp(H).toarray()
    assert np.abs(S @ S.T - S.T @ S).max() > 1e-3  # genuinely non-normal
    _, tr = O.expm(H, 1e-12)
    assert tr["normal"] == 0
    assert tr["a"] == pytest.approx(min(1.0, 1.0 / tr["norm"]), rel=1e-15)


def test_symmetric_and_skew_are_normal():
    for H in (make_config(1), dense_to_csr(np.array([[0.0, 2.0], [-2.0, 0.0]]))):
        _, tr = O.expm(H, 1e-16)
        assert tr["normal"] == 1
        assert tr["a"] == pytest.approx(1.0 / (tr["N"] + 1), rel=1e-15)


def test_nonsymmetric_normal_circulant_reading_R16():
    n = 6
    C = np.zeros((n, n))
    for i in range(n):
        C[i, (i + 1) % n] = 0.5
        C[i, (i + 2) % n] = 0.25
    assert np.allclose(C @ C.T, C.T @ C)  # normal
    _, tr = O.expm(dense_to_csr(C), 1e-16)
    assert tr["normal"] == 0  # R16: only bit-exact (skew-)symmetry counts as normal
    _, tr1 = O.expm(dense_to_csr(C), 1e-16, normal=1)
    assert tr1["normal"] == 1
