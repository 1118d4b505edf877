"""Pins of the oracle's N3 reordering: reverse Cuthill-McKee for the real
bandwidth lambda(A) = min_P l(P A P^T) of Def. 3.2a.

Pinned against: the optimum of a shuffled path graph (bandwidth 1, closed form), the
bandwidth of shuffled grid / banded matrices restored (compared with scipy's RCM, a library
routine), the exact order on isolated nodes, and the method's permutation invariance
e^{P H P^T} = P e^H P^T checked with the north-star parity criteria.
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

import oracle as O
from synth import diagonal, laplacian_2d, make_config, random_banded, tridiag
from synth.configs import CSR

from gpu_helpers import last_tau, parity


def _sp(H):
    return sp.csr_matrix((H.val, H.col, H.rowptr), shape=(H.n, H.n))


def _from_sp(A):
    A = A.tocsr()
    A.sort_indices()
    return CSR(A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int32),
               A.data.astype(np.float64))


def permute(H, p):
    """P H P^T with perm[new] = old."""
    return _from_sp(_sp(H)[p][:, p])


def bw(H):
    c = _sp(H).tocoo()
    return int(np.abs(c.row - c.col).max()) if c.nnz else 0


def shuffled(H, seed):
    q = np.random.default_rng(seed).permutation(H.n)
    return permute(H, q), q


def test_rcm_path_graph_is_optimal():
    """A path graph under any labelling: RCM finds bandwidth 1 (the optimum)."""
    H = tridiag(200, 1.0, -2.0, 1.0)
    Hs, _ = shuffled(H, 3)
    p = O.rcm(Hs)
    assert sorted(p.tolist()) == list(range(200))
    assert bw(Hs) > 50 and bw(permute(Hs, p)) == 1


@pytest.mark.parametrize("which", ["grid", "banded", "structural"])
def test_rcm_restores_bandwidth(which):
    if which == "grid":
        H = laplacian_2d(40, 30, 1.0)
    elif which == "banded":
        H = random_banded(600, 12, 0.3, 1.0, seed=4, symmetric=True)
    else:
        H = make_config(3, scale_down=20)
    Hs, _ = shuffled(H, 5)
    p = O.rcm(Hs)
    assert sorted(p.tolist()) == list(range(H.n))
    b = bw(permute(Hs, p))
    ps = reverse_cuthill_mckee(_sp(Hs), symmetric_mode=False)
    assert b <= 1.25 * bw(permute(Hs, ps)) + 2
    assert b <= 1.5 * bw(H) + 2 and bw(Hs) > 4 * b


def test_rcm_isolated_nodes():
    """Diagonal H: every node is its own component, started in index order (all degrees 0);
    reversing gives n-1, ..., 0."""
    p = O.rcm(diagonal(np.arange(1.0, 8.0)))
    assert p.tolist() == list(range(6, -1, -1))


def test_expm_permutation_invariant():
    """e^{P H P^T} = P e^H P^T: the filter and the products are permutation invariant up to
    rounding (summation order), so the two sides meet the north-star parity criteria."""
    H = laplacian_2d(30, 20, 1.0)
    Hs, _ = shuffled(H, 7)
    p = O.rcm(Hs)
    Hr = permute(Hs, p)
    E1, tr1 = O.expm(Hs, 1e-16)
    E2, tr2 = O.expm(Hr, 1e-16)
    inv = np.empty_like(p)
    inv[p] = np.arange(len(p))
    E2back = permute(E2, inv)
    ok, res = parity(E2back, E1, max(last_tau(tr1), last_tau(tr2)))
    assert ok, res


def test_geometric_graph_input_and_rcm():
    """The N4 input law: symmetric, no diagonal, ||H||_1 = 4 exactly, random node order
    (bandwidth ~ n); RCM brings the bandwidth within 1.25x of scipy's."""
    from synth import geometric_graph
    H = geometric_graph(3000, 6.0, 4.0, 1)
    A = _sp(H)
    assert (A != A.T).nnz == 0 and A.diagonal().max() == 0.0
    assert O.norm_one(H) == pytest.approx(4.0, rel=1e-15)
    assert bw(H) > H.n // 2
    p = O.rcm(H)
    ps = reverse_cuthill_mckee(A, symmetric_mode=True)
    assert bw(permute(H, p)) <= 1.25 * bw(permute(H, ps)) + 2
