"""GPU parity of N3: the device reverse Cuthill-McKee equals the oracle's
(same deterministic rules) permutation for permutation, and e^H computed in RCM order and
mapped back (option reorder) meets the north-star parity against the oracle's e^H."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from synth import diagonal, laplacian_2d, make_config, random_banded, tridiag
from synth.configs import CSR

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


def _from_sp(A):
    A = A.tocsr()
    A.sort_indices()
    return CSR(A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64))


def shuffled(H, seed):
    q = np.random.default_rng(seed).permutation(H.n)
    A = sp.csr_matrix((H.val, H.col, H.rowptr), shape=(H.n, H.n))
    return _from_sp(A[q][:, q])


def _two_components():
    A = sp.block_diag([sp.csr_matrix((tridiag(30, 1.0, -2.0, 1.0).val, tridiag(30, 1.0, -2.0, 1.0).col,
                                      tridiag(30, 1.0, -2.0, 1.0).rowptr), shape=(30, 30)),
                       sp.identity(5), sp.csr_matrix(np.ones((4, 4)))])
    return shuffled(_from_sp(A), 2)


CASES = {
    "grid": lambda: shuffled(laplacian_2d(40, 30, 1.0), 5),
    "banded": lambda: shuffled(random_banded(600, 12, 0.3, 1.0, seed=4), 6),
    "structural": lambda: shuffled(make_config(3, scale_down=20), 7),
    "diagonal": lambda: diagonal(np.arange(1.0, 9.0)),
    "components": _two_components,
    "n1": lambda: diagonal(np.array([2.0])),
    # components above the host threshold (4096 nodes) run the device BFS / CM kernels
    "grid_device": lambda: shuffled(laplacian_2d(80, 70, 1.0), 8),
    "graph_mixed": lambda: __import__("synth").geometric_graph(20000, 6.0, 4.0, 3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_rcm_equals_oracle(B, name):
    H = CASES[name]()
    pg = B.sexpm_rcm(H.n, to_dev(H)).cpu().numpy()
    po = O.rcm(H)
    assert np.array_equal(pg, po)


@pytest.mark.parametrize("name", ["grid", "structural", "banded"])
def test_expm_reorder_parity(B, name):
    H = CASES[name]()
    rp, ci, va = to_dev(H)
    (a, b, c), st = B.expm(H.n, rp, ci, va, 1e-16, reorder=1)
    Eg = from_dev(H.n, a, b, c)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    # in RCM order the iterates are banded: T^_0's bandwidth is far below the shuffled one
    _, st0 = B.expm(H.n, rp, ci, va, 1e-16)
    assert 2 * st["sq_l1"][0] < st0["sq_l1"][0]
