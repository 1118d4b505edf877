"""GPU parity of N1 apply: Y = R^steps X through the C ABI
(sexpm_spmm / sexpm_apply) vs the oracle's or_spmm on the same seeded inputs."""
import numpy as np
import pytest

import oracle as O
from synth import csr_to_dense, dense_to_csr, make_config, neumann_laplacian_2d, random_banded

from gpu_helpers import NTHREADS, to_dev

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def B():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_04493_b200 import binding
    from paper_2110_04493_b200.build import build
    build()
    binding.lib()
    return binding


def _rand_csr(n, bw, dens, seed, empty_rows=()):
    A = csr_to_dense(random_banded(n, bw, dens, 1.0, seed))
    for r in empty_rows:
        A[r, :] = 0
    return dense_to_csr(A)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8, 9, 16, 17, 31, 32, 33, 64, 100, 129, 300])
def test_spmm_vs_oracle(B, m):
    """Ragged rows (bandwidth 40, 30 % fill, > 32 entries in most rows), empty rows; m over
    every lane-group width and ragged column tiles.  m > 16: each lane adds its columns in
    the oracle's order -> bit-identical; m <= 16: fixed tree over lane groups -> within the
    running-sum bound nnz(row) u (|A| |X|)."""
    import torch
    n = 533
    A = _rand_csr(n, 40, 0.3, 70 + m, empty_rows=(0, 17, 532))
    X = np.random.default_rng(m).standard_normal((n, m))
    Yg = B.sexpm_spmm(n, to_dev(A), torch.from_numpy(X).cuda()).cpu().numpy()
    Yo = O.spmm(A, X)
    if m > 16:
        assert np.array_equal(Yg, Yo)
    else:
        bound = 2 * 81 * U * (np.abs(csr_to_dense(A)) @ np.abs(X))
        assert np.all(np.abs(Yg - Yo) <= bound + 1e-300)
    assert np.all(Yg[[0, 17, 532]] == 0.0)


def test_spmm_strided_and_vector(B):
    """Row strides ldx > m, ldy > m (column slices of wider tensors) and a 1-D X."""
    import torch
    n = 300
    A = _rand_csr(n, 9, 0.5, 5)
    Xw = torch.from_numpy(np.random.default_rng(1).standard_normal((n, 50))).cuda()
    X = Xw[:, 3:43]
    Yw = torch.full((n, 60), 7.0, dtype=torch.float64, device="cuda")
    Y = Yw[:, 10:50]
    B.sexpm_spmm(n, to_dev(A), X, Y)
    assert np.array_equal(Y.cpu().numpy(), O.spmm(A, X.cpu().numpy()))
    assert torch.all(Yw[:, :10] == 7.0) and torch.all(Yw[:, 50:] == 7.0)
    x = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()
    y = B.sexpm_spmm(n, to_dev(A), x)
    assert y.shape == (n,)
    yo = O.spmm(A, x.cpu().numpy())
    assert np.all(np.abs(y.cpu().numpy() - yo) <= 64 * U * (np.abs(csr_to_dense(A)) @ np.abs(x.cpu().numpy())))


@pytest.mark.parametrize("steps", [1, 2, 5])
def test_apply_config2_vs_oracle(B, steps):
    """Y = E^steps X with the GPU's E of BASELINE config 2 against the oracle's E applied by
    the oracle: E agrees within the north-star parity (1e-11 max|E|), so Y agrees within
    steps * 1e-11 * max|E| * max row sum of |E|^(steps-1) * sum|X| per row."""
    import torch
    H = make_config(2)
    rp, ci, va = to_dev(H)
    P = B.Plan(H.n, rp, ci, va, 1e-16)
    P.run()
    X = np.random.default_rng(steps).standard_normal((H.n, 40))
    Yg = P.apply(torch.from_numpy(X).cuda(), steps=steps).cpu().numpy()
    P.close()
    Eo, _ = O.expm(H, 1e-16, nthreads=NTHREADS)
    Yo = O.spmm(Eo, X, steps=steps)
    Ed = np.abs(Eo.val).max()
    rowsum = np.add.reduceat(np.abs(Eo.val), Eo.rowptr[:-1]).max()
    nnz_row = np.diff(Eo.rowptr).max()
    tol = steps * 1e-11 * Ed * nnz_row * rowsum ** (steps - 1) * np.abs(X).max()
    assert np.abs(Yg - Yo).max() <= tol


def test_apply_zero_row_sum_generator(B):
    """e^H 1 = 1 for a Neumann Laplacian: ten GPU steps keep the ones vector."""
    import torch
    H = neumann_laplacian_2d(40, 30, 0.7, seed=3)
    rp, ci, va = to_dev(H)
    P = B.Plan(H.n, rp, ci, va, 1e-16)
    P.run()
    y = P.apply(torch.ones(H.n, dtype=torch.float64, device="cuda"), steps=10)
    P.close()
    assert (y - 1.0).abs().max().item() <= 1e-12


def test_apply_errors(B):
    import torch
    H = make_config(1)
    rp, ci, va = to_dev(H)
    P = B.Plan(H.n, rp, ci, va, 1e-16)
    X = torch.ones((H.n, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(B.SexpmError, match="ESTATE"):
        P.apply(X)  # before run
    P.run()
    with pytest.raises(B.SexpmError, match="EINVAL"):
        P.apply(X, steps=0)
    with pytest.raises(B.SexpmError, match="EINVAL"):
        P.apply(X, Y=X)  # overlap
    Z = torch.empty((H.n, 0), dtype=torch.float64, device="cuda")
    assert P.apply(Z).shape == (H.n, 0)  # m = 0: nothing to do
    P.close()
