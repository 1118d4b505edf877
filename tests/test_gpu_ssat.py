"""GPU parity of the SSAT baseline (Table 1's SSAT column):
E_0 = I + T^_0, E_i = E_{i-1}^2 on the device (K3b / K5d kernels, no filter) vs the
oracle's SSAT on the same inputs.  Unfiltered, every product is accumulated in the oracle's
order, so E must match bit for bit; the filtered PIM on the same matrices is far more
accurate (Table 1)."""
import numpy as np
import pytest

import oracle as O
from synth import csr_to_dense, dense_to_csr, make_config, random_banded

import refs
from gpu_helpers import NTHREADS, from_dev, to_dev

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


def _both(B, H, **opts):
    rp, ci, va = to_dev(H)
    (erp, eci, eva), st = B.expm(H.n, rp, ci, va, 1e-16, **opts)
    oo = {k: v for k, v in opts.items() if k not in ("kernel", "exact_products")}
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS, **oo)
    return from_dev(H.n, erp, eci, eva), st, Eo, tr


CASES = [("table1_%d" % k, lambda k=k: dense_to_csr(refs.table1_matrices()[k]), "fro") for k in range(1, 6)] + [
    ("config1", lambda: make_config(1), "one"),
    ("config2_30x30", lambda: make_config(2, scale_down=30), "one"),
    ("banded_nonsym", lambda: random_banded(700, 5, 0.6, 0.4, seed=9), "one"),
]


@pytest.mark.parametrize("name,make,norm", CASES, ids=[c[0] for c in CASES])
def test_ssat_bit_exact(B, name, make, norm):
    H = make()
    Eg, st, Eo, tr = _both(B, H, plan_norm=norm, filter=False, ssat=True, exact_products=1)
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    assert np.array_equal(Eg.rowptr, Eo.rowptr) and np.array_equal(Eg.col, Eo.col)
    assert np.array_equal(Eg.val, Eo.val)


def test_ssat_vs_pim_accuracy_on_gpu(B):
    """H_1 (N = 20): the GPU's SSAT loses ~5 digits, its PIM stays at the rounding level."""
    H = dense_to_csr(refs.table1_matrices()[1])
    Ex = refs.table1_exact(1)
    rp, ci, va = to_dev(H)
    (a, b, c), _ = B.expm(H.n, rp, ci, va, 1e-16, plan_norm="fro", filter=False, ssat=True)
    (d, e, f), _ = B.expm(H.n, rp, ci, va, 1e-16, plan_norm="fro")
    es = np.linalg.norm(csr_to_dense(from_dev(H.n, a, b, c)) - Ex) / np.linalg.norm(Ex)
    ep = np.linalg.norm(csr_to_dense(from_dev(H.n, d, e, f)) - Ex) / np.linalg.norm(Ex)
    assert ep <= 2e-15 and es >= 1e-11


def test_ssat_output_T_rejected(B):
    H = make_config(1)
    rp, ci, va = to_dev(H)
    with pytest.raises(B.SexpmError, match="EINVAL"):
        B.expm(H.n, rp, ci, va, 1e-16, ssat=True, output_T=True)
