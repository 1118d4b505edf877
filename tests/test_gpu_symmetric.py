"""The symmetric squaring path (option sym_squaring, reading R21): for a bit-exactly
symmetric H the squarings compute only the output blocks J >= I of T~ = 2T + T^2 (K3s) and
assemble every row from those blocks and their transposes (K3c / K3a).  Checked against the
oracle with the north-star criteria, against the full product (sym_squaring = 0), for exact
symmetry of E, and for the cases the block assembly must get right: ragged last block rows,
empty diagonal blocks, non-stencil (non-window) Taylor phases, 3D rows (the long-list launch
shape), n = 1, diagonal and zero matrices, and non-symmetric H (path not taken)."""
import numpy as np
import pytest

import oracle as O
from synth import (diagonal, geometric_graph, laplacian_2d, laplacian_3d, make_config,
                   random_banded, tridiag)
from synth.configs import coo_to_csr

from gpu_helpers import NTHREADS, from_dev, last_tau, parity, scipy_of, to_dev

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


def run(B, H, **opts):
    rp, ci, va = to_dev(H)
    (a, b, c), st = B.expm(H.n, rp, ci, va, 1e-16, **opts)
    return from_dev(H.n, a, b, c), st


def exactly_symmetric(E):
    S = scipy_of(E)
    D = (S - S.T).tocsr()
    D.eliminate_zeros()
    return D.nnz == 0


def bipartite_sym(n, seed):
    """[[0, C], [C^T, 0]] with a sparse banded C: a symmetric H whose powers alternate
    between the diagonal and off-diagonal blocks (iterates with empty diagonal 8x8 blocks
    appear in the Taylor terms)."""
    rng = np.random.default_rng(seed)
    h = n // 2
    r, c, v = [], [], []
    for i in range(h):
        for j in range(max(0, i - 3), min(h, i + 4)):
            if rng.random() < 0.6:
                x = rng.uniform(-1.0, 1.0)
                r += [i, h + j]
                c += [h + j, i]
                v += [x, x]
    return coo_to_csr(n, np.array(r), np.array(c), np.array(v))


CASES = {
    "config1": lambda: make_config(1),
    "config2": lambda: make_config(2),
    "config5_law_96": lambda: make_config(5, scale_down=96),
    "config2_law_37_ragged": lambda: laplacian_2d(37, 29, 1.0, "pm10", 5),  # n = 1073: ragged
    "config4_law_12": lambda: laplacian_3d(12, 12, 12, 0.25, "u0812", 7),
    "graph_1500": lambda: geometric_graph(1500, 6.0, 4.0, 3),
    "banded_sym_203": lambda: random_banded(203, 9, 0.5, 0.6, 11, symmetric=True),
    "bipartite_402": lambda: bipartite_sym(402, 4),
}


@pytest.mark.parametrize("name", list(CASES))
def test_symmetric_path_vs_oracle(B, name):
    H = CASES[name]()
    Eg, st = run(B, H)
    N = int(st["N"])
    assert st["sq_sym_used"] == N, (name, st["sq_sym_used"], N)  # the path ran every squaring
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, (name, res)
    assert exactly_symmetric(Eg), name  # mirrored blocks: E = E^T bit for bit


@pytest.mark.parametrize("name", ["config2", "config5_law_96", "config4_law_12", "graph_1500"])
def test_symmetric_path_vs_full_product(B, name):
    """The two squaring paths differ only in summation order (and T^_0's mirror, R21)."""
    H = CASES[name]()
    Es, ss = run(B, H)
    Ef, sf = run(B, H, sym_squaring=0)
    assert sf["sq_sym_used"] == 0 and ss["sq_sym_used"] == int(ss["N"])
    N = int(ss["N"])
    assert N >= 1
    ok, res = parity(Es, Ef, max(float(ss["sq_tau"][N]), float(sf["sq_tau"][N])), rel_tol=1e-13)
    assert ok, (name, res)
    # the filter's decisions agree (kept counts within the entries near tau)
    assert abs(int(ss["sq_nnz"][int(ss["N"])]) - int(sf["sq_nnz"][int(sf["N"])])) <= 1e-4 * Ef.rowptr[-1] + 8


def test_symmetric_block_products_halved(B):
    """K3s executes about half the 8x8x8 block products of the full kernel."""
    H = make_config(5, scale_down=128)
    _, ss = run(B, H)
    _, sf = run(B, H, sym_squaring=0)
    N = int(ss["N"])
    bs = float(np.sum(ss["sq_block_products"][1:N + 1]))
    bf = float(np.sum(sf["sq_block_products"][1:N + 1]))
    assert 0.45 * bf <= bs <= 0.6 * bf, (bs, bf)


@pytest.mark.parametrize("H", [
    lambda: make_config(3, scale_down=12),                         # structural: non-symmetric
    lambda: random_banded(150, 6, 0.5, 0.5, 3, symmetric=False),  # generic non-symmetric
], ids=["structural", "nonsym_banded"])
def test_nonsymmetric_not_taken(B, H):
    H = H()
    Eg, st = run(B, H)
    assert st["sq_sym_used"] == 0
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res


@pytest.mark.parametrize("H", [
    lambda: diagonal([0.3]),                                     # n = 1
    lambda: diagonal(np.linspace(-2.0, 1.5, 19)),                # diagonal, ragged
    lambda: tridiag(9, 0.7, -1.4, 0.7),                          # n = 9: one row in block 1
    lambda: coo_to_csr(16, np.array([0, 8]), np.array([8, 0]), np.array([1.25, 1.25])),
], ids=["n1", "diag19", "tridiag9", "offdiag_blocks16"])
def test_symmetric_edge_cases(B, H):
    H = H()
    Eg, st = run(B, H)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    assert exactly_symmetric(Eg)


def test_symmetric_option_off(B):
    H = make_config(1)
    _, st = run(B, H, sym_squaring=0)
    assert st["sq_sym_used"] == 0


@pytest.mark.parametrize("fail", [1, 2, 4, 6])
def test_symmetric_fallbacks(B, fail, monkeypatch):
    """The symmetric product refused at chosen squarings (test hook SEXPM_SYM_FAIL, a bitmask):
    squaring 1 with T^_0 still in index order relabels it and runs the full product; a later
    squaring whose input is in block form converts the view to CSR (k_bsr_to_csr) first.  The
    result keeps parity with the oracle and the other squarings stay on the symmetric path."""
    H = make_config(2)  # N = 4: three block-form hand-offs
    monkeypatch.setenv("SEXPM_SYM_FAIL", str(fail))
    Eg, st = run(B, H)
    monkeypatch.delenv("SEXPM_SYM_FAIL")
    N = int(st["N"])
    assert N == 4
    assert st["sq_sym_used"] == N - bin(fail).count("1")
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, (fail, res)


def test_symmetric_wide_union(B, monkeypatch):
    """K3c's first launch uses small candidate bitmaps; block rows whose union is wider set flag
    32 and the count runs again with the widest (test hook SEXPM_K3C_WORDS shrinks the first
    bitmaps to 2 words so that every 2D block row takes that path).  Parity with the oracle."""
    H = make_config(5, scale_down=96)
    monkeypatch.setenv("SEXPM_K3C_WORDS", "2")
    Eg, st = run(B, H)
    monkeypatch.delenv("SEXPM_K3C_WORDS")
    assert st["sq_sym_used"] == int(st["N"]) >= 1
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    assert exactly_symmetric(Eg)


@pytest.mark.parametrize("opts", [dict(output_T=True), dict(filter=0), dict(threshold_mode=1),
                                  dict(plan_norm="fro")],
                         ids=["output_T", "unfiltered", "abs_threshold", "fro_plan"])
def test_symmetric_path_options(B, opts):
    """The symmetric path (with its block-form hand-offs: config 2 squares 4+ times) under the
    options that change what the squarings filter or return: T^_N instead of E, the unfiltered
    PIM, the printed absolute budget, the Frobenius plan -- all against the oracle."""
    # (the unfiltered oracle is slow on config 2: a 40 x 40 grid of the same law there)
    H = laplacian_2d(40, 40, 1.0, "pm10", 5) if opts.get("filter") == 0 else make_config(2)
    Eg, st = run(B, H, **opts)
    N = int(st["N"])
    assert N >= 3 and st["sq_sym_used"] == N
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS, **opts)
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
    assert exactly_symmetric(Eg)
