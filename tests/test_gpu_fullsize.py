"""Full-size checks at BASELINE.json's largest configs, in the launch configuration
bench.py times (default options, 1-norm plan, eps_tol = 1e-16).

Config 5 (uniform 2D Dirichlet heat, n = 1449^2) has a closed form that holds at any
size: H = r L (x) I + I (x) r L, so e^H = e^{rL} (x) e^{rL} with the 1D factor given by
the Bessel-image heat kernel (tests/refs.py).  Sampled rows of the GPU result are compared
entry by entry with it, within the method's own error budget."""
import numpy as np
import pytest

from synth import make_config

import refs
from gpu_helpers import from_dev, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    assert torch.cuda.is_available()
    from paper_2110_04493_b200 import binding
    from paper_2110_04493_b200.build import build
    build()
    return binding


def _rows(E, rows):
    out = []
    for r in rows:
        a, b = E.rowptr[r], E.rowptr[r + 1]
        out.append((E.col[a:b], E.val[a:b]))
    return out


def test_config5_kronecker_closed_form(B):
    g = 1449
    H = make_config(5)
    rp, ci, va = to_dev(H)
    (erp, eci, eva), st = B.expm(H.n, rp, ci, va, 1e-16)
    E = from_dev(H.n, erp, eci, eva)
    rng = np.random.default_rng(0)
    rows = np.concatenate([[0, 1, g - 1, g, H.n // 2, H.n - 1], rng.integers(0, H.n, 60)])
    rN = st["r0"] * 2.0 ** st["N"]
    worst = 0.0
    for r in rows:
        a, b = E.rowptr[r], E.rowptr[r + 1]
        cols = E.col[a:b]
        ex = refs.heat2d_entry(g, g, 0.5, r, cols)
        worst = max(worst, np.abs(E.val[a:b] - ex).max())
        # entries the filter dropped: the exact value there is below the final thresholds
        x, y = divmod(int(r), g)
        nb = np.array([(x + dx) * g + (y + dy) for dx in range(-40, 41) for dy in range(-40, 41)
                       if 0 <= x + dx < g and 0 <= y + dy < g])
        missing = np.setdiff1d(nb, cols)
        if len(missing):
            assert np.abs(refs.heat2d_entry(g, g, 0.5, r, missing)).max() < 1e-12
    # max |E| = E_ii ~ 0.1: forward error r_N plus filter budget plus rounding
    assert worst <= 1e-13, worst
    assert st["sq_nnz"][st["N"]] > 0 and st["gpu_launches"] > 0
