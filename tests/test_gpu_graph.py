"""N4: unstructured sparse graphs as a second workload -- communicability
e^{beta A} of a random geometric graph in random node order (synth.geometric_graph), on the
GPU as given and with the device RCM (option reorder), against the oracle."""
import numpy as np
import pytest

import oracle as O
from synth import geometric_graph

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


@pytest.mark.parametrize("reorder", [0, 1])
@pytest.mark.parametrize("n,seed", [(3000, 1), (800, 2)])
def test_geometric_graph_parity(B, n, seed, reorder):
    H = geometric_graph(n, 6.0, 4.0, seed)
    rp, ci, va = to_dev(H)
    (a, b, c), st = B.expm(H.n, rp, ci, va, 1e-16, reorder=reorder)
    Eg = from_dev(H.n, a, b, c)
    Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
    assert (st["M"], st["N"]) == (tr["M"], tr["N"])
    ok, res = parity(Eg, Eo, last_tau(tr, st))
    assert ok, res
