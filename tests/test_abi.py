"""CPU-only checks of the C ABI boundary: the library builds, loads, exports every
symbol include/sexpm.h declares, struct layouts agree, the host-side partition / halo
logic (Lemma 3.1) is right, and compute calls fail loudly without a GPU."""
import os
import re

import numpy as np
import pytest

from paper_2110_04493_b200 import binding as B
from paper_2110_04493_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sexpm.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(sexpm_\w+)\(", src, re.M)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 15
    L = B.lib()
    for f in names:
        assert hasattr(L, f), f"{f} declared in sexpm.h but not exported"
    assert set(names) == set(B.EXPORTED)


def test_struct_layouts_match():
    B.lib()  # raises on mismatch
    o = B.sexpm_options_init()
    assert o.struct_size == B.C.sizeof(B.Options)
    assert o.plan_norm == 0 and o.normal == -1 and o.filter == 1 and o.e_r == 0.1
    assert o.m_cap == 120 and o.n_window == 50 and o.force_M == -1


def test_sass_is_sm100a():
    """The kernels are compiled for sm_100a (cuobjdump lists the arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("l1,l2", [(0, 0), (3, 5), (40, 40), (1000, 7)])
def test_halo_ranges_cover_needed_rows(world, l1, l2):
    n = 500
    bounds = B.sexpm_partition_rows(n, None, world)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
    assert all(b % 8 == 0 or b == n for b in bounds)  # whole 8-row blocks per rank
    for g in range(world):
        lo, hi = B.sexpm_halo_ranges(world, g, bounds, n, l1, l2)
        # Lemma 3.1's rows [r0 - l2, r1 + l1), widened to whole 8-row blocks (block kernel)
        need = set(range(max(0, ((bounds[g] - l2) // 8) * 8), min(n, -(-(bounds[g + 1] + l1) // 8) * 8)))
        have = set(range(bounds[g], bounds[g + 1]))
        for h in range(world):
            rng = set(range(lo[h], hi[h]))
            assert not (rng & have)
            assert rng <= set(range(bounds[h], bounds[h + 1]))
            have |= rng
        assert have == need


def test_partition_balances_work():
    rng = np.random.default_rng(0)
    w = rng.uniform(1, 3, 10_000)
    b = B.sexpm_partition_rows(len(w), w, 8)
    loads = [w[b[g]:b[g + 1]].sum() for g in range(8)]
    assert max(loads) <= 1.01 * (w.sum() / 8) + 8 * w.max()  # bounds on multiples of 8


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    o = B.sexpm_options_init()
    rp = np.array([0, 1], np.int64)
    ci = np.array([0], np.int32)
    va = np.array([1.0])
    H = B._csr_in(1, rp, ci, va, host=True)
    with pytest.raises(B.SexpmError):
        B.sexpm_plan_host(H, 1e-16, o)


def test_stream_handle_maps_default_stream_to_legacy_handle():
    """torch's default stream has handle 0, which sexpm_options.stream reads as "create a
    stream": the binding passes cudaStreamLegacy (1) instead; other handles pass through."""
    from types import SimpleNamespace
    assert B.stream_handle(SimpleNamespace(cuda_stream=0)) == B.CUDA_STREAM_LEGACY == 1
    assert B.stream_handle(SimpleNamespace(cuda_stream=0x7F00DEAD)) == 0x7F00DEAD
