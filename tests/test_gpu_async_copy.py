"""sexpm_result_copy_async / sexpm_result_wait (include/sexpm.h): the detached result copied
on the library's copy stream while the next e^H runs must be the result sexpm_result_copy
delivers (bit for bit), and both must meet the north-star parity against the oracle."""
import numpy as np
import pytest

import oracle as O
from synth import CSR, make_config

from gpu_helpers import NTHREADS, last_tau, parity, to_dev

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


def _pinned(rows, nnz):
    import torch
    return (torch.empty(rows + 1, dtype=torch.int64).pin_memory(),
            torch.empty(max(nnz, 1), dtype=torch.int32).pin_memory(),
            torch.empty(max(nnz, 1), dtype=torch.float64).pin_memory())


def _plan_run(B, H, dev):
    import torch
    o = B.sexpm_options_init()
    o.stream = B.stream_handle(torch.cuda.current_stream())
    h = B.sexpm_plan(B._csr_in(H.n, *dev, 0, None), 1e-16, o)
    E = B.sexpm_run(h)
    return h, E


def test_async_copy_pipeline_matches_sync_copy_and_oracle(B):
    """Three consecutive e^H (configs 1, 2, 1): each result's copy is started, its plan
    destroyed and the next e^H planned and run before the copy is waited for."""
    import torch
    Hs = [make_config(1), make_config(2), make_config(1)]
    devs = [to_dev(H) for H in Hs]
    # the synchronous results first
    sync = []
    for H, d in zip(Hs, devs):
        h, E = _plan_run(B, H, d)
        bufs = _pinned(H.n, E.nnz)
        B.sexpm_result_copy(h, *(b.data_ptr() for b in bufs))
        st = B.sexpm_stats_get(h)
        B.sexpm_destroy(h)
        sync.append((bufs, E.nnz, st))
    pending = None
    got = []
    for H, d in zip(Hs, devs):
        h, E = _plan_run(B, H, d)
        if pending is not None:
            B.sexpm_result_wait(pending[0])
            got.append(pending[1:])
        bufs = _pinned(H.n, E.nnz)
        for b in bufs:
            b.fill_(-1)
        t = B.sexpm_result_copy_async(h, *(b.data_ptr() for b in bufs))
        # the plan has no result any more
        with pytest.raises(B.SexpmError) as ei:
            B.sexpm_result_copy(h, *(b.data_ptr() for b in bufs))
        assert ei.value.code == 8  # SEXPM_ESTATE
        B.sexpm_destroy(h)
        pending = (t, bufs, E.nnz)
    B.sexpm_result_wait(pending[0])
    got.append(pending[1:])
    B.sexpm_result_wait(None)  # no-op
    for H, (sb, snnz, st), (ab, annz) in zip(Hs, sync, got):
        assert snnz == annz
        assert torch.equal(sb[0], ab[0])
        assert torch.equal(sb[1][:snnz], ab[1][:annz])
        assert torch.equal(sb[2][:snnz], ab[2][:annz])
        Eo, tr = O.expm(H, 1e-16, nthreads=NTHREADS)
        Eg = CSR(H.n, ab[0].numpy().copy(), ab[1][:annz].numpy().copy(), ab[2][:annz].numpy().copy())
        ok, res = parity(Eg, Eo, last_tau(tr, st))
        assert ok, res


def test_async_copy_errors_and_device_destination(B):
    """No result -> SEXPM_ESTATE; null ticket -> SEXPM_EINVAL; a DEVICE destination receives
    the result sexpm_result_copy delivers."""
    import ctypes as C
    import torch
    H = make_config(1)
    d = to_dev(H)
    o = B.sexpm_options_init()
    o.stream = B.stream_handle(torch.cuda.current_stream())
    h = B.sexpm_plan(B._csr_in(H.n, *d, 0, None), 1e-16, o)
    bufs = _pinned(H.n, 1)
    with pytest.raises(B.SexpmError) as ei:
        B.sexpm_result_copy_async(h, *(b.data_ptr() for b in bufs))
    assert ei.value.code == 8
    E = B.sexpm_run(h)
    assert B.lib().sexpm_result_copy_async(h, C.c_void_p(bufs[0].data_ptr()), None, None, None) == 1
    ref = [torch.empty(H.n + 1, dtype=torch.int64, device="cuda"),
           torch.empty(E.nnz, dtype=torch.int32, device="cuda"),
           torch.empty(E.nnz, dtype=torch.float64, device="cuda")]
    B.sexpm_result_copy(h, *(t.data_ptr() for t in ref))
    out = [torch.empty_like(t) for t in ref]
    t = B.sexpm_result_copy_async(h, *(x.data_ptr() for x in out))
    B.sexpm_destroy(h)
    B.sexpm_result_wait(t)
    for a, b in zip(ref, out):
        assert torch.equal(a, b)


def test_async_copy_pageable_and_unaligned_destinations(B):
    """Pageable host arrays (copy-engine path) and pinned arrays that are not 16-byte aligned
    (k_copy_out refuses them: copy-engine path) receive the result of sexpm_result_copy."""
    import torch
    H = make_config(2)
    d = to_dev(H)
    res = []
    for kind in ("sync", "pageable", "unaligned"):
        h, E = _plan_run(B, H, d)
        if kind == "sync":
            bufs = _pinned(H.n, E.nnz)
            B.sexpm_result_copy(h, *(b.data_ptr() for b in bufs))
            out = [bufs[0].numpy().copy(), bufs[1][:E.nnz].numpy().copy(), bufs[2][:E.nnz].numpy().copy()]
        elif kind == "pageable":
            out = [np.full(H.n + 1, -1, np.int64), np.full(E.nnz, -1, np.int32), np.full(E.nnz, -1.0)]
            t = B.sexpm_result_copy_async(h, *(a.ctypes.data for a in out))
            B.sexpm_result_wait(t)
        else:
            raw = (torch.empty(H.n + 2, dtype=torch.int64).pin_memory(),
                   torch.empty(E.nnz + 1, dtype=torch.int32).pin_memory(),
                   torch.empty(E.nnz + 1, dtype=torch.float64).pin_memory())
            views = [r[1:] for r in raw]  # offsets of 8, 4 and 8 bytes
            assert all(v.data_ptr() % 16 != 0 for v in views)
            t = B.sexpm_result_copy_async(h, *(v.data_ptr() for v in views))
            B.sexpm_result_wait(t)
            out = [v.numpy().copy() for v in views]
        B.sexpm_destroy(h)
        res.append(out)
    for out in res[1:]:
        for a, b in zip(res[0], out):
            assert np.array_equal(a, b)
