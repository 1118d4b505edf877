"""Pipelined e2e probe (config 5): consecutive e^H with sexpm_result_copy_async; prints the
per-step wall time.  SEXPM_COPY_CHUNK_MB sets the copy chunk."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2110_04493_b200 import binding as B
from synth import make_config
H = make_config(int(os.environ.get("CONFIG", "5")))
n = H.n
hrp, hci, hva = (torch.from_numpy(x).pin_memory() for x in (H.rowptr, H.col, H.val))
stream = torch.cuda.current_stream()
sets = None
def one(i, pending):
    o = B.sexpm_options_init(); o.stream = B.stream_handle(stream)
    Hin = B._csr_in(n, hrp.numpy(), hci.numpy(), hva.numpy(), 0, n, host=True)
    t0 = time.perf_counter()
    h = B.sexpm_plan_host(Hin, 1e-16, o)
    t1 = time.perf_counter()
    E = B.sexpm_run(h)
    t2 = time.perf_counter()
    st = B.sexpm_stats_get(h)
    print(f"   misses {st['cache_misses']} releases {st['cache_releases']} allocated {st['cache_bytes_allocated']/1e9:.1f} GB cached {st['cache_bytes_cached']/1e9:.1f} GB sym {st['sq_sym_used']} | dev ms: plan {st['ms_plan']:.1f} taylor {st['ms_taylor']:.1f} sq {st['ms_squaring']:.1f} fin {st['ms_finalize']:.1f} | taylor terms {[round(x,1) for x in st['taylor_ms'][2:20]]} sq {[round(x,1) for x in st['sq_ms'][1:3]]}")
    return h, E, (t1 - t0, t2 - t1)
h, E, _ = one(0, None)
cap = int(E.nnz * 1.01) + 1024
sets = [(torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(cap, dtype=torch.int32).pin_memory(),
         torch.empty(cap, dtype=torch.float64).pin_memory()) for _ in range(2)]
B.sexpm_destroy(h)
pending = None
K = int(os.environ.get("STEPS", "6"))
torch.cuda.synchronize()
T0 = time.perf_counter()
for i in range(K):
    ta = time.perf_counter()
    h, E, (tp, tr) = one(i, pending)
    tb = time.perf_counter()
    if pending is not None:
        B.sexpm_result_wait(pending)
    tc = time.perf_counter()
    bs = sets[i % 2]
    pending = B.sexpm_result_copy_async(h, bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr())
    B.sexpm_destroy(h)
    td = time.perf_counter()
    print(f"step {i}: plan {1e3*tp:.1f} run {1e3*tr:.1f} wait {1e3*(tc-tb):.1f} issue+destroy {1e3*(td-tc):.1f} total {1e3*(td-ta):.1f}", flush=True)
B.sexpm_result_wait(pending)
torch.cuda.synchronize()
print(f"{K} steps in {time.perf_counter()-T0:.3f} s -> {K/(time.perf_counter()-T0):.3f} e^H/s")
