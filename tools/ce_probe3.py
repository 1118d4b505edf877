import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2110_04493_b200 import binding as B
from synth import make_config
H = make_config(5)
n = H.n
dev = torch.device("cuda", 0)
rp, ci, va = (torch.from_numpy(x).to(dev) for x in (H.rowptr, H.col, H.val))
hin = torch.from_numpy(H.val).pin_memory()
din = torch.empty_like(hin, device=dev)
small = torch.ones(8, dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream()
def t(f, name):
    t0 = time.perf_counter(); f(); stream.synchronize()
    return f"{name} {1e3*(time.perf_counter()-t0):.2f}"
sets = None
pending = None
mode = os.environ.get("MODE", "ops")
for i in range(5):
    o = B.sexpm_options_init(); o.stream = stream.cuda_stream
    t0 = time.perf_counter()
    h = B.sexpm_plan(B._csr_in(n, rp, ci, va, 0, None), 1e-16, o)
    t1 = time.perf_counter()
    E = B.sexpm_run(h)
    t2 = time.perf_counter()
    if sets is None:
        sets = [(torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(E.nnz, dtype=torch.int32).pin_memory(),
                 torch.empty(E.nnz, dtype=torch.float64).pin_memory()) for _ in range(2)]
    if pending is not None:
        B.sexpm_result_wait(pending)
    t3 = time.perf_counter()
    pending = B.sexpm_result_copy_async(h, *(b.data_ptr() for b in sets[i % 2]))
    if mode != "nodestroy_first":
        B.sexpm_destroy(h)
    t4 = time.perf_counter()
    msg = ""
    if mode == "ops":
        msg = " | ".join([t(lambda: small.cpu(), "D2H small"), t(lambda: din.copy_(hin, non_blocking=True), "H2D"),
                          t(lambda: small.add_(1.0), "kernel")])
    print(f"step {i}: plan(device H) {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} wait {1e3*(t3-t2):.1f} issue+destroy {1e3*(t4-t3):.1f} {msg}", flush=True)
    if mode == "nodestroy_first":
        hold = h
B.sexpm_result_wait(pending)
