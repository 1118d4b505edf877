"""While the library's copy worker moves config 5's E, time small operations on the plan's stream."""
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
o = B.sexpm_options_init(); o.stream = stream.cuda_stream
h = B.sexpm_plan(B._csr_in(n, rp, ci, va, 0, None), 1e-16, o)
E = B.sexpm_run(h)
bufs = (torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(E.nnz, dtype=torch.int32).pin_memory(),
        torch.empty(E.nnz, dtype=torch.float64).pin_memory())
import ctypes as C
rt = C.CDLL('libcudart.so.12')
hv = C.c_double()
def t(f, name):
    t0 = time.perf_counter(); f(); stream.synchronize()
    return f"{name} {1e3*(time.perf_counter()-t0):.2f}"
torch.cuda.synchronize()
T0 = time.perf_counter()
tk = B.sexpm_result_copy_async(h, *(b.data_ptr() for b in bufs))
if os.environ.get("DESTROY"):
    B.sexpm_destroy(h); h = None
s2 = torch.cuda.Stream(priority=int(os.environ.get('PRIO', '0')))
def t2(f, name):
    t0 = time.perf_counter(); f(); s2.synchronize()
    return f"{name} {1e3*(time.perf_counter()-t0):.2f}"
for i in range(8):
    time.sleep(0.01)
    with torch.cuda.stream(s2):
        print(f"t={1e3*(time.perf_counter()-T0):6.1f} ms [fresh stream]: " + " | ".join([
            t2(lambda: small.add_(1.0), "kernel"),
            t2(lambda: rt.cudaMemsetAsync(C.c_void_p(small.data_ptr()), 0, 4, C.c_void_p(s2.cuda_stream)), "cudaMemsetAsync"),
            t2(lambda: rt.cudaMemcpyAsync(C.byref(hv), C.c_void_p(small.data_ptr()), 8, 2, C.c_void_p(s2.cuda_stream)), "D2H to stack")]), flush=True)
for i in range(4):
    print(f"t={1e3*(time.perf_counter()-T0):6.1f} ms: " + " | ".join([
        t(lambda: small.add_(1.0), "kernel"),
        t(lambda: small.cpu(), "D2H small pageable"),
        t(lambda: din.copy_(hin, non_blocking=True), "H2D 84 MB"),
        t(lambda: small.zero_(), "fill kernel"),
        t(lambda: rt.cudaMemsetAsync(C.c_void_p(small.data_ptr()), 0, 4, C.c_void_p(0)), "cudaMemsetAsync"),
        t(lambda: rt.cudaMemcpyAsync(C.byref(hv), C.c_void_p(small.data_ptr()), 8, 2, C.c_void_p(0)), "D2H to stack")]), flush=True)
    time.sleep(0.015)
B.sexpm_result_wait(tk)
print(f"copy done at {1e3*(time.perf_counter()-T0):.1f} ms")
if h is not None:
    B.sexpm_destroy(h)
