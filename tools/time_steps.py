import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2110_04493_b200 import binding as B
from synth import make_config
H = make_config(5)
dev = torch.device("cuda", 0)
rp, ci, va = (torch.from_numpy(x).to(dev) for x in (H.rowptr, H.col, H.val))
stream = torch.cuda.current_stream()
for it in range(int(os.environ.get("STEPS", "5"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = B.Plan(H.n, rp, ci, va, 1e-16, stream=stream)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    p.run_only()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    st = p.stats()
    p.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"plan {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} close {1e3*(t3-t2):.1f} | dev total {st['ms_total']:.1f} taylor {st['ms_taylor']:.1f} sq {st['ms_squaring']:.1f} wait {st['ms_order_wait']:.1f} misses {st['cache_misses']}", flush=True)
