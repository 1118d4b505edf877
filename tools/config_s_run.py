"""Config S (0.5 tridiag(1,-2,1), n = 2^25) once through the C ABI with the step log: the
SURVEY's HBM-roofline case (1D rows)."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2110_04493_b200 import binding as B
ns = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 25)
dev = torch.device("cuda", 0)
r_ = torch.arange(ns, device=dev, dtype=torch.int64)
cnt_ = torch.full((ns,), 3, dtype=torch.int64, device=dev)
cnt_[0] = 2
cnt_[-1] = 2
rp = torch.zeros(ns + 1, dtype=torch.int64, device=dev)
rp[1:] = torch.cumsum(cnt_, 0)
cols_ = torch.stack([r_ - 1, r_, r_ + 1], 1).reshape(-1)
vals_ = torch.tensor([0.5, -1.0, 0.5], dtype=torch.float64, device=dev).repeat(ns)
keep_ = (cols_ >= 0) & (cols_ < ns)
ci = cols_[keep_].to(torch.int32).contiguous()
va = vals_[keep_].contiguous()
for rep in range(2):
    p = B.Plan(ns, rp, ci, va, 1e-16)
    p.run_only()
    st = p.stats()
    p.close()
    N = int(st["N"])
    print(json.dumps({"rep": rep, "plan": st["ms_plan"], "taylor": st["ms_taylor"], "squaring": st["ms_squaring"],
                      "finalize": st["ms_finalize"], "total": st["ms_total"], "order_wait": st["ms_order_wait"],
                      "sq_kernel_ms": [float(x) for x in st["sq_kernel_ms"][1:N + 1]], "sym": int(st["sq_sym_used"]),
                      "order": int(st["sq_order_used"]), "window": int(st["taylor_window"])}), flush=True)
