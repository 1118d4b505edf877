"""Probe: 0.5 tridiag(1,-2,1) at several n on the symmetric path (sym used? nnz of E)."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2110_04493_b200 import binding as B
dev = torch.device("cuda", 0)
for lg in [int(x) for x in sys.argv[1:]]:
    ns = 1 << lg
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
    for sym in (-1, 0):
        p = B.Plan(ns, rp, ci, va, 1e-16, sym_squaring=sym)
        p.run_only()
        st = p.stats()
        p.close()
        print(json.dumps({"lg": lg, "sym_opt": sym, "sym": int(st["sq_sym_used"]), "nnz": int(st["nnz_out"]),
                          "sq_nnz0": int(st["sq_nnz"][0])}), flush=True)
