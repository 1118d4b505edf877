"""SURVEY's proposed config S (HBM-roofline validation): 0.5 tridiag(1,-2,1), n = 2^26, one-norm
plan, eps_tol 1e-16.  One e^H after a warm-up; prints phases and the Taylor kernel's
compulsory HBM throughput (not part of the default bench)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2110_04493_b200 import binding as B


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
    B.lib()
    dev = torch.device("cuda", 0)
    # tridiag(1,-2,1) * 0.5 in CSR (built on the device: 3 entries per row, 2 at the ends)
    r = torch.arange(n, device=dev, dtype=torch.int64)
    cnt = torch.full((n,), 3, dtype=torch.int64, device=dev)
    cnt[0] = 2
    cnt[-1] = 2
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(cnt, 0)
    cols = torch.stack([r - 1, r, r + 1], 1).reshape(-1)
    vals = torch.tensor([0.5, -1.0, 0.5], dtype=torch.float64, device=dev).repeat(n)
    keep = (cols >= 0) & (cols < n)
    ci = cols[keep].to(torch.int32).contiguous()
    va = vals[keep].contiguous()
    del cols, vals, keep, r, cnt
    out = {}
    for rep in range(2):
        p = B.Plan(n, rp, ci, va, 1e-16)
        t0 = time.perf_counter()
        p.run_only()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = p.stats()
        p.close()
    M, N = int(st["M"]), int(st["N"])
    ty = [i for i in range(2, M + 1) if st["taylor_numeric_ms"][i] > 0]
    by = sum(float(st["taylor_numeric_bytes"][i]) for i in ty)
    ms = sum(float(st["taylor_numeric_ms"][i]) for i in ty)
    out = {"workload": f"config S: 0.5 tridiag(1,-2,1), n = {n}", "M": M, "N": N,
           "nnz_E": int(st["nnz_out"]), "phase_ms": {k: float(st["ms_" + k]) for k in ("plan", "taylor", "squaring", "finalize")},
           "wall_s": wall, "taylor_kernel_ms": ms, "taylor_kernel_compulsory_gbs": by / ms / 1e6,
           "sq_kernel_ms": [float(x) for x in st["sq_kernel_ms"][1:N + 1]],
           "sq_numeric_gbs_compulsory": [float(st["sq_numeric_bytes"][i]) / float(st["sq_numeric_ms"][i]) / 1e6 for i in range(1, N + 1)],
           "device_gb_allocated": float(st["cache_bytes_allocated"]) / 1e9, "retries": int(st["retries"])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
