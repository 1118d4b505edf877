"""North-star parity of the GPU path against the CPU oracle on a large instance of a
BASELINE config law (default: config 5's uniform 2D Dirichlet heat, r = 0.5, on a G x G
grid), all three criteria, with timings and the SHA-256 of the oracle's CSR.  Run on the GPU
box (the oracle uses every host core):

    python tools/oracle_parity_report.py --grid 512 > profiles/r02_parity_config5_law_512.json
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--grid", type=int, default=512)
    ap.add_argument("--eps-tol", type=float, default=1e-16)
    args = ap.parse_args()
    import numpy as np
    import torch
    import oracle as O
    from gpu_helpers import NTHREADS, from_dev, last_tau, parity, to_dev
    from paper_2110_04493_b200 import binding as B
    from synth import make_config
    H = make_config(args.config, scale_down=args.grid)
    rp, ci, va = to_dev(H)
    B.expm(H.n, rp, ci, va, args.eps_tol)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    (erp, eci, eva), st = B.expm(H.n, rp, ci, va, args.eps_tol)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    Eg = from_dev(H.n, erp, eci, eva)
    t0 = time.perf_counter()
    Eo, tr = O.expm(H, args.eps_tol, nthreads=NTHREADS)
    t_cpu = time.perf_counter() - t0
    h = hashlib.sha256()
    for a in (Eo.rowptr, Eo.col, Eo.val):
        h.update(np.ascontiguousarray(a).tobytes())
    tau = last_tau(tr, st)
    ok, res = parity(Eg, Eo, tau)
    out = {"workload": f"config {args.config} law on a {args.grid}x{args.grid} grid", "n": H.n,
           "eps_tol": args.eps_tol, "M": int(st["M"]), "N": int(st["N"]),
           "plan_equal": (int(st["M"]), int(st["N"])) == (tr["M"], tr["N"]),
           "nnz_E_gpu": int(Eg.nnz), "nnz_E_oracle": int(Eo.nnz),
           "criteria": {"max_abs_err_over_max": res["rel"], "max_abs_err_bound": 1e-11,
                        "jaccard": res["jaccard"], "jaccard_bound": 0.999,
                        "positions_one_side": res["n_only"], "symdiff_max": res["symdiff_max"],
                        "tau_N": tau, "symdiff_bound": 10 * tau},
           "pass": bool(ok), "gpu_expm_s": t_gpu, "oracle_s": t_cpu, "oracle_threads": NTHREADS,
           "oracle_csr_sha256": h.hexdigest()}
    print(json.dumps(out, default=float))


if __name__ == "__main__":
    main()
