"""Run one e^H of a BASELINE config with W virtual ranks on ONE GPU (the row-partitioned
multi-GPU code path: all-gather of H, halo exchange per squaring, rank-order scalar sums)
and print per-rank phase timings as JSON.  The ranks share one GPU, so the times show the
exchange and synchronisation overheads of the path, not multi-GPU scaling.

    python tools/virtual_ranks.py --config 5 --world 2
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2110_04493_b200 import binding as B
    from synth import make_config
    B.lib()
    H = make_config(args.config, scale_down=args.scale or None)
    W = args.world
    bounds = B.sexpm_partition_rows(H.n, np.diff(H.rowptr).astype(np.float64) ** 2, W)
    for rep in range(args.repeat):
        comms = B.sexpm_virtual_comm_create(W)
        res = [None] * W

        def rank_main(r):
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            Hl = H.rows(r0, r1)
            with torch.cuda.stream(s):
                t = [torch.from_numpy(a).cuda() for a in (Hl.rowptr, Hl.col, Hl.val)]
                s.synchronize()
                t0 = time.perf_counter()
                p = B.Plan(H.n, *t, 1e-16, row_begin=r0, row_end=r1, nccl_comm=comms[r], stream=s)
                p.run_only()
                s.synchronize()
                wall = time.perf_counter() - t0
                st = p.stats()
                p.close()
            N = int(st["N"])
            res[r] = {"rank": r, "rows": [r0, r1], "wall_ms": wall * 1e3,
                      "plan_ms": float(st["ms_plan"]), "taylor_ms": float(st["ms_taylor"]),
                      "squaring_ms": float(st["ms_squaring"]), "finalize_ms": float(st["ms_finalize"]),
                      "sq_exchange_ms": [round(float(x), 2) for x in st["sq_exchange_ms"][1:N + 1]],
                      "sq_kernel_ms": [round(float(x), 2) for x in st["sq_kernel_ms"][1:N + 1]],
                      "sq_fallback_rows": [int(x) for x in st["sq_fallback_rows"][1:N + 1]],
                      "sq_order_used": int(st["sq_order_used"]), "nnz_E_rank": int(st["nnz_out"]),
                      "order_host_ms": float(st["ms_order_host"]), "order_wait_ms": float(st["ms_order_wait"])}

        ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(W)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for c in comms:
            B.sexpm_nccl_comm_destroy(c)
        print(json.dumps({"config": args.config, "n": H.n, "world": W, "repeat": rep, "ranks": res}))


if __name__ == "__main__":
    main()
