"""Run one e^H of a BASELINE config (optionally scaled down) through the C ABI and print
the library's per-step stats as JSON (used for ncu captures and step breakdowns)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--plan-norm", default="one")
    ap.add_argument("--eps-tol", type=float, default=1e-16)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--exact", type=int, default=0)
    ap.add_argument("--sq-order", type=int, default=1)
    ap.add_argument("--sym", type=int, default=-1)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2110_04493_b200 import binding as B
    from synth import make_config
    H = make_config(args.config, scale_down=args.scale or None)
    dev = torch.device("cuda", 0)
    rp, ci, va = (torch.from_numpy(x).to(dev) for x in (H.rowptr, H.col, H.val))
    for rep in range(args.repeat):
        p = B.Plan(H.n, rp, ci, va, args.eps_tol, plan_norm=args.plan_norm, kernel=args.kernel,
                   exact_products=args.exact, sq_order=args.sq_order,
                   sym_squaring=args.sym)
        p.run_only()
        st = p.stats()
        p.close()
        N = int(st["N"])
        sys.stderr.write(
            f"repeat {rep}: plan {st['ms_plan']:.1f} taylor {st['ms_taylor']:.1f} (numeric "
            f"{sum(st['taylor_numeric_ms']):.1f}) squaring {st['ms_squaring']:.1f} sq_numeric "
            f"{[round(float(x), 1) for x in st['sq_numeric_ms'][1:N + 1]]} sq_first "
            f"{[round(float(x), 1) for x in st['sq_first_ms'][1:N + 1]]} sq_fallback "
            f"{[int(x) for x in st['sq_fallback_rows'][1:N + 1]]} cache hits/misses/releases "
            f"{st['cache_hits']}/{st['cache_misses']}/{st['cache_releases']} order host/wait "
            f"{st['ms_order_host']:.1f}/{st['ms_order_wait']:.1f} ms cached "
            f"{st['cache_bytes_cached'] / 1e9:.1f} GB allocated {st['cache_bytes_allocated'] / 1e9:.1f} GB\n")
        sys.stderr.write(f"  taylor_numeric_ms {[round(float(x), 1) for x in st['taylor_numeric_ms'][2:int(st['M_eff']) + 1]]} "
                         f"taylor_fallback {[int(x) for x in st['taylor_fallback_rows'][2:int(st['M_eff']) + 1]]}\n")
        sys.stderr.write(f"  sq_kernel_ms {[round(float(x), 1) for x in st['sq_kernel_ms'][1:N + 1]]} "
                         f"block products {[float(x) for x in st['sq_block_products'][1:N + 1]]} "
                         f"fmas {[float(x) for x in st['sq_fmas'][1:N + 1]]} sym {st['sq_sym_used']} "
                         f"assemble_ms {[round(float(x), 1) for x in st['sq_assemble_ms'][1:N + 1]]}\n")
    M, N = int(st["M"]), int(st["N"])
    out = {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in st.items()}
    for k, v in list(out.items()):
        if isinstance(v, list):
            out[k] = v[: max(M, N) + 2]
    out["n"] = H.n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
