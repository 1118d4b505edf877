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
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2110_04493_b200 import binding as B
    from synth import make_config
    H = make_config(args.config, scale_down=args.scale or None)
    dev = torch.device("cuda", 0)
    rp, ci, va = (torch.from_numpy(x).to(dev) for x in (H.rowptr, H.col, H.val))
    for _ in range(args.repeat):
        p = B.Plan(H.n, rp, ci, va, args.eps_tol, plan_norm=args.plan_norm)
        p.run_only()
        st = p.stats()
        p.close()
    M, N = int(st["M"]), int(st["N"])
    out = {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in st.items()}
    for k, v in list(out.items()):
        if isinstance(v, list):
            out[k] = v[: max(M, N) + 2]
    out["n"] = H.n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
