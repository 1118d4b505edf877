"""One e^H of BASELINE config 5, then Y = E X for m = 1 and m = 64 (ncu target for k_spmm)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_04493_b200 import binding as B
from synth import make_config

def main():
    B.lib()
    H = make_config(5)
    dev = torch.device("cuda", 0)
    rp, ci, va = (torch.from_numpy(a).to(dev) for a in (H.rowptr, H.col, H.val))
    p = B.Plan(H.n, rp, ci, va, 1e-16)
    p.run_only()
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for m in (1, 64):
        X = torch.randn((H.n, m), dtype=torch.float64, device=dev, generator=g)
        p.apply(X)
    torch.cuda.synchronize()
    p.close()

if __name__ == "__main__":
    main()
