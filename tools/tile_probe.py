"""Experiment: config 5 in 2x4-tile order (rows of an 8-row block = a 2x4 patch of the grid):
squaring kernel time vs lexicographic order."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp
from paper_2110_04493_b200 import binding as B
from synth import make_config

def main():
    B.lib()
    H = make_config(5)
    G = 1449
    X, Y = np.meshgrid(np.arange(G), np.arange(G), indexing="ij")
    idx = (X * G + Y).ravel()
    Xr, Yr = X.ravel(), Y.ravel()
    tx, ty = int(sys.argv[1]), int(sys.argv[2])
    key = ((Xr // tx) * ((G + ty - 1) // ty) + (Yr // ty)) * (tx * ty) + (Xr % tx) * ty + (Yr % ty)
    perm = idx[np.argsort(key, kind="stable")]
    A = sp.csr_matrix((H.val, H.col, H.rowptr), shape=(H.n, H.n))[perm][:, perm].tocsr()
    A.sort_indices()
    dev = torch.device("cuda", 0)
    rp, ci, va = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in
                  (A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64)))
    for rep in range(2):
        p = B.Plan(H.n, rp, ci, va, 1e-16)
        p.run_only()
        st = p.stats()
        p.close()
    N = int(st["N"])
    print("tile", tx, ty, "sq_kernel_ms", [round(float(x), 1) for x in st["sq_kernel_ms"][1:N + 1]],
          "block_products", [float(x) for x in st["sq_block_products"][1:N + 1]],
          "bsr_blocks", [int(x) for x in st["sq_bsr_blocks"][1:N + 1]],
          "taylor_ms", round(float(st["ms_taylor"]), 1), "nnz_E", int(st["nnz_out"]), flush=True)

if __name__ == "__main__":
    main()
