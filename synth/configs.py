"""Seeded generators for the workloads of BASELINE.json `configs` (and the
small matrices the oracle pins use).

Recipe (stated again in DESIGN.md §"Inputs"):
  * heat conduction: H = r * (graph Laplacian of a grid with per-edge
    conductivities c_e), Dirichlet ends realised as "ghost" edges to the
    boundary (drawn from the same law), lexicographic node order
    idx = x*ny + y (2D) or (x*ny + y)*nz + z (3D).  Off-diagonal
    H_ij = r*c_e, diagonal H_ii = -r * sum of c_e over the incident edges
    (ghost edges included).  Uniform c_e = 1 gives r*tridiag(1,-2,1),
    r*(5-point) and r*(7-point) exactly (paper Eq. (2.1)-(2.2) heat context,
    PAPER.md §5.2 P:459 Toeplitz; BASELINE.json configs 1, 2, 4, 5).
  * structural state space, Eq. (2.1): Theta = [[0, I], [-M^-1 K,
    -M^-1 C]] with lumped unit mass M = I and C = 0, H = t*Theta.  K is the
    stiffness of a 2D scalar spring lattice (4-neighbour springs, boundary
    nodes tied to ground by springs; all k ~ U(0.5, 1.5)); DOFs are
    node-interleaved [u_0, v_0, u_1, v_1, ...] (a symmetric permutation of
    Eq. (2.1)'s block order; e^{P H P^T} = P e^H P^T) (BASELINE.json config 3).

Random numbers come from numpy's PCG64 seeded with `20211010 + config_id`
unless a seed is given; draws are made in a fixed order (edges along the
last axis first, then the next axis, ..., then ghost edges in node order).
No arithmetic of the paper's method lives here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 20211010


@dataclass
class CSR:
    """Canonical CSR: int64 rowptr (n+1), int32 col (sorted per row), float64 val,
    no explicit zeros, no duplicates."""

    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def rows(self, r0: int, r1: int) -> "CSR":
        """Row block [r0, r1) with global column indices (n stays global)."""
        a, b = int(self.rowptr[r0]), int(self.rowptr[r1])
        rp = (self.rowptr[r0:r1 + 1] - a).astype(np.int64)
        return CSR(self.n, rp, self.col[a:b].copy(), self.val[a:b].copy())

    def check(self) -> None:
        assert self.rowptr.dtype == np.int64 and self.col.dtype == np.int32
        assert self.val.dtype == np.float64
        assert self.rowptr[0] == 0 and np.all(np.diff(self.rowptr) >= 0)
        assert len(self.col) == len(self.val) == self.rowptr[-1]
        assert np.all(self.val != 0) and np.all(np.isfinite(self.val))
        if self.nnz:
            assert self.col.min() >= 0 and self.col.max() < self.n
            # strictly increasing columns inside each row
            d = np.diff(self.col.astype(np.int64))
            row_start = np.zeros(self.nnz, dtype=bool)
            row_start[self.rowptr[:-1][np.diff(self.rowptr) > 0]] = True
            assert np.all((d > 0) | row_start[1:])


def coo_to_csr(n: int, r: np.ndarray, c: np.ndarray, v: np.ndarray) -> CSR:
    """Sort (row, col); duplicates are not allowed; zeros are dropped."""
    r = np.asarray(r, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    keep = v != 0
    r, c, v = r[keep], c[keep], v[keep]
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    if len(r) > 1:
        dup = (np.diff(r) == 0) & (np.diff(c) == 0)
        if np.any(dup):
            raise ValueError("duplicate entries")
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, r + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int64)
    return CSR(n, rowptr, c.astype(np.int32), v.copy())


def dense_to_csr(A: np.ndarray) -> CSR:
    A = np.asarray(A, dtype=np.float64)
    r, c = np.nonzero(A)
    return coo_to_csr(A.shape[0], r, c, A[r, c])


def csr_to_dense(H: CSR) -> np.ndarray:
    D = np.zeros((H.n, H.n), dtype=np.float64)
    rows = np.repeat(np.arange(H.n), np.diff(H.rowptr))
    D[rows, H.col] = H.val
    return D


def _grid_laplacian(shape, r: float, coef, rng, ghost: bool = True) -> CSR:
    """r * weighted grid Laplacian. coef(rng, size) draws edge conductivities."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    idx = np.arange(n, dtype=np.int64).reshape(shape)
    rows, cols, vals = [], [], []
    diag = np.zeros(n, dtype=np.float64)
    nd = len(shape)
    # interior edges, last axis first
    for ax in reversed(range(nd)):
        sl_a = [slice(None)] * nd
        sl_b = [slice(None)] * nd
        sl_a[ax] = slice(0, shape[ax] - 1)
        sl_b[ax] = slice(1, shape[ax])
        a = idx[tuple(sl_a)].ravel()
        b = idx[tuple(sl_b)].ravel()
        c = coef(rng, a.size)
        rows += [a, b]
        cols += [b, a]
        vals += [r * c, r * c]
        np.add.at(diag, a, c)
        np.add.at(diag, b, c)
    if ghost:
        # Dirichlet ends: one ghost edge per boundary face of each boundary node
        for ax in reversed(range(nd)):
            for side in (0, shape[ax] - 1):
                sl = [slice(None)] * nd
                sl[ax] = side
                a = idx[tuple(sl)].ravel()
                c = coef(rng, a.size)
                np.add.at(diag, a, c)
                if shape[ax] == 1:  # both faces belong to the same node
                    c2 = coef(rng, a.size)
                    np.add.at(diag, a, c2)
                    break
    rows.append(np.arange(n))
    cols.append(np.arange(n))
    vals.append(-r * diag)
    return coo_to_csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _uniform(rng, size):
    return np.ones(size)


def tridiag(n: int, lo: float, d: float, up: float) -> CSR:
    """tridiag(lo, d, up) as in MATLAB gallery / PAPER.md §5.2."""
    i = np.arange(n)
    r = np.concatenate([i[1:], i, i[:-1]])
    c = np.concatenate([i[:-1], i, i[1:]])
    v = np.concatenate([np.full(n - 1, lo), np.full(n, d), np.full(n - 1, up)])
    return coo_to_csr(n, r, c, v)


def laplacian_2d(nx: int, ny: int, r: float, perturb: str | None = None, seed: int = 0) -> CSR:
    rng = np.random.default_rng(seed)
    if perturb is None:
        coef = _uniform
    elif perturb == "pm10":  # c_e = 1 + 0.1 U(-1, 1)
        coef = lambda g, s: 1.0 + 0.1 * g.uniform(-1.0, 1.0, s)  # noqa: E731
    elif perturb == "u0812":  # c_e ~ U(0.8, 1.2)
        coef = lambda g, s: g.uniform(0.8, 1.2, s)  # noqa: E731
    else:
        raise ValueError(perturb)
    return _grid_laplacian((nx, ny), r, coef, rng)


def laplacian_3d(nx: int, ny: int, nz: int, r: float, perturb: str | None = None, seed: int = 0) -> CSR:
    rng = np.random.default_rng(seed)
    if perturb is None:
        coef = _uniform
    elif perturb == "u0812":
        coef = lambda g, s: g.uniform(0.8, 1.2, s)  # noqa: E731
    else:
        raise ValueError(perturb)
    return _grid_laplacian((nx, ny, nz), r, coef, rng)


def neumann_laplacian_2d(nx: int, ny: int, r: float, seed: int = 0) -> CSR:
    """Zero-row-sum generator (no ghost edges): e^H 1 = 1 exactly."""
    rng = np.random.default_rng(seed)
    coef = lambda g, s: g.uniform(0.5, 1.5, s)  # noqa: E731
    return _grid_laplacian((nx, ny), r, coef, rng, ghost=False)


def structural_state_space(gx: int, gy: int, t: float, seed: int = 0) -> CSR:
    """H = t * [[0, I], [-K, 0]] with node-interleaved DOFs (Eq. (2.1),
    M = I lumped, C = 0)."""
    rng = np.random.default_rng(seed)
    coef = lambda g, s: g.uniform(0.5, 1.5, s)  # noqa: E731
    # K = weighted Laplacian + ground springs (same construction, r = -1 gives +K)
    K = _grid_laplacian((gx, gy), -1.0, coef, rng)  # stores +K (SPD)
    m = K.n
    n = 2 * m
    p = np.arange(m, dtype=np.int64)
    # du/dt = v : H[2p, 2p+1] = t
    r_i = [2 * p]
    c_i = [2 * p + 1]
    v_i = [np.full(m, t)]
    # dv/dt = -K u : H[2p+1, 2q] = -t K[p, q]
    kr = np.repeat(np.arange(m, dtype=np.int64), np.diff(K.rowptr))
    r_i.append(2 * kr + 1)
    c_i.append(2 * K.col.astype(np.int64))
    v_i.append(-t * K.val)
    return coo_to_csr(n, np.concatenate(r_i), np.concatenate(c_i), np.concatenate(v_i))


def random_banded(n: int, bw: int, density: float, scale: float, seed: int,
                  symmetric: bool = False) -> CSR:
    """Random sparse banded matrix with entries U(-1,1)*scale inside |i-j| <= bw."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - bw), min(n, i + bw + 1)):
            if rng.random() < density:
                A[i, j] = scale * rng.uniform(-1.0, 1.0)
    if symmetric:
        A = np.triu(A) + np.triu(A, 1).T
    return dense_to_csr(A)


def random_skew(n: int, bw: int, density: float, scale: float, seed: int) -> CSR:
    B = csr_to_dense(random_banded(n, bw, density, scale, seed))
    return dense_to_csr(B - B.T)


def diagonal(d) -> CSR:
    d = np.asarray(d, dtype=np.float64)
    n = len(d)
    i = np.arange(n)
    return coo_to_csr(n, i, i, d)


# --------------------------------------------------------------------------------------
# BASELINE.json configs (index = position in BASELINE.json "configs", 1-based here)
# --------------------------------------------------------------------------------------
CONFIGS = {
    1: dict(name="heat1d_n1000", desc="H = 0.5*tridiag(1,-2,1), n=1000, Dirichlet",
            n=1000),
    2: dict(name="heat2d_100x100_pm10", desc="H = 1.0*(5-pt Laplacian) 100x100, c_e = 1+0.1U(-1,1)",
            n=10_000),
    3: dict(name="structural_300x300", desc="H = 0.5*[[0,I],[-K,0]], K spring lattice 300x300, k~U(0.5,1.5), interleaved",
            n=180_000),
    4: dict(name="heat3d_64cube_u0812", desc="H = 0.25*(7-pt Laplacian) 64^3, c_e~U(0.8,1.2)",
            n=262_144),
    5: dict(name="heat2d_1449x1449", desc="H = 0.5*(5-pt Laplacian) 1449x1449, uniform",
            n=1449 * 1449),
}


def geometric_graph(n: int, avg_deg: float, norm1: float, seed: int) -> CSR:
    """N4 workload (§5.3's network matrices): a random
    geometric graph -- n points uniform in the unit square, an edge between points closer
    than r with pi r^2 n = avg_deg -- as H = beta A (communicability e^{beta A}), beta set so
    that ||H||_1 = norm1.  Nodes keep the random order of the points (unstructured input:
    the bandwidth is ~n until reordered)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = np.sqrt(avg_deg / (np.pi * n))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    rows = np.concatenate([pairs[:, 0], pairs[:, 1]])
    cols = np.concatenate([pairs[:, 1], pairs[:, 0]])
    deg = np.bincount(rows, minlength=n)
    beta = norm1 / max(int(deg.max()), 1)
    return coo_to_csr(n, rows, cols, np.full(len(rows), beta))


def make_config(cid: int, seed: int | None = None, scale_down: int | None = None) -> CSR:
    """Build BASELINE.json config `cid` (1..5).  `scale_down` (tests only) shrinks
    the grid side to the given value while keeping the law of the entries."""
    if seed is None:
        seed = SEED_BASE + cid
    if cid == 1:
        n = 1000 if scale_down is None else scale_down
        return _grid_laplacian((n,), 0.5, _uniform, np.random.default_rng(seed))
    if cid == 2:
        g = 100 if scale_down is None else scale_down
        return laplacian_2d(g, g, 1.0, "pm10", seed)
    if cid == 3:
        g = 300 if scale_down is None else scale_down
        return structural_state_space(g, g, 0.5, seed)
    if cid == 4:
        g = 64 if scale_down is None else scale_down
        return laplacian_3d(g, g, g, 0.25, "u0812", seed)
    if cid == 5:
        g = 1449 if scale_down is None else scale_down
        return laplacian_2d(g, g, 0.5, None, seed)
    raise ValueError(cid)
