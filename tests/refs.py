"""Independent references that PIN the oracle (test-side only).

None of these re-types the oracle's recurrence: they are closed forms
(modified-Bessel images for the 1D Dirichlet heat kernel, Kronecker products
for separable 2D operators, eigen closed forms for the paper's 2x2/3x3
matrices) or library / high-precision routines (mpmath 50-digit expm,
numpy long-double dense Taylor scaling-and-squaring).
"""
from __future__ import annotations

import mpmath as mp
import numpy as np
from scipy.special import ive


def heat1d_exact(n: int, r: float) -> np.ndarray:
    """e^{r tridiag(1,-2,1)} (Dirichlet, n points) by the method of images:
    E_ij = sum_m K(i-j-2m(n+1)) - K(i+j-2m(n+1)),  K(d) = e^{-2r} I_|d|(2r)
    (1-based i, j).  K is the lattice heat kernel; the odd reflection about
    0 and n+1 imposes the Dirichlet ends."""
    i = np.arange(1, n + 1)[:, None].astype(np.int64)
    j = np.arange(1, n + 1)[None, :].astype(np.int64)
    E = np.zeros((n, n))
    P = 2 * (n + 1)
    for m in range(-2, 3):
        E += ive(np.abs(i - j - m * P), 2 * r) - ive(np.abs(i + j - m * P), 2 * r)
    return E


def heat2d_uniform_exact(nx: int, ny: int, r: float) -> np.ndarray:
    """r*(5-point Dirichlet Laplacian) on nx x ny, idx = x*ny + y:
    H = r L_x (x) I + I (x) r L_y  =>  e^H = e^{r L_x} (x) e^{r L_y}."""
    return np.kron(heat1d_exact(nx, r), heat1d_exact(ny, r))


def heat2d_entry(nx: int, ny: int, r: float, row: int, cols: np.ndarray) -> np.ndarray:
    """Entries E[row, cols] of the 2D separable closed form without forming E."""
    x, y = divmod(int(row), ny)
    cx, cy = np.divmod(np.asarray(cols, dtype=np.int64), ny)
    return _k1(nx, r, x + 1, cx + 1) * _k1(ny, r, y + 1, cy + 1)


def _k1(n, r, i, j):
    j = np.asarray(j, dtype=np.int64)
    P = 2 * (n + 1)
    s = np.zeros(j.shape)
    for m in range(-2, 3):
        s += ive(np.abs(i - j - m * P), 2 * r) - ive(np.abs(i + j - m * P), 2 * r)
    return s


def mp_expm(A: np.ndarray, dps: int = 50) -> np.ndarray:
    """mpmath expm at `dps` digits (the paper's 50-digit vpa reference)."""
    with mp.workdps(dps):
        M = mp.matrix(A.tolist())
        E = mp.expm(M)
        return np.array([[float(E[i, j]) for j in range(A.shape[1])] for i in range(A.shape[0])])


def table1_matrices():
    """The five small matrices of PAPER.md §5.1."""
    return {
        1: np.array([[6.1, 1e6], [0.0, 6.1]]),
        2: np.array([[1.0, 1e6, 0.5e12], [0.0, 1.0, 1e6], [0.0, 0.0, 1.0]]),
        3: np.array([[1.0, np.sqrt(3) * 1e6], [0.0, 0.9]]),
        4: np.array([[-49.0, 24.0], [-64.0, 31.0]]),
        5: np.array([[1 + 1e-5, 1.0], [0.0, 1 - 1e-5]]),
    }


def table1_exact(k: int) -> np.ndarray:
    """Closed forms in 50-digit arithmetic of e^{H_k}, Table 1 inputs."""
    with mp.workdps(60):
        if k == 1:  # a I + b N, N^2 = 0 -> e^a (I + b N)
            a, b = mp.mpf("6.1"), mp.mpf(10) ** 6
            E = [[mp.e ** a, b * mp.e ** a], [0, mp.e ** a]]
        elif k == 2:  # I + N, N = [[0,b,c],[0,0,b],[0,0,0]] -> e (I + N + N^2/2)
            b, c = mp.mpf(10) ** 6, mp.mpf("0.5") * mp.mpf(10) ** 12
            E = [[mp.e, mp.e * b, mp.e * (c + b * b / 2)], [0, mp.e, mp.e * b], [0, 0, mp.e]]
        elif k == 3:  # upper triangular [[a, b],[0, d]]
            a, d, b = mp.mpf(1), mp.mpf("0.9"), mp.sqrt(3) * mp.mpf(10) ** 6
            E = [[mp.e ** a, b * (mp.e ** a - mp.e ** d) / (a - d)], [0, mp.e ** d]]
        elif k == 4:  # eigenvalues -1, -17; V = [[3, 1], [4, 2]] hmm -> compute by eigen
            H = mp.matrix([[-49, 24], [-64, 31]])
            # H v = lam v: lam=-1: v=(1,2); lam=-17: v=(3,4)
            V = mp.matrix([[1, 3], [2, 4]])
            D = mp.diag([mp.e ** -1, mp.e ** -17])
            Em = V * D * V ** -1
            assert mp.norm(H * V - V * mp.diag([-1, -17])) < mp.mpf(10) ** -40
            E = [[Em[0, 0], Em[0, 1]], [Em[1, 0], Em[1, 1]]]
        elif k == 5:
            dl = mp.mpf(10) ** -5
            a, d = 1 + dl, 1 - dl
            E = [[mp.e ** a, (mp.e ** a - mp.e ** d) / (a - d)], [0, mp.e ** d]]
        else:
            raise ValueError(k)
        return np.array([[float(x) for x in row] for row in E])


def dense_pim_longdouble(H: np.ndarray, M: int, N: int) -> np.ndarray:
    """Unfiltered PIM in numpy long double (80-bit on x86): T_0 = sum_{s=1}^M
    (H 2^-N)^s / s! built from explicit powers, T_i = 2 T + T T, E = I + T_N
    (Eqs. (2.6)-(2.7)); a dense reference for the filter-off oracle."""
    ld = np.longdouble
    A = H.astype(ld) * ld(2.0) ** (-N)
    n = H.shape[0]
    T = np.zeros((n, n), dtype=ld)
    P = np.eye(n, dtype=ld)
    fact = ld(1)
    for s in range(1, M + 1):
        P = P @ A
        fact *= s
        T += P / fact
    for _ in range(N):
        T = 2 * T + T @ T
    return (np.eye(n, dtype=ld) + T).astype(np.float64)
